#pragma once
// Umbrella header of the B200 drop-in (reference: proj/include/fgfrft/fgfrft.hpp). ADDITIVE: with
// the reference headers on the include path (Eigen builds, include/ before proj/include) this is
// the reference's own umbrella, whose includes of transform.hpp / spectral.hpp / learn.hpp resolve
// to the drop-in (the hot path) and everything else (graph, io, metrics, bench, adam, image, ...)
// to the reference. Without Eigen it gathers the drop-in and its standalone restatements of the
// input-preparation headers (graph, gft, rng, metrics).
#include "fgfrft/matrix.hpp"

#if defined(FGFRFT_HAVE_EIGEN) && __has_include_next(<fgfrft/fgfrft.hpp>)
#include_next <fgfrft/fgfrft.hpp>
#else
#include "fgfrft/errors.hpp"
#include "fgfrft/gft.hpp"
#include "fgfrft/graph.hpp"
#include "fgfrft/learn.hpp"
#include "fgfrft/metrics.hpp"
#include "fgfrft/rng.hpp"
#include "fgfrft/sinc.hpp"
#include "fgfrft/spectral.hpp"
#include "fgfrft/transform.hpp"
#endif
