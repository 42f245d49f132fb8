#pragma once
// Umbrella header of the B200 drop-in (reference: proj/include/fgfrft/fgfrft.hpp): the hot path
// (transform) and its adjacent consumers (spectral form / exact operator, cascaded order learning).
// Graph building, IO and the CLI stay with the reference.
#include "fgfrft/errors.hpp"
#include "fgfrft/gft.hpp"
#include "fgfrft/learn.hpp"
#include "fgfrft/matrix.hpp"
#include "fgfrft/sinc.hpp"
#include "fgfrft/spectral.hpp"
#include "fgfrft/transform.hpp"
