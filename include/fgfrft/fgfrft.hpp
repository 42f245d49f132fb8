#pragma once
// Umbrella header of the B200 drop-in (reference: proj/include/fgfrft/fgfrft.hpp). Only the
// hot-path headers are provided; graph building, spectral solvers, learning loops and IO stay
// with the reference.
#include "fgfrft/errors.hpp"
#include "fgfrft/gft.hpp"
#include "fgfrft/matrix.hpp"
#include "fgfrft/sinc.hpp"
#include "fgfrft/transform.hpp"
