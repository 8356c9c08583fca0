// Drop-in for rgfvar's include/rgf/covariance.hpp (covariance.hpp:17-79).
// Put include/rgf_b200/dropin ahead of the reference's include directory;
// every `#include "rgf/covariance.hpp"` (diagnostics.hpp:13, solver.hpp:13,
// rgfvar.cpp, the tests) then resolves here. The reference's types.hpp and
// grid.hpp are used as they are; HorizontalCovarianceOp runs on the device
// through librgf_b200.so. See INTEGRATION.md.
#pragma once
#ifndef RGF_B200_USE_EIGEN
#define RGF_B200_USE_EIGEN
#endif
#include "rgf_b200/covariance.hpp"
