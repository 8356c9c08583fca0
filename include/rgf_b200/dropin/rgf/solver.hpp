// Drop-in for rgfvar's include/rgf/solver.hpp (solver.hpp:19-55): SolveOptions,
// Analysis, CostReport, cost and solve with the CG loop device-resident.
// ObsSet and obs_operator(_transpose)/misfit stay the reference's (obs.hpp,
// obs.cpp). See INTEGRATION.md.
#pragma once
#ifndef RGF_B200_USE_EIGEN
#define RGF_B200_USE_EIGEN
#endif
#include "rgf_b200/solver.hpp"
