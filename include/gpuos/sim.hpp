// Reference-compatible include path: gpuos/sim.hpp. Declarations live in the
// B200 library's grouped headers listed below.
#pragma once
#include "gpuos/scenario.hpp"
#include "gpuos/replay.hpp"
