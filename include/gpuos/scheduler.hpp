// Reference-compatible include path: gpuos/scheduler.hpp. Declarations live in the
// B200 library's grouped headers listed below.
#pragma once
#include "gpuos/replay.hpp"
#include "gpuos/tpc_scheduler.hpp"
