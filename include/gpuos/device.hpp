// Reference-compatible include path: gpuos/device.hpp. Declarations live in the
// B200 library's grouped headers listed below.
#pragma once
#include "gpuos/core.hpp"
#include "gpuos/replay.hpp"
