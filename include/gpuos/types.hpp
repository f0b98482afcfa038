// Reference-compatible include path: gpuos/types.hpp. Declarations live in the
// B200 library's grouped headers listed below.
#pragma once
#include "gpuos/core.hpp"
