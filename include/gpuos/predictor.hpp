// Reference-compatible include path: gpuos/predictor.hpp. Declarations live in the
// B200 library's grouped headers listed below.
#pragma once
#include "gpuos/policy.hpp"
