// Reference-compatible include path: gpuos/workload.hpp. Declarations live in the
// B200 library's grouped headers listed below.
#pragma once
#include "gpuos/tenants.hpp"
