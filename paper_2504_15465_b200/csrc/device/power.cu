// Power / clock telemetry and DVFS actuation for the B200 backend through
// NVML, loaded at run time (dlopen: no link-time dependency, and a host
// without the driver library reports GPUOS_E_CUDA instead of failing to
// load). The reference's power manager decides a frequency per interval
// (power_manager.cpp:27-105) and its engine integrates modelled power into
// energy (device.cpp:221-242); on the B200 the energy is the GPU's own
// counter and a decided frequency can be applied as a locked SM clock.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvml.h>

#include <mutex>
#include <type_traits>

#include "gpuos_dev.h"

namespace {

struct Nvml {
  bool ok = false;
  nvmlReturn_t (*init)() = nullptr;
  nvmlReturn_t (*by_pci)(const char*, nvmlDevice_t*) = nullptr;
  nvmlReturn_t (*energy)(nvmlDevice_t, unsigned long long*) = nullptr;
  nvmlReturn_t (*clock)(nvmlDevice_t, nvmlClockType_t, unsigned int*) = nullptr;
  nvmlReturn_t (*power)(nvmlDevice_t, unsigned int*) = nullptr;
  nvmlReturn_t (*reasons)(nvmlDevice_t, unsigned long long*) = nullptr;
  nvmlReturn_t (*lock)(nvmlDevice_t, unsigned int, unsigned int) = nullptr;
  nvmlReturn_t (*unlock)(nvmlDevice_t) = nullptr;
};

Nvml& nvml() {
  static Nvml n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnvidia-ml.so.1", RTLD_NOW | RTLD_LOCAL);
    if (!h) return;
    auto sym = [&](auto& fn, const char* name) { fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name)); };
    sym(n.init, "nvmlInit_v2");
    sym(n.by_pci, "nvmlDeviceGetHandleByPciBusId_v2");
    sym(n.energy, "nvmlDeviceGetTotalEnergyConsumption");
    sym(n.clock, "nvmlDeviceGetClockInfo");
    sym(n.power, "nvmlDeviceGetPowerUsage");
    sym(n.reasons, "nvmlDeviceGetCurrentClocksEventReasons");
    if (!n.reasons) sym(n.reasons, "nvmlDeviceGetCurrentClocksThrottleReasons");
    sym(n.lock, "nvmlDeviceSetGpuLockedClocks");
    sym(n.unlock, "nvmlDeviceResetGpuLockedClocks");
    n.ok = n.init && n.by_pci && n.energy && n.clock && n.init() == NVML_SUCCESS;
  });
  return n;
}

int handle_of(int32_t cuda_device, nvmlDevice_t* h) {
  Nvml& n = nvml();
  if (!n.ok) return GPUOS_E_CUDA;
  char bus[32] = {};
  if (cudaDeviceGetPCIBusId(bus, sizeof(bus), cuda_device) != cudaSuccess) return GPUOS_E_CUDA;
  return n.by_pci(bus, h) == NVML_SUCCESS ? GPUOS_OK : GPUOS_E_CUDA;
}

}  // namespace

extern "C" int gpuos_power_sample(int32_t cuda_device, gpuos_power_sample_t* out) {
  if (!out) return GPUOS_E_CONFIG;
  nvmlDevice_t h;
  if (const int rc = handle_of(cuda_device, &h); rc != GPUOS_OK) return rc;
  Nvml& n = nvml();
  *out = gpuos_power_sample_t{};
  unsigned long long mj = 0, why = 0;
  unsigned int sm = 0, mem = 0, mw = 0;
  if (n.energy(h, &mj) != NVML_SUCCESS) return GPUOS_E_CUDA;
  n.clock(h, NVML_CLOCK_SM, &sm);
  n.clock(h, NVML_CLOCK_MEM, &mem);
  if (n.power) n.power(h, &mw);
  if (n.reasons) n.reasons(h, &why);
  out->energy_mj = mj;
  out->sm_mhz = sm;
  out->mem_mhz = mem;
  out->power_mw = mw;
  out->clock_event_reasons = why;
  return GPUOS_OK;
}

extern "C" int gpuos_power_lock_sm_clock(int32_t cuda_device, uint32_t mhz) {
  nvmlDevice_t h;
  if (const int rc = handle_of(cuda_device, &h); rc != GPUOS_OK) return rc;
  Nvml& n = nvml();
  if (!n.lock || !n.unlock) return GPUOS_E_CUDA;
  const nvmlReturn_t r = mhz == 0 ? n.unlock(h) : n.lock(h, mhz, mhz);
  return r == NVML_SUCCESS ? GPUOS_OK : GPUOS_E_CUDA;
}
