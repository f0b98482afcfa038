/*
 * gpuos_sim.h — C ABI of the host scheduler path ("plugin" entry points).
 *
 * The reference exposes the path as C++ (Scheduler + DeviceEngine,
 * proj/include/gpuos/scheduler.hpp:72-102, and run_scenario,
 * proj/include/gpuos/sim.hpp:46); its CLI (proj/tools/gpuos_sim.cpp:72-77)
 * is a thin loop over run_scenario. These entry points expose the same
 * operations to any FFI (Python ctypes in bench.py and tests/):
 *
 *   gpuos_session_open / _run / _close   run_scenario (sim.cpp:375-461) on a
 *                                        chosen backend: "replay" (bit-exact
 *                                        with the reference), "b200" (live
 *                                        persistent dispatcher) or "mirror"
 *                                        (replay timing + GPU execution and
 *                                        verification of every atom)
 *   gpuos_plan_atoms ...                 the pure policy functions of the hot
 *                                        path (atomizer.cpp, rightsizer.cpp,
 *                                        device.cpp:56-72, predictor.cpp)
 *
 * Requests and results are JSON text (schema in paper_2504_15465_b200/api.py).
 * Return codes: 0 ok, 2 configuration error, 3 invariant error (the
 * reference CLI's exit codes, gpuos_sim.cpp:240-249).
 */
#ifndef GPUOS_SIM_H_
#define GPUOS_SIM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gpuos_session gpuos_session;

int gpuos_session_open(const char* request_json, gpuos_session** out);
/* overrides_json may be NULL; *result_json is malloc'd (gpuos_free_text). */
int gpuos_session_run(gpuos_session* s, const char* overrides_json, char** result_json);
int gpuos_session_close(gpuos_session* s);
/* One-shot convenience: open + run + close. */
int gpuos_run_json(const char* request_json, char** result_json);
void gpuos_free_text(char* text);
/* Dispatcher overhead probe on the live path (serial round trips of empty
 * atoms, publish -> first block start, pipelined empty-atom rate); options
 * {"serial", "pipelined", "depth", "tpc", "device", "workers_per_sm"}.    */
int gpuos_probe_dispatch(const char* opts_json, char** result_json);
const char* gpuos_sim_last_error(void);

/* ---- pure policy functions (parity against the reference's vectors) ---- */
/* Writes up to cap [lo, hi) pairs; returns the atom count or -2. */
int64_t gpuos_plan_atoms(int64_t total_blocks, int64_t predicted_ns,
                         int64_t atom_duration_ns, int64_t min_blocks_per_atom,
                         int64_t* out_ranges, int64_t cap);
int gpuos_should_atomize(int64_t predicted_ns, int64_t total_blocks,
                         int64_t atom_duration_ns, double disable_factor);
int gpuos_filter_cap(int64_t total_blocks, int32_t occupancy, int32_t total_tpcs);
int gpuos_fit_scaling(int64_t l1_ns, int64_t lT_ns, int32_t T, double* m_ns,
                      double* b_ns, int32_t* valid);
int gpuos_choose_tpcs(double m_ns, double b_ns, int32_t valid, int32_t t_alloc,
                      double slip_k, int32_t cap);
int gpuos_choose_tpcs_wave(double m_ns, double b_ns, int32_t valid,
                           int32_t t_alloc, double slip_k, int64_t blocks,
                           int32_t occ);
/* B200 extension of the right-sizer (RightsizerConfig::plateau): the
 * three-point measured-curve fit l(t) = max(m/t + b, floor) through
 * (1, l1), (t_mid, l_mid) and the full-width plateau lT, and the wave-aware
 * chooser on that model (floor_ns = 0 is exactly gpuos_choose_tpcs_wave). */
int gpuos_fit_scaling_plateau(int64_t l1_ns, int32_t t_mid, int64_t l_mid_ns, int64_t lT_ns,
                              int32_t T, double* m_ns, double* b_ns, double* floor_ns,
                              int32_t* valid);
int gpuos_choose_tpcs_wave_floor(double m_ns, double b_ns, double floor_ns, int32_t valid,
                                 int32_t t_alloc, double slip_k, int64_t blocks, int32_t occ);
/* The measured-curve right-sizer's search step (RightsizerConfig::plateau):
 * n samples (width t[i], mean latency l_ns[i]) -> *ok = narrowest width
 * within slip_k of the widest sample's latency, *probe = next width to
 * measure (0: converged). */
int gpuos_choose_measured(const int32_t* t, const double* l_ns, int32_t n, double slip_k,
                          int32_t* ok, int32_t* probe);
/* Block latency and the closed-form lone-kernel latency at frequency f_mhz
 * for the default A100-like table (540..1410 MHz). */
int64_t gpuos_block_latency(int64_t d0_ns, double s, int32_t f_mhz);
int64_t gpuos_reference_kernel_latency(int64_t blocks, int64_t d0_ns, double s,
                                       int32_t occ, int32_t t, int32_t f_mhz);
int32_t gpuos_select_frequency(double S, double slip_k);
/* Predictor: replays `n` records (t, f, blocks, observed) for one key, then
 * answers `q` queries (t, f, blocks) into out_latency / out_confidence. */
int gpuos_predictor_replay(const int64_t* records, int32_t n,
                           const int64_t* queries, int32_t q,
                           int64_t* out_latency, int32_t* out_confidence);

#ifdef __cplusplus
}
#endif

#endif /* GPUOS_SIM_H_ */
