/*
 * poas_b200.h -- C ABI of the B200-native POAS co-executed GEMM.
 *
 * The reference (arXiv 2209.10245, /root/reference/proj) is a C++20 library
 * with no FFI of its own; these entry points are what a foreign caller (or
 * the reference's own CLI) binds to reach the same
 * predict -> optimize -> adapt -> schedule -> execute path. Each entry point
 * names the reference interface it replaces.
 *
 * Conventions
 *  - Plain C types only; no exceptions cross the boundary.
 *  - Every int-returning function returns POAS_OK (0) or an error code;
 *    poas_b200_last_error() then holds a thread-local message.
 *  - Strings returned through char** are malloc'ed by the library and must
 *    be released with poas_b200_free().
 *  - Matrices are row-major: A[m x k] (lda), B[k x n] (ldb), C[m x n] (ldc).
 */
#ifndef POAS_B200_H
#define POAS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes: poas::errc (reference proj/include/poas/error.hpp:8-21) in
 * declaration order, shifted by one so that 0 means success. */
enum {
  POAS_OK = 0,
  POAS_E_INVALID_ARGUMENT = 1,
  POAS_E_DEGENERATE_SAMPLES = 2,
  POAS_E_NON_POSITIVE_TIME = 3,
  POAS_E_BACKEND_FAILURE = 4,
  POAS_E_PARSE_FAILURE = 5,
  POAS_E_NOT_ROW_ALIGNED = 6,
  POAS_E_UNALIGNABLE_K = 7,
  POAS_E_NO_FEASIBLE_TILING = 8,
  POAS_E_TOO_MANY_DEVICES = 9,
  POAS_E_MISSING_DEVICE = 10,
  POAS_E_NUMERICAL_FAILURE = 11,
  POAS_E_HASH_MISMATCH = 12,
  POAS_E_IO_FAILURE = 13,
  POAS_E_CUDA = 100,    /* CUDA runtime / driver error (message has details) */
  POAS_E_INTERNAL = 101 /* any other C++ exception */
};

enum { POAS_DTYPE_F32 = 0, POAS_DTYPE_F16 = 1, POAS_DTYPE_BF16 = 2 };

const char* poas_b200_last_error(void);
void poas_b200_free(void* p);
const char* poas_b200_version(void);

/* ------------------------------------------------------------------------
 * Plan (Optimize -> Adapt -> Schedule). Pure host code, byte-identical to
 * the reference for the same profile.
 * --------------------------------------------------------------------- */

/* solve_split -> build_tile_plan -> build_schedule -> format_schedule.
 * Replaces cmd_plan (proj/tools/poas.cpp:66-83) over solve_split
 * (proj/include/poas/optimizer.hpp:67), build_tile_plan (adapter.hpp:71-72),
 * build_schedule (scheduler.hpp:35), format_schedule (scheduler.hpp:45).
 * `profile_text` is a "poas-profile v1" file body. */
int poas_b200_plan(const char* profile_text, int64_t m, int64_t n, int64_t k,
                   char** schedule_json);

/* poas_b200_plan with a planner policy: "reference" (== poas_b200_plan),
 * "best-subset" -- an opt-in B200 extension that also plans every subset of
 * units and keeps the smallest predicted makespan (the reference LP charges
 * every unit the full B transfer; proj/src/optimizer.cpp:21-32,257-275) --
 * or "overlap": best-subset with each link unit's rows cut into row parts
 * whose copies overlap compute (full-duplex link), predicted by the
 * pipelined timeline of poas/overlap.hpp; run it with an "overlap=1"
 * executor (the paper's "memory copies with overlap"). */
int poas_b200_plan_policy(const char* profile_text, int64_t m, int64_t n, int64_t k,
                          const char* policy, char** schedule_json);

/* SM partition of one GPU between its tensor unit and its CUDA-core unit,
 * chosen by the planner (B200 extension; no reference counterpart: the
 * reference's units are fixed devices). The profile describes the units at
 * their measured budgets tc_sms / simt_sms; each candidate CUDA-core budget
 * (simt_budgets[i], 0 = unit left out and its SMs lent to the tensor unit)
 * scales the units' compute slopes inversely with their SM counts and the
 * CUDA-core unit's resident-operand bandwidth with its budget, and is
 * planned with `policy`. *out_json: {"best": index, "candidates": [{"simt_sms",
 * "tc_sms", "makespan", "rows": {id: rows}}]}; free with poas_b200_free. */
int poas_b200_plan_partitions(const char* profile_text, int64_t m, int64_t n, int64_t k,
                              const char* tc_id, int tc_sms, const char* simt_id, int simt_sms,
                              const int* simt_budgets, int count, const char* policy,
                              char** out_json);

/* Predict again after the partition decision: `profile_text` with unit
 * `unit_id`'s measured model (slope, intercept, bandwidth, ops window)
 * replaced by the same unit's entry in `unit_profile_text` -- the unit
 * re-probed on its decided SM budget (e.g. a poas_b200_profile_machine of
 * that one unit). Identity, kind, priority, alignment and the machine hash
 * are unchanged. *out_profile: poas-profile v1 text (poas_b200_free). */
int poas_b200_profile_splice_unit(const char* profile_text, const char* unit_profile_text,
                                  const char* unit_id, char** out_profile);

/* standalone_schedule (proj/include/poas/scheduler.hpp:40-41). */
int poas_b200_plan_standalone(const char* profile_text, const char* device_id, int64_t m,
                              int64_t n, int64_t k, char** schedule_json);

/* The intermediate WorkloadSplit of solve_split (optimizer.hpp:30-35) as
 * JSON with %.17g doubles: {"makespan","lp_objective","lp_iterations",
 * "shares":[{"id","rows","ops","fraction","copy_in":[s,e],"compute":[s,e],
 * "copy_out":[s,e],"finish"}]}. */
int poas_b200_split(const char* profile_text, int64_t m, int64_t n, int64_t k, char** split_json);

/* oracle_grid_search / _serial (optimizer.hpp:77-80): same JSON as above. */
int poas_b200_oracle_split(const char* profile_text, int64_t m, int64_t n, int64_t k,
                           int64_t resolution, int parallel, char** split_json);

/* build_tile_plan (adapter.hpp:71-72) for a given whole-row assignment
 * (evaluate_rows, optimizer.hpp:62-63) in machine order:
 * {"devices":[{"id","rows","k_prime","sq","window_fallback","tiles":[[m,k,n],...]}]} */
int poas_b200_tile_plan(const char* profile_text, int64_t m, int64_t n, int64_t k,
                        const int64_t* rows, size_t count, char** plan_json);

/* parse_schedule -> format_schedule (scheduler.hpp:45-46): canonical bytes,
 * or an error for a malformed schedule. */
int poas_b200_schedule_roundtrip(const char* schedule_json, char** canonical_json);

/* parse_profile -> format_profile (profiler.hpp:71-72). */
int poas_b200_profile_roundtrip(const char* profile_text, char** canonical_text);

/* machine_hash (device_model.hpp:135) of a profile, 16 hex chars + NUL. */
int poas_b200_machine_hash(const char* profile_text, char out[17]);

/* fit_linear (device_model.hpp:77): centred OLS in long double. */
int poas_b200_fit_linear(const uint64_t* ops, const double* seconds, size_t count,
                         double* slope, double* intercept);

/* transfer_bytes (device_model.hpp:93) for device `device_id` of a profile. */
int poas_b200_transfer_bytes(const char* profile_text, const char* device_id, uint64_t ops,
                             int64_t m, int64_t n, int64_t k, uint64_t* in_bytes,
                             uint64_t* out_bytes);

/* Dense two-phase Bland simplex (simplex.hpp:25): minimise c.x s.t.
 * Aeq x = beq, Age x >= bge, x >= 0. Matrices row-major. */
int poas_b200_simplex(int num_vars, const double* objective, int n_eq, const double* eq_a,
                      const double* eq_b, int n_ge, const double* ge_a, const double* ge_b,
                      double* x_out, double* objective_out, long* iterations_out);

/* ------------------------------------------------------------------------
 * Predict: compute units and the profiler. A unit is one concurrently
 * running share of the machine: the host CPU cores, the CUDA cores of one
 * GPU (SIMT fp32 kernel) or its tensor cores (tcgen05 kernel).
 *
 * Unit spec strings: "<id>=<kind>[:key=value]*" with kind cpu|gpu|xpu
 *   cpu : threads=<n>                       (0 = all online cores)
 *   gpu : dev=<cuda ordinal>, sms=<n>       (SM budget, 0 = all), exclusive=0|1
 *   xpu : dev=<ordinal>, sms=<n>, dtype=bf16|f16, elem=<bytes on the link>
 * and, for any kind: probe=MIN-MAX (the unit's own probe side range),
 * link=pcie|hbm|fused (what time_transfer measures: pinned host memory
 * over PCIe; resident operands streamed into the unit's own SMs; or
 * resident operands streamed inside the probed GEMM itself -- a tensor
 * unit's fat share -- reported as a nominal 1 PB/s), align=<rows> (xpu);
 * GPU units: preroll=<ms> (each timed probe follows back-to-back launches
 * of the same GEMM worth that long: probes in the continuous-load, power-
 * capped regime a co-executed step runs in; default 0 = one launch).
 * --------------------------------------------------------------------- */
typedef struct poas_unit_s* poas_unit_t;

int poas_b200_unit_create(const char* spec, poas_unit_t* out);
void poas_b200_unit_destroy(poas_unit_t unit);
/* DeviceBackend::time_gemm (proj/include/poas/backend.hpp:15-17). */
int poas_b200_time_gemm(poas_unit_t unit, int64_t side, double* seconds);
/* DeviceBackend::time_transfer (backend.hpp:19-21): pinned host -> device. */
int poas_b200_time_transfer(poas_unit_t unit, uint64_t bytes, double* seconds);
/* DeviceBackend::has_transfers (backend.hpp:23). */
int poas_b200_has_transfers(poas_unit_t unit);

/* profile_machine (proj/include/poas/simulator.hpp:28) over real units:
 * run_compute_probes + run_bandwidth_probe per unit, fit_machine, and
 * format_profile. `units` is a ';'-separated list of unit specs;
 * `profiling` is "probes=..,repetitions=..,cpu_min_side=..,cpu_max_side=..,
 * accel_min_side=..,accel_max_side=..,bandwidth_payload=.." (any subset;
 * defaults as ProfilingConfig, profiler.hpp:28-38). `bus` is 1 or 0. */
int poas_b200_profile_machine(const char* units, const char* profiling, int bus,
                              char** profile_text);

/* The same Predict pipeline over caller-supplied backends: the C form of
 * the reference plugin `class DeviceBackend` (proj/include/poas/backend.hpp:
 * 11-24), for a caller whose timing source is its own -- e.g. the
 * reference's SyntheticBackend (proj/src/simulator.cpp:25-45) or recorded
 * measurements. Per backend, exactly what profile_machine
 * (proj/src/simulator.cpp:53-74) does per device: run_compute_probes over
 * the kind's side range (or probe_min/max_side when both > 0),
 * run_bandwidth_probe when time_transfer is non-NULL, align for xpu,
 * cache_bytes for cpu; then fit_machine and format_profile. A callback
 * returning <= 0 or a non-finite time fails with POAS_E_NON_POSITIVE_TIME
 * (profiler.cpp:47-50,67-69). Priorities: all >= 0 (fixed) or all -1
 * (ranked by modelled throughput), else POAS_E_INVALID_ARGUMENT. */
enum { POAS_KIND_CPU = 0, POAS_KIND_GPU = 1, POAS_KIND_XPU = 2 };
typedef struct {
  const char* id;
  int kind;               /* POAS_KIND_* */
  uint32_t elem_size;
  int64_t align;          /* used for xpu */
  uint64_t cache_bytes;   /* used for cpu */
  int priority;           /* >= 0 fixed; -1 ranked */
  int64_t probe_min_side, probe_max_side;
  double (*time_gemm)(void* ctx, int64_t side);
  double (*time_transfer)(void* ctx, uint64_t bytes);  /* NULL: has_transfers() false */
  void* ctx;
} poas_probe_backend;
int poas_b200_profile_backends(const poas_probe_backend* backends, size_t count,
                               const char* profiling, int bus, char** profile_text);

/* ------------------------------------------------------------------------
 * Execute: the real replacement of simulate() (simulator.hpp:68-69).
 * --------------------------------------------------------------------- */
typedef struct poas_executor_s* poas_executor_t;
typedef struct poas_comm_s* poas_comm_t;  /* see "Multi-GPU" below */

typedef struct {
  int64_t m, n, k;
  /* Host fp32 operands. Pinned memory (cudaHostAlloc / cudaHostRegister)
   * is the fast path; pageable ranges a GPU unit copies are page-locked
   * (cudaHostRegister) for the duration of execute() and released after
   * it, which costs time on every call. Required when
   * resident == 0 -- every GPU unit then copies its A rows and all of B over
   * its link, computes, and copies its C rows back, inside execute() -- and
   * whenever a CPU unit has rows (it computes in place on these). */
  const float* a_host;
  int64_t lda_host;
  const float* b_host;
  int64_t ldb_host;
  float* c_host;
  int64_t ldc_host;
  /* resident == 1: operands already in HBM of the GPU the units run on.
   * CUDA-core units read a_dev/b_dev (fp32); tensor units read a16/b16
   * (bf16 or fp16, row pitch a multiple of 8 elements) when given, else
   * convert a_dev/b_dev on the device. GPU units write c_dev rows. */
  const float* a_dev;
  int64_t lda_dev;
  const float* b_dev;
  int64_t ldb_dev;
  const void* a16_dev;
  int64_t lda16_dev;
  const void* b16_dev;
  int64_t ldb16_dev;
  float* c_dev;
  int64_t ldc_dev;
  int resident;
  /* Optional (resident == 1): B arrives in `b_panels` column panels (e.g.
   * chunks of a broadcast). Panel p = columns [p*n/P, (p+1)*n/P) stored
   * contiguously as a [k x n/P] matrix at b_dev + p*k*(n/P) (and likewise
   * b16_dev); each GPU unit waits on b_ready[p] (a cudaEvent_t recorded on
   * the same GPU after the panel landed) before computing that panel, so the
   * transfer of later panels overlaps compute on earlier ones. n must be a
   * multiple of b_panels. b_panels <= 1: B is one row-major matrix and, if
   * b_ready is given, every GPU unit waits on b_ready[0] before computing. */
  int b_panels;
  void* const* b_ready;
  /* Optional (resident == 0): host copies of A and B in the tensor units'
   * 16-bit type. A tensor unit whose link element size is 2 (elem=2) then
   * copies these -- half the bytes of fp32, the reference's XPU link model
   * (elem_size 2) -- instead of copying fp32 and converting on the GPU.
   * Row pitches are in elements. */
  const void* a16_host;
  int64_t lda16_host;
  const void* b16_host;
  int64_t ldb16_host;
  /* Optional (resident == 1, b_panels > 1): device readiness flags, one int
   * per panel. A tensor unit then computes every panel in ONE launch whose
   * producers start on panel p once b_flags[p] >= b_epoch (the deliverer
   * writes the flags in panel order, e.g. poas_b200_signal_flag on its
   * stream after each panel's broadcast) instead of one launch per panel
   * behind b_ready[p]. n/b_panels must be a multiple of 256. Units without
   * this path (CUDA cores) still wait on b_ready. */
  const int* b_flags;
  int b_epoch;
  /* Optional (resident == 1): row-sharded multi-GPU run. The executor
   * broadcasts B itself every repeat over this communicator (B registered
   * with poas_b200_comm_register_b, b_panels panels): rank 0's b16_dev /
   * b_dev are served, the other ranks' units read the comm's receive
   * buffers; b_flags / b_ready must be NULL (the executor signals B).
   * b_transport: 0 = copy-engine chain over CUDA IPC (no SMs), 1 = NCCL. */
  poas_comm_t comm;
  int b_transport;
} poas_gemm_io;

/* One executor per process per machine description (same unit specs as
 * the profile that produced the schedule; "bus=0|1" token for the link
 * topology, default shared; "lend=0|1": when a schedule leaves all but one
 * unit of a GPU idle, the busy unit runs on their SMs too, default 1;
 * "overlap=0|1": host-operand runs overlap every link unit's copies with its
 * GEMMs over the schedule's grid of row parts x column panels (its tiles) on
 * separate H2D / compute / D2H streams, default 0 = the paper's synchronous
 * copy-in, compute, copy-out; "pipeline=0|1": with overlap and one busy
 * streamed tensor unit, consecutive repeats overlap too, default 0). */
int poas_b200_executor_create(const char* units, poas_executor_t* out);
void poas_b200_executor_destroy(poas_executor_t ex);
/* machine_identity_hash over the executor's units (device_model.hpp:130). */
int poas_b200_executor_hash(poas_executor_t ex, char out[17]);

/* Runs the schedule `repeats` times, every unit's share concurrently (one
 * CUDA stream per GPU unit, host threads for the CPU unit), each phase
 * timed on a common clock. report_json (optional) has the shape of the
 * reference's simulate report (proj/tools/poas.cpp:85-114): per device
 * copy_in/compute/copy_out/copy/finish {measured, predicted, error_pct},
 * makespans and RMSE. Rows are contiguous in schedule order. */
int poas_b200_execute(poas_executor_t ex, const char* schedule_json, const poas_gemm_io* io,
                      int repeats, char** report_json);

/* ------------------------------------------------------------------------
 * Dynamic scheduling (paper §3.4.2; the reference has only
 * the static scheduler -- B200 extension).
 * --------------------------------------------------------------------- */
/* The profile with every unit of an execution report (poas_b200_execute's
 * report_json) re-fitted: slope and intercept scaled by 1 + alpha (r - 1),
 * r = measured/predicted compute; link bandwidth likewise from the copy
 * phases. alpha in (0, 1]. Identity (and machine hash) unchanged. */
int poas_b200_refit_profile(const char* profile_text, const char* report_json, double alpha,
                            char** out_profile);
/* `iterations` rounds of an m x n x k GEMM with re-planning: plan from the
 * profile with `policy` (NULL = "reference"), execute `repeats` times
 * back to back (the mean is the observation; use the duty cycle of the real
 * workload, since power-capped clocks depend on it), re-fit, re-plan when
 * |makespan error| > replan_threshold_pct, repeat. out_json:
 * {"iterations": [{iteration, replanned, rows{id: n}, predicted_makespan,
 * measured_makespan, makespan_error_pct}], "replans", "profile" (final,
 * poas-profile v1 text), "best_iteration", "last_schedule" (the last
 * re-plan, possibly never executed), "schedule" (the plan to run next: the
 * fastest MEASURED one -- or the last plan when it splits the rows the same
 * way, for its fresher prediction)}. */
int poas_b200_run_dynamic(poas_executor_t ex, const char* profile_text, int64_t m, int64_t n,
                          int64_t k, const char* policy, const poas_gemm_io* io, int iterations,
                          int repeats, double alpha, double replan_threshold_pct,
                          char** out_json);

/* ------------------------------------------------------------------------
 * Multi-GPU: the GEMM row-sharded over the GPUs of one box,
 * one process per GPU, B broadcast from rank 0 once per GEMM. No reference
 * counterpart beyond the private-link timeline and LP rows the level-1 plan
 * uses (proj/src/timeline.cpp:24-35, proj/src/optimizer.cpp:108-115).
 * --------------------------------------------------------------------- */

/* Join the job's ranks: `name` is a token identical on every rank and
 * unique per job (e.g. derived from the launcher's rendezvous); `device` is
 * this rank's CUDA ordinal, or -1 for a host-only comm (barrier and
 * all-gather only). Collective. */
int poas_b200_comm_create(const char* name, int rank, int world, int device, poas_comm_t* out);
void poas_b200_comm_destroy(poas_comm_t comm);
int poas_b200_comm_barrier(poas_comm_t comm);
/* Every rank's `text` (<= 64 KiB) as a JSON array of strings in rank
 * order. Collective. */
int poas_b200_comm_allgather(poas_comm_t comm, const char* text, char** json_array);
/* max over ranks. Collective. */
int poas_b200_comm_max(poas_comm_t comm, double value, double* out);
/* NCCL (libnccl.so.2 loaded at run time): rank 0 makes the id, the caller
 * distributes it (e.g. poas_b200_comm_allgather of its hex), every rank
 * initialises. Needed only for b_transport = 1 and the "nccl" probe. */
int poas_b200_nccl_unique_id(unsigned char* id, size_t capacity, size_t* length);
int poas_b200_comm_init_nccl(poas_comm_t comm, const unsigned char* id, size_t length);
/* Register this rank's panel-major B ([panels][k][n/panels]; b16 in the
 * tensor units' type, b32 fp32 or NULL): rank 0's are broadcast, the other
 * ranks receive into buffers the comm owns (two, for alternate GEMMs).
 * Device memory from cudaMalloc (any offset). Collective. */
int poas_b200_comm_register_b(poas_comm_t comm, const void* b16, const float* b32, int64_t k,
                              int64_t n, int panels);
/* The level-1 link probe (DeviceBackend::time_transfer of a GPU in the
 * level-1 plan, backend.hpp:19-21): seconds to deliver `bytes` from rank 0
 * to every rank by `transport` ("ce" | "nccl"), max over ranks, mean of
 * `repetitions`. Collective. */
int poas_b200_comm_time_broadcast(poas_comm_t comm, const char* transport, uint64_t bytes,
                                  int repetitions, double* seconds);

/* Two-level plan (poas/sharded.hpp): level 1 splits m over the GPUs (each
 * GPU = its units' combined model on a private link of bandwidth
 * link_bandwidth[g], the reference pipeline), level 2 plans each GPU's rows
 * over its units with `policy`. `gpu_profiles[g]`: GPU g's poas-profile v1.
 * Out: {"level1_profile": text, "level1": schedule, "rows": [..],
 * "row0": [..], "plans": [schedule | null, ...]}. */
int poas_b200_plan_sharded(const char* const* gpu_profiles, const double* link_bandwidth, int gpus,
                           int64_t m, int64_t n, int64_t k, const char* policy, char** out_json);

/* ------------------------------------------------------------------------
 * Raw unit kernels (device pointers, caller's cudaStream_t or NULL).
 * --------------------------------------------------------------------- */
int poas_b200_tc_gemm(int dtype, int64_t m, int64_t n, int64_t k, const void* a, int64_t lda,
                      const void* b, int64_t ldb, float* c, int64_t ldc, int accumulate,
                      int num_ctas, void* stream);
/* poas_b200_tc_gemm over panel-major B (`panels` column panels, panel p a
 * row-major [k x n/panels] block with row pitch ldb at b + p*k*ldb), one
 * launch; with `flags`, tiles of panel p start once flags[p] >= epoch
 * (10 s timeout, then the launch traps). n/panels % 256 == 0. */
int poas_b200_tc_gemm_panels(int dtype, int64_t m, int64_t n, int64_t k, const void* a, int64_t lda,
                             const void* b, int64_t ldb, float* c, int64_t ldc, int accumulate,
                             int num_ctas, int panels, const int* flags, int epoch, void* stream);
/* *flag = value on `stream`, in stream order (cuStreamWriteValue32). */
int poas_b200_signal_flag(int* flag, int value, void* stream);
/* `stream` waits until *flag >= value (cuStreamWaitValue32, GEQ). */
int poas_b200_wait_flag(const int* flag, int value, void* stream);
/* Name of the kernel poas_b200_tc_gemm launches for this shape
 * ("tc_gemm_2cta_kernel" or "tc_gemm_kernel"; static string). */
const char* poas_b200_tc_kernel_name(int64_t m, int64_t n, int64_t k);
/* Its tile scheduler for this shape: "dynamic" or "wave" (static string). */
const char* poas_b200_tc_scheduler_name(int64_t m, int64_t n, int64_t k);
int poas_b200_simt_gemm(int64_t m, int64_t n, int64_t k, const float* a, int64_t lda,
                        const float* b, int64_t ldb, float* c, int64_t ldc, int accumulate,
                        int num_ctas, int exclusive_sm, void* stream);
/* Host CPU unit (AVX-512/AVX2 + threads), host pointers. */
int poas_b200_host_gemm(int64_t m, int64_t n, int64_t k, const float* a, int64_t lda,
                        const float* b, int64_t ldb, float* c, int64_t ldc, int accumulate,
                        int threads);
int poas_b200_fill_uniform(int dtype, void* dst, int64_t ld, int64_t rows, int64_t cols,
                           int64_t row0, int64_t col0, int64_t total_cols, uint64_t seed,
                           void* stream);
/* Host twin of the device generator (fp32). */
int poas_b200_fill_uniform_host(float* dst, int64_t ld, int64_t rows, int64_t cols,
                                int64_t row0, int64_t col0, int64_t total_cols, uint64_t seed);
int poas_b200_convert_f32(int dtype, const float* src, int64_t ld_src, void* dst, int64_t ld_dst,
                          int64_t rows, int64_t cols, void* stream);
int poas_b200_sm_count(void);
/* Rng::for_stream(master, name).state (proj/include/poas/rng.hpp:43-50). */
uint64_t poas_b200_stream_seed(uint64_t master_seed, const char* name);

#ifdef __cplusplus
}
#endif

#endif /* POAS_B200_H */
