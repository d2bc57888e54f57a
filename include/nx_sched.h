/* nx_sched.h — C-ABI of the B200 NexusSched hot path.
 *
 * Plain C: pointers, sizes, status codes; no torch / C++ types cross it.
 * Every entry point names the reference interface it replaces. Errors never
 * throw across the ABI; the status maps 1:1 onto the reference's exception
 * types (proj/src/*.cpp):
 *   NX_EINVAL   <- std::invalid_argument  (bad shapes / params / inputs)
 *   NX_ERUNTIME <- std::runtime_error     (config, I/O, prefill_priority cap)
 *   NX_ELOGIC   <- std::logic_error       (internal invariants)
 *   NX_ECUDA    no reference analogue: a CUDA call failed (no GPU, OOM, ...)
 * nx_last_error() returns the message of the calling thread's last failure.
 *
 * Threading: one stream per handle; handles are not shared between threads;
 * distinct handles are reentrant (proj/include/servesim/sim.h:78-100 —
 * run_simulation is reentrant).
 */
#ifndef NX_SCHED_H_
#define NX_SCHED_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { NX_OK = 0, NX_EINVAL = 1, NX_ERUNTIME = 2, NX_ELOGIC = 3, NX_ECUDA = 4 };
enum { NX_DETERMINISTIC_FP64 = 0, NX_FAST_FP32 = 1 };

const char* nx_last_error(void);
int nx_device_count(void);

/* ---- K1: batched perf-model evaluation ------------------------------------
 * Replaces servesim::throughput / predict_latency
 * (proj/include/servesim/perf_model.h:45-50, proj/src/perf_model.cpp:38-49).
 * params: n_params x 8 doubles in PerfParams order
 *         {tau0, w0, ws, tauB, tauS, p_max, kB, kS};
 * idx/b/s: n evaluation records (engine-params index, batch size, tokens).
 * out_T (and out_thr if non-NULL): n results.
 * mode NX_DETERMINISTIC_FP64: bit-identical expression order, no FMA;
 * NX_FAST_FP32: float math, <= 1e-4 relative.
 * Returns NX_EINVAL (like the reference's std::invalid_argument) if any
 * record has b < 1, s < b, idx out of range, or invalid params.
 * _dev variant: all pointers are device pointers, async on `stream`.
 * _host variant: host pointers; copies in/out are part of the call. */
int nx_perf_eval_dev(const double* params, int32_t n_params, const int32_t* idx,
                     const int32_t* b, const int32_t* s, double* out_T, double* out_thr,
                     int64_t n, int32_t mode, void* stream);
/* Stream-ordered variant: no host synchronisation; bit 0 of *dev_status (a
 * device word the caller zeroes) is set if any record or row is invalid. */
int nx_perf_eval_async(const double* params, int32_t n_params, const int32_t* idx,
                       const int32_t* b, const int32_t* s, double* out_T, double* out_thr,
                       int64_t n, int32_t mode, uint32_t* dev_status, void* stream);
int nx_perf_eval_host(const double* params, int32_t n_params, const int32_t* idx,
                      const int32_t* b, const int32_t* s, double* out_T, double* out_thr,
                      int64_t n, int32_t mode);

/* ---- K5 (+K2/K3/K4 inside): batched replica simulation --------------------
 * Replaces servesim::run_simulation / sweep (proj/include/servesim/sim.h:
 * 78-100, proj/src/sim.cpp:245-347, 596-642): each config is a RunConfig JSON
 * document (RunConfig::from_json_text schema, proj/src/sim.cpp:454-582); one
 * replica per document. Workloads are synthesised on the host exactly like
 * the reference (arrival doubles come from host libm). */
typedef struct nx_sim* nx_sim_t;

typedef struct nx_replica_summary {
  int64_t arrived, completed, rejected, unfinished;
  int64_t events;        /* processed events (hashed) */
  int64_t decisions;     /* routes + executed batches = arrived + sum(samples) */
  uint64_t arrival_hash, event_hash;
  int32_t status;        /* NX_OK or the reference exception class */
  int32_t err_site;
} nx_replica_summary;

typedef struct nx_request_record { /* servesim::RequestRecord, metrics.h:12-20 */
  int64_t request_id;
  double arrival_ms, first_token_ms, completed_ms;
  int64_t prompt_tokens, output_tokens;
  int32_t engine_id, pad_;
} nx_request_record;

/* Parse + validate configs, synthesise workloads (host threads), pack the
 * SoA image into pinned host memory. No device work. */
int nx_sim_create_json(const char* const* configs, int32_t n_replicas, int32_t device,
                       int32_t host_threads, nx_sim_t* out);
/* Upload (H2D), launch, download (D2H) on the handle's stream; each is async. */
int nx_sim_upload(nx_sim_t h);
int nx_sim_launch(nx_sim_t h);
int nx_sim_download(nx_sim_t h);
int nx_sim_synchronize(nx_sim_t h);
/* upload + launch + download + synchronize */
int nx_sim_run(nx_sim_t h);
/* Device time of the last launch (CUDA events on the handle's stream). */
int nx_sim_last_kernel_ms(nx_sim_t h, float* ms);
/* Bytes moved per upload / download (e2e accounting). */
int nx_sim_io_bytes(nx_sim_t h, int64_t* h2d, int64_t* d2h);
int nx_sim_replica_count(nx_sim_t h);
int nx_sim_summaries(nx_sim_t h, nx_replica_summary* out);
/* Byte-identical to RunResult::summary_json (proj/src/sim.cpp:349-392). */
int nx_sim_summary_json(nx_sim_t h, int32_t replica, char* buf, int64_t cap, int64_t* len);
int nx_sim_records(nx_sim_t h, int32_t replica, nx_request_record* out, int64_t cap,
                   int64_t* n);
/* Work counters of a replica (roofline accounting): [0] executed steps,
 * [1] sum of batch sizes, [2] LENS candidate-window waiters scanned,
 * [3] linear-refit window samples, [4] structural-refit window samples,
 * [5] gauged (profiled) fits. */
int nx_sim_work(nx_sim_t h, int32_t replica, int64_t* out6);
/* SM cycles per phase of a replica (lane-0 clock64): [0] event selection +
 * hash, [1] routing + admission, [2] step planning, [3] step completion,
 * [4] state reports, [5] linear refits, [6] structural refits (on the refit
 * warp, overlapped with the event loop), [7] deliveries, [8] event loop
 * blocked on a pending refit, [9]-[15] refit internals (diagnostic) */
int nx_sim_phase_cycles(nx_sim_t h, int32_t replica, int64_t* out10);
/* Learner state per engine: params[8] + samples + counters[7]. */
int nx_sim_learner(nx_sim_t h, int32_t replica, int32_t engine, double* params8,
                   int64_t* samples, int64_t* counters7);
void nx_sim_destroy(nx_sim_t h);

/* ---- K6: multi-GPU result gather ------------------------------------------
 * The per-replica nx_replica_summary array is the only data that crosses
 * GPUs (one collective per run; no per-step exchange). Device pointer to the
 * handle's summaries, filled by nx_sim_launch, for an NCCL all-gather. */
int nx_sim_summaries_dev(nx_sim_t h, void** dev_ptr, int64_t* bytes);
/* Device-to-device copy of those summaries into a caller buffer (e.g. the
 * send buffer of an ncclAllGather); ordered on the handle's stream. */
int nx_sim_copy_summaries(nx_sim_t h, void* dst_dev);

/* ---- host utilities (reference workload generator semantics) -------------
 * synth_generate (proj/src/workload.cpp:137-166): prompts/outputs/session
 * ids for n requests. session_ids: n * 16-byte NUL-terminated strings. */
/* Parse a RunConfig JSON and synthesise its workload on the host only:
 * arrival fingerprint (sim.cpp:132-139), request and session counts. Raises
 * the reference's config errors (RunConfig::validate, sim.cpp:418-452). */
int nx_workload_info(const char* config_json, uint64_t* arrival_hash, int64_t* n_requests,
                     int64_t* n_sessions);
int nx_synth_generate(const char* scenario, int64_t n, uint64_t seed, int64_t* prompts,
                      int64_t* outputs, char* session_ids16);

#ifdef __cplusplus
}
#endif
#endif /* NX_SCHED_H_ */
