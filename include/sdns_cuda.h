/*
 * sdns_cuda.h — C ABI of the B200-native spectral-DNS hot path.
 *
 * Drop-in boundary for the reference solver's hot path (arXiv 1607.00850,
 * C++ library `sdns`, /root/reference/proj). Every entry point replaces one
 * reference interface; the citation after each declaration is the reference
 * file:line it stands in for. Plain pointers and sizes only — no C++ or torch
 * types cross this boundary. INTEGRATION.md shows the reference-side binding.
 *
 * Conventions
 *  - Status codes map 1:1 onto the reference's exception types
 *    (proj/core/include/sdns/types.hpp:28-62); the message of the last
 *    failure on the calling thread is returned by sdns_last_error().
 *  - Host arrays use the reference's rank-local block layout
 *    (RankLayout, proj/core/include/sdns/layout.hpp:24-41): row-major,
 *    z fastest; spectral values are interleaved (re, im) doubles; vector
 *    fields are `ncomp` component blocks back to back (SoA, like
 *    VectorField3, proj/core/include/sdns/fields.hpp:33-46).
 *  - All allocation happens in the *_create / *_alloc calls; transforms and
 *    steps never allocate (proj/core/include/sdns/fft.hpp:22-25).
 *  - Every transform / RHS / step call is collective over the context's
 *    communicator, in identical order on all ranks (fft.hpp:22-24).
 *  - Work is enqueued on the context's CUDA stream; calls that return host
 *    values (stats, finite flags, downloads) synchronise that stream.
 */
#ifndef SDNS_CUDA_H
#define SDNS_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (types.hpp:28-62) ------------------------------------ */
enum {
  SDNS_OK = 0,
  SDNS_CONFIG_ERROR = 1,     /* ConfigError      types.hpp:29-32 */
  SDNS_PROTOCOL_ERROR = 2,   /* ProtocolError    types.hpp:36-39 */
  SDNS_TIMEOUT_ERROR = 3,    /* TimeoutError     types.hpp:42-45 */
  SDNS_DIVERGENCE_ERROR = 4, /* DivergenceError  types.hpp:48-56 */
  SDNS_IO_ERROR = 5,         /* IoError          types.hpp:59-62 */
  SDNS_CUDA_ERROR = 6,       /* device / driver failure (no reference analogue) */
  SDNS_INTERNAL_ERROR = 9
};

enum { SDNS_SLAB = 0, SDNS_PENCIL = 1 };
enum { SDNS_REAL = 0, SDNS_SPECTRAL = 1 };

/* SolverConfig, proj/core/include/sdns/config.hpp:14-30 */
typedef struct sdns_config {
  int n;          /* grid points per axis */
  int decomp;     /* SDNS_SLAB | SDNS_PENCIL */
  int p, p1, p2;  /* ranks; pencil grid p = p1*p2 */
  double nu;
  double dt;
  double t_end;
  int dealias;    /* strict 2/3 rule */
  int out_every;
} sdns_config;

/* RankLayout, proj/core/include/sdns/layout.hpp:24-41 (one transpose stage
 * for slab, two for pencil; counts in complex elements, per group peer). */
#define SDNS_MAX_PEERS 64
typedef struct sdns_layout {
  int rank, p, p1, p2, coord1, coord2;
  int64_t n, nf;
  int64_t real_shape[3], real_offset[3];
  int64_t spec_shape[3], spec_offset[3];
  int nstages;
  int stage_peers[2];
  int64_t send_counts[2][SDNS_MAX_PEERS];
  int64_t recv_counts[2][SDNS_MAX_PEERS];
} sdns_layout;

typedef struct sdns_comm sdns_comm;
typedef struct sdns_ctx sdns_ctx;
typedef struct sdns_field sdns_field;
typedef struct sdns_state sdns_state;

/* ---- errors ------------------------------------------------------------- */
const char* sdns_last_error(void);

/* ---- host-only setup (no device needed) --------------------------------- */
int sdns_config_validate(const sdns_config* cfg);                  /* config.cpp:17-50 */
int sdns_build_layout(const sdns_config* cfg, int rank,
                      sdns_layout* out);                            /* layout.hpp:48 */
int64_t sdns_block_size(int64_t total, int parts, int index);       /* layout.hpp:44 */
int64_t sdns_block_start(int64_t total, int parts, int index);      /* layout.hpp:45 */
int64_t sdns_step_count(double t_end, double dt);                   /* rk4.hpp:43 */
int sdns_spectrum_shells(int64_t n);                                /* diagnostics.hpp:22 */
/* Seeded isotropic initial field (BASELINE configs 2-4):
 * writes the rank's spectral block (3 comps) into `out`. Identical for every
 * decomposition. The reference has no such case (navier_stokes.cpp:27-32). */
int sdns_iso_init_host(int64_t n, uint64_t seed, double k0, double energy,
                       const sdns_layout* lo, double* out);
/* Library build string. */
const char* sdns_version(void);

/* Device layout of a rank's fields: spectral components are
 * s0 x planes of `prow` = s1 + 1 rows (one pad row) of `pitch` =
 * round_up(s2, 8) complex; `np` = n / p; element counts per component. */
typedef struct sdns_dev_layout {
  int pitch, prow, np;
  int64_t spec_cs, real_cs;
} sdns_dev_layout;
int sdns_device_layout(const sdns_config* cfg, int rank, sdns_dev_layout* out);
/* The transpose plan the context executes for `nfields` fields: *count
 * entries of (peer, source offset, destination offset, complex count),
 * offsets relative to the x-layout / receive-layout work buffers. Replaces
 * the pack -> all_to_all -> unpack of fft.cpp:89-122 (slab). out may be NULL
 * to query the count. */
int sdns_exchange_plan(const sdns_config* cfg, int rank, int inverse, int nfields,
                       int64_t* out, int* count);

/* ---- communicators (Communicator, transport.hpp:46-94) ------------------ */
int sdns_comm_loopback(sdns_comm** out);                            /* transport.hpp:96-98 */
/* Threads-as-ranks on ONE device (InProcessBackend, transport.hpp:109-131):
 * out[r] is handed to the host thread driving rank r. Exchanges are
 * stream-ordered device copies; no kernel waits on another. */
int sdns_comm_inprocess_group(int size, int device, double timeout_s, sdns_comm** out);
/* One process per GPU over NCCL (NVLink / NVSwitch). The 128-byte unique id
 * is created on rank 0 and distributed by the caller. */
int sdns_comm_nccl_unique_id(unsigned char id[128]);
int sdns_comm_nccl_init(const unsigned char id[128], int size, int rank, int device,
                        sdns_comm** out);
/* One process per rank over the caller's host all-gather (e.g.
 * torch.distributed on gloo): `allgather(send, bytes, recv, user)` must put
 * every rank's `bytes` of the group `user` into recv in rank order and
 * return 0. split() calls `group(ranks, n, user, &child_user)` once per new
 * group, in the same order and with the same member list (indices in the
 * group `user`) on every rank, and the child uses child_user (NULL group
 * callback: no split). Buffers and stream barriers go through CUDA IPC
 * (memory and events), so several ranks may share one GPU and no kernel
 * waits on another. The RHS transposes run peer-direct; all_to_all (the
 * checkpoint gathers/scatters, sdns_comm_all_to_all_bytes) goes through the
 * all-gather (every rank receives every packed buffer). The callback
 * returns 2 when the caller's transport timed out (SDNS_TIMEOUT_ERROR),
 * any other nonzero value for other failures (SDNS_PROTOCOL_ERROR).
 * Collective. */
typedef int (*sdns_allgather_fn)(const void* send, size_t bytes, void* recv, void* user);
typedef int (*sdns_group_fn)(const int* ranks, int n, void* user, void** child_user);
int sdns_comm_host_init(int size, int rank, int device, sdns_allgather_fn allgather,
                        sdns_group_fn group, void* user, sdns_comm** out);
int sdns_comm_rank(const sdns_comm* c);
int sdns_comm_size(const sdns_comm* c);
int sdns_comm_barrier(sdns_comm* c);                                 /* transport.hpp:64 */
/* In-place reduction in ascending rank order (op 0 sum, 1 max, 2 min). */
int sdns_comm_allreduce(sdns_comm* c, double* values, int count, int op); /* :61 */
/* broadcast_bytes (transport.hpp:62): the root's `nbytes` HOST bytes into
 * every rank's `data`. root and nbytes must agree on every rank, else every
 * rank fails with SDNS_PROTOCOL_ERROR (validate_broadcast,
 * transport.cpp:332-349); the loopback accepts only root 0. Collective. */
int sdns_comm_broadcast_bytes(sdns_comm* c, void* data, int64_t nbytes, int root);
int sdns_comm_destroy(sdns_comm* c);
/* InProcessBackend::poison (transport.hpp:125-128): every pending and later
 * collective of the group fails with SDNS_PROTOCOL_ERROR naming `reason`; a
 * no-op on transports without shared state (loopback, NCCL, host). */
int sdns_comm_poison(sdns_comm* c, const char* reason);
/* Collective deadline in seconds (the reference's collective_timeout,
 * runner.hpp:15, default 30 s; <= 0: none). On the NCCL and host-callback
 * transports every host wait on a stream holding the group's collectives
 * polls the stream and the transport (ncclCommGetAsyncError): a peer that
 * stalls past the deadline raises SDNS_TIMEOUT_ERROR, an asynchronous
 * transport error SDNS_PROTOCOL_ERROR (transport.cpp:105-140), the
 * communicator is aborted (ncclCommAbort) and every later collective on it
 * fails with the same status. Children made by split inherit the deadline. */
int sdns_comm_set_timeout(sdns_comm* c, double seconds);
/* split(color, key): members ordered by (key, rank) (transport.hpp:66-67). */
int sdns_comm_split(sdns_comm* c, int color, int key, sdns_comm** out);
/* all_to_all_bytes (transport.hpp:55-58, BlockTable :18-35) on DEVICE
 * buffers: block q of `send` (send_bytes[q], displacements the prefix sums)
 * goes to peer q, which receives it as its block for this rank. Enqueued on
 * `stream` (a cudaStream_t; NULL = legacy stream, and the call returns after
 * the exchange completed). Collective. */
int sdns_comm_all_to_all_bytes(sdns_comm* c, const void* send, const int64_t* send_bytes,
                               void* recv, const int64_t* recv_bytes, void* stream);

/* ---- context (DistributedFFT ctor + wavenumbers + workspaces) ----------- */
/* fft.cpp:15-57, mesh.cpp:23-72, navier_stokes.hpp:32-41. `stream` is a
 * cudaStream_t or NULL (the context then owns a stream). */
int sdns_ctx_create(const sdns_config* cfg, int rank, int device, sdns_comm* comm,
                    void* stream, sdns_ctx** out);
/* Execution choices of a context; none changes a result bit (every
 * combination runs the same transforms and arithmetic). Zero-initialised
 * options are the defaults sdns_ctx_create uses. Nothing is read from the
 * environment. */
typedef struct sdns_ctx_options {
  int all_to_all;   /* 1: transposes as all-to-alls (NCCL send/recv, copies)
                       instead of peer-direct stores fused into the passes */
  int serial;       /* 1: slab all-to-alls not overlapped with the passes */
  int ldgsts_tiles; /* 1: column-pass tiles by LDGSTS instead of TMA boxes */
  int plain_layout; /* 1: p = 1 keeps the natural work layouts (no chunk-major
                       P1 output / chunked P2..P5a layout) */
  int no_graph;     /* 1: p = 1 steps launch eagerly, not as a captured graph */
  int p1_single;    /* x inverse pass (P1) as five single-transform items on one
                       128 B-row tile buffer instead of three items with two
                       transforms and a scratch tile. 0: by size (on at
                       n >= 1024, where two 128 B-row tiles do not fit), 1: on
                       (tuned n >= 128), -1: off */
} sdns_ctx_options;
int sdns_ctx_create_ex(const sdns_config* cfg, int rank, int device, sdns_comm* comm,
                       void* stream, const sdns_ctx_options* opts, sdns_ctx** out);
int sdns_ctx_destroy(sdns_ctx* ctx);
int sdns_ctx_layout(const sdns_ctx* ctx, sdns_layout* out);
void* sdns_ctx_stream(const sdns_ctx* ctx);
int sdns_ctx_sync(sdns_ctx* ctx);
/* Which transposes of the RHS pipeline run peer-direct: bit 0
 * the slab / pencil-column ones, bit 1 the pencil-row ones; 0 = all-to-all. */
int sdns_ctx_transposes(const sdns_ctx* ctx);
/* Device bytes held by the context (workspaces) and per field. */
int64_t sdns_ctx_device_bytes(const sdns_ctx* ctx);

/* ---- device fields (Field3d / VectorField3, fields.hpp:10-49) ----------- */
int sdns_field_alloc(sdns_ctx* ctx, int kind, int ncomp, sdns_field** out);
int sdns_field_free(sdns_field* f);
int sdns_field_upload(sdns_ctx* ctx, sdns_field* f, const double* host);
int sdns_field_download(sdns_ctx* ctx, const sdns_field* f, double* host);
int sdns_field_copy(sdns_ctx* ctx, const sdns_field* src, sdns_field* dst);

/* ---- DistributedFFT::forward / inverse (fft.hpp:34-38, fft.cpp:59-227) -- */
/* Forward is unnormalised; inverse applies 1/n^3 once. All components. */
int sdns_fft_forward(sdns_ctx* ctx, const sdns_field* real, sdns_field* spec);
int sdns_fft_inverse(sdns_ctx* ctx, const sdns_field* spec, sdns_field* real);

/* ---- pointwise operators (navier_stokes.hpp:17-29) ---------------------- */
int sdns_curl_hat(sdns_ctx* ctx, const sdns_field* u_hat, sdns_field* omega_hat);
int sdns_cross(sdns_ctx* ctx, const sdns_field* a, const sdns_field* b, sdns_field* out);
int sdns_project(sdns_ctx* ctx, sdns_field* u_hat);
int sdns_pressure_hat(sdns_ctx* ctx, const sdns_field* nl_hat, sdns_field* p_hat);

/* ---- compute_rhs (navier_stokes.hpp:47-49, navier_stokes.cpp:104-139) --- */
int sdns_compute_rhs(sdns_ctx* ctx, const sdns_field* u_hat, double nu, sdns_field* du_hat);

/* ---- RK4 (Rk4State / rk4_step / advance, rk4.hpp:18-62) ----------------- */
int sdns_state_create(sdns_ctx* ctx, sdns_state** out);
int sdns_state_destroy(sdns_state* st);
int sdns_state_set(sdns_ctx* ctx, sdns_state* st, const sdns_field* u_hat, double t,
                   int64_t step);           /* carry reset to 0 */
int sdns_state_get(sdns_ctx* ctx, const sdns_state* st, sdns_field* u_hat);
/* The state's u_hat as a field view (owned by the state; do not free). */
sdns_field* sdns_state_u_hat(sdns_state* st);
int sdns_state_time(const sdns_state* st, double* t, int64_t* step);
/* One classical RK4 step with the fused pipeline (rk4.cpp:27-71); if
 * post_project, the solenoidal cleanup of runner.cpp:107 is fused into the
 * last stage. *finite (if not NULL) receives the collective finite flag
 * (rk4.cpp:97) and forces a stream synchronisation. */
int sdns_rk4_step(sdns_ctx* ctx, sdns_state* st, double dt, int post_project, int* finite);
/* advance(): rk4.cpp:86-107, including the shortened final step, t = k*dt,
 * the collective divergence check (SDNS_DIVERGENCE_ERROR, *fail_step set)
 * and the sample hook cadence (step 0, every out_every, final step). */
typedef void (*sdns_sample_fn)(int64_t step, double t, void* user);
int sdns_advance(sdns_ctx* ctx, sdns_state* st, sdns_sample_fn sample, void* user,
                 int64_t* fail_step);
/* Host-buffer tier (reference-facing, e2e): uploads u_hat, runs `steps`
 * fused steps with post-step projection, downloads u_hat. */
int sdns_rk4_step_host(sdns_ctx* ctx, sdns_state* st, double* host_u_hat, double dt,
                       int steps);

/* ---- diagnostics (diagnostics.hpp:22-44) -------------------------------- */
/* row = [t, E, Z, eps, div_max, spectrum[shells]] identical on every rank. */
int sdns_collect_stats(sdns_ctx* ctx, const sdns_field* u_hat, double nu, double t,
                       double* row);
int sdns_l2_diff(sdns_ctx* ctx, const sdns_field* a, const sdns_field* b, double* out);

/* ---- checkpoints (checkpoint.hpp:11-33, checkpoint.cpp:64-187) ---------- */
/* Collective. u_real: this rank's block of the real velocity (3 comps). The
 * file is the reference's format: 32-byte header (magic "SDNS", u32 version
 * 1, u32 n, u32 components 3, f64 t, u64 step) + three n^3 little-endian f64
 * payloads in global x-major order, so any decomposition reads any other's
 * file bit-exactly (and the reference reads ours). Rank 0 gathers and
 * writes; SDNS_IO_ERROR on every rank when the path cannot be written. */
int sdns_checkpoint_write(sdns_ctx* ctx, const sdns_field* u_real, const char* path, double t,
                          int64_t step);
/* Collective inverse: rank 0 reads and validates (magic, version, n,
 * components, size -> SDNS_IO_ERROR on every rank), scatters the blocks;
 * every rank receives t and step. */
int sdns_checkpoint_read(sdns_ctx* ctx, const char* path, sdns_field* u_real, double* t,
                         int64_t* step);

/* ---- advance with the full hook set (AdvanceHooks, rk4.hpp:45-55) ------- */
/* timing(step, seconds): wall time of one step, from before the update to
 * after its collective finite flag (rk4.cpp:93-105); the step synchronises
 * its stream to read that flag, so the interval covers the device work. */
typedef void (*sdns_timing_fn)(int64_t step, double seconds, void* user);
typedef struct sdns_advance_hooks {
  sdns_sample_fn sample; /* AdvanceHooks::sample, or NULL */
  sdns_timing_fn timing; /* AdvanceHooks::timing, or NULL */
  void* user;
} sdns_advance_hooks;
int sdns_advance_hooks_run(sdns_ctx* ctx, sdns_state* st, const sdns_advance_hooks* hooks,
                           int64_t* fail_step);

/* ---- runner, bench harness, config files (runner.hpp, config_file.hpp) -- */
/* SolverConfig defaults (config.hpp:14-30): n 32, slab, p = p1 = p2 = 1,
 * nu 1/1600, dt 1e-3, t_end 0.1, dealias on, out_every 10. */
void sdns_config_defaults(sdns_config* cfg);
/* parse_config_text / parse_config_file (config_file.hpp:24-29,
 * config_file.cpp:57-147): `key = value` lines, '#' comments; keys n,
 * decomp, p, p1, p2, nu, re, dt, t_end, dealias, case, out_every; then the
 * ordered overrides (keys[i] = values[i]); then validate. initial_case
 * receives `case`; notices receives the '\n'-terminated notices. */
typedef struct sdns_parsed_config {
  sdns_config cfg;
  char initial_case[64];
  char notices[512];
} sdns_parsed_config;
int sdns_parse_config_text(const char* text, const char* const* keys, const char* const* values,
                           int n_overrides, sdns_parsed_config* out);
int sdns_parse_config_file(const char* path, const char* const* keys, const char* const* values,
                           int n_overrides, sdns_parsed_config* out);
/* default_pencil_grid (config_file.cpp:43-55). */
int sdns_default_pencil_grid(int n, int p, int* p1, int* p2);

/* RunOptions (runner.hpp:11-15) plus the device and the isotropic seed. */
typedef struct sdns_run_options {
  const char* out_dir;          /* default "out" */
  const char* backend;          /* "auto" | "loopback" | "inprocess" */
  double collective_timeout_s;  /* default 30 */
  int device;                   /* CUDA device of every rank of sdns_run */
  uint64_t seed;                /* case "isotropic" only */
  sdns_ctx_options ctx;         /* execution options of every rank's context */
} sdns_run_options;
/* RunResult (runner.hpp:28-36). samples: optional caller buffers of
 * sample_cap rows (step, and 5 + shells doubles: t, E, Z, eps, div_max,
 * spectrum), filled on rank 0; n_samples is the count produced. */
typedef struct sdns_run_result {
  char backend[16];
  char status[256];
  int64_t steps;
  double step_min_s, step_mean_s, step_max_s;
  int64_t timed_steps;
  int shells;
  int64_t n_samples, sample_cap;
  int64_t* sample_steps;
  double* sample_rows;
  char csv_path[512], checkpoint_path[512], manifest_path[512];
} sdns_run_result;
/* run() (runner.hpp:44, runner.cpp:197-213): one host thread per rank on
 * `device` (threads-as-ranks for p > 1), initial condition (`taylor_green`
 * = the reference's cos x sin y sin z case, navier_stokes.cpp:7-32;
 * `taylor_green_baseline` = BASELINE configs[0]'s sin x cos y cos z;
 * `isotropic` = BASELINE configs[1-3]'s seeded field set in spectral space)
 * -> forward + project -> advance with sampling, per-step timing and the
 * post-step projection -> final (or last-good) checkpoint ->
 * diagnostics.csv and manifest.txt in out_dir (rank 0). On divergence the
 * last sampled state is checkpointed, the manifest records the failure and
 * SDNS_DIVERGENCE_ERROR is returned (the result is still filled). */
int sdns_run(const sdns_config* cfg, const char* initial_case, const sdns_run_options* opts,
             sdns_run_result* out);
/* run_worker (runner.cpp:67-146) for one rank of a caller-made communicator
 * (e.g. one process per GPU over NCCL); collective over `comm`. */
int sdns_run_rank(const sdns_config* cfg, const char* initial_case, const sdns_run_options* opts,
                  int rank, sdns_comm* comm, sdns_run_result* out);

/* BenchEntry / BenchRow (runner.hpp:40-58). */
typedef struct sdns_bench_entry {
  int n, decomp, p, p1, p2; /* p1 = p2 = 0: near-square pencil grid */
} sdns_bench_entry;
typedef struct sdns_bench_row {
  sdns_bench_entry entry;
  int64_t nodes_per_rank;
  double sec_per_step;
  char status[256]; /* "ok" or the failure message */
} sdns_bench_row;
/* parse_bench_matrix_text/file (runner.cpp:249-297): `n, decomp, p[, p1,
 * p2]` lines, '#' comments, commas or blanks. *count = entries (at most cap
 * written; out may be NULL to count). */
int sdns_parse_bench_matrix_text(const char* text, sdns_bench_entry* out, int cap, int* count);
int sdns_parse_bench_matrix_file(const char* path, sdns_bench_entry* out, int cap, int* count);
/* bench() (runner.cpp:375-397): per entry, the reference's Taylor-Green case
 * (nu 1/1600, dt 1e-3, dealias), 5 warm-up steps, then `steps` timed fused
 * RK4 steps with the post-step projection between barriers; rank 0's mean
 * wall seconds per step. Per-entry failures go to status. */
int sdns_bench(const sdns_bench_entry* entries, int count, int steps,
               const sdns_run_options* opts, sdns_bench_row* rows);
/* write_bench_csv / write_diagnostics_csv / write_manifest
 * (runner.cpp:215-247, :399-414): byte-identical formats ("%.17g"). */
int sdns_write_bench_csv(const char* path, const sdns_bench_row* rows, int count);
int sdns_write_diagnostics_csv(const char* path, const int64_t* steps, const double* rows,
                               int64_t nrows, int shells);
int sdns_write_manifest(const char* path, const sdns_config* cfg, const char* initial_case,
                        const sdns_run_result* result);

/* run_acceptance_suite (verification.hpp:17-24, verification.cpp:548-614):
 * the reference's nine acceptance criteria, evaluated on the device
 * pipeline (FFT vs the serial transform for every decomposition, Parseval,
 * divergence-free evolution, energy identities, RK4 order, parallel
 * invariance, checkpoint portability, transport conformance, bench
 * harness). Ranks are threads on `device`. If `print`, one
 * "[PASS]/[FAIL] <index> <name> (<detail>, <s> s)" line per criterion goes
 * to stdout. results (may be NULL) receives 9 entries. */
typedef struct sdns_criterion_result {
  int index;
  char name[64];
  int passed;
  char detail[512];
  double seconds;
} sdns_criterion_result;
int sdns_acceptance_suite(int device, int print, sdns_criterion_result* results,
                          int* all_passed);

/* ---- per-pass timing (CUDA events on the context stream) --------------- */
/* Pass tags of one RHS evaluation. */
enum {
  SDNS_PASS_X_INV_CURL = 0, /* P1 */
  SDNS_PASS_Y_INV = 1,      /* P2 */
  SDNS_PASS_Z_FUSED = 2,    /* P3 */
  SDNS_PASS_Y_FWD = 3,      /* P4 */
  SDNS_PASS_X_FWD_TAIL = 4, /* P5b, compute_rhs tail */
  SDNS_PASS_X_FWD_RK0 = 5,  /* P5b, RK4 stage 0 */
  SDNS_PASS_X_FWD_RK12 = 6, /* P5b, RK4 stages 1-2 */
  SDNS_PASS_X_FWD_RK3 = 7,  /* P5b, RK4 stage 3 + projection */
  SDNS_PASS_A2A_INV = 8,
  SDNS_PASS_A2A_FWD = 9,
  SDNS_PASS_X_FWD_FFT = 10, /* P5a, x-axis forward FFT of the nonlinear term */
  SDNS_NPASS = 11
};
/* Enables (and resets) event timing of every pipeline launch. */
int sdns_ctx_timing(sdns_ctx* ctx, int enable);
/* Synchronises, then returns per-tag total milliseconds and launch counts
 * accumulated since the last enable/read (arrays of SDNS_NPASS). */
int sdns_ctx_timing_read(sdns_ctx* ctx, double* ms, int64_t* launches);

/* ---- host memory helpers (pinned buffers for the e2e tier) ------------- */
void* sdns_host_alloc(size_t bytes);
void sdns_host_free(void* p);

#ifdef __cplusplus
}
#endif

#endif /* SDNS_CUDA_H */
