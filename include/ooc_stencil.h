/* ooc_stencil.h — C ABI of the ooc-b200 runtime (libooc.so).
 *
 * The binding surface a foreign-language caller (ctypes / cgo / JNI / N-API)
 * would use in place of the reference's C++ API. Each entry point replaces one
 * reference interface:
 *
 *   ooc_rt_create / ooc_rt_destroy   ooc::Runtime(RuntimeOptions)      proj/include/ooc/runtime.hpp:33-57
 *   ooc_rt_declare                   Runtime::declare / declare_dataset proj/include/ooc/runtime.hpp:61-68,
 *                                                                       proj/src/dataset.cpp:5-38
 *   ooc_rt_enqueue_loop              Runtime::enqueue_loop(ParLoop)      proj/include/ooc/runtime.hpp:72,
 *                                    (loop bodies as prefix expressions, proj/src/expr.cpp:73-147)
 *   ooc_rt_fetch_dataset             Runtime::fetch_dataset              proj/include/ooc/runtime.hpp:76
 *   ooc_rt_fetch_reduction           Runtime::fetch_reduction            proj/include/ooc/runtime.hpp:79
 *   ooc_rt_set_cyclic                Runtime::set_cyclic_flag            proj/include/ooc/runtime.hpp:81
 *   ooc_rt_flush / ooc_rt_finish     Runtime::flush / finish             proj/include/ooc/runtime.hpp:84-85
 *   ooc_rt_run_app                   run_app                             proj/include/ooc/apps.hpp:34
 *   ooc_rt_*_json                    flush_log / audit_rows / report /   proj/include/ooc/runtime.hpp:90-104
 *                                    plan_dump_json                      proj/include/ooc/tiler.hpp:110-114
 *
 * Errors: every call returns 0 on success or a negative code naming the
 * reference exception type (proj/include/ooc/errors.hpp:9-47); the message is in
 * ooc_rt_last_error(). JSON strings returned by the *_json calls stay valid
 * until the next call on the same thread.
 */
#ifndef OOC_STENCIL_H
#define OOC_STENCIL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OOC_E_VALIDATION (-1)
#define OOC_E_STALE (-2)
#define OOC_E_INFEASIBLE (-3)
#define OOC_E_CAPACITY (-4)
#define OOC_E_DEVICE (-5)
#define OOC_E_OTHER (-9)

/* ExecutorKind (runtime.hpp): 0 reference (= resident, 1 tile), 2 tiled_explicit, 4 resident */
#define OOC_EXEC_REFERENCE 0
#define OOC_EXEC_EXPLICIT 2
#define OOC_EXEC_RESIDENT 4
/* Planning only: chains are flushed, planned and recorded but nothing executes
 * (no device needed) — used to check plans against the reference on CPU. */
#define OOC_EXEC_PLAN_ONLY 5

/* AccessMode / ReduceOp / FlushReason numbering of the reference. */
#define OOC_READ 0
#define OOC_WRITE 1
#define OOC_READ_WRITE 2
#define OOC_REDUCE_NONE 0
#define OOC_REDUCE_SUM 1
#define OOC_REDUCE_MIN 2
#define OOC_REDUCE_MAX 3

typedef struct ooc_runtime ooc_runtime;

typedef struct {
  int executor;
  int tiles;                 /* 0: choose by capacity (explicit) / 1 tile (resident) */
  int tiled_dim;
  long long capacity_bytes;  /* the artificial HBM budget of the three slots */
  long long resident_budget; /* resident: >0 skew-tiles chains to this budget (L2 tiling) */
  int prefetch;
  int record_chains;
  int gpu;
  int profile_loops;
  int arena_fill;            /* debug: 0 none, 1 zero, 2 NaN */
  int no_fuse;               /* 1: one launch per par_loop (disable loop fusion) */
  /* slab decomposition (new; the reference is single-device): this rank owns rows
   * [own_lo, own_hi) of dimension 0 and recomputes `ghost` rows each side */
  int dist_rank, dist_world;
  long long own_lo, own_hi, ghost;
  int timeline;              /* 1: record a real event timeline (CUDA events per command) */
} ooc_runtime_options;

void ooc_rt_default_options(ooc_runtime_options* o);
const char* ooc_rt_last_error(void);

int ooc_rt_create(const ooc_runtime_options* o, ooc_runtime** out);
void ooc_rt_destroy(ooc_runtime* rt);

/* fill_expr: prefix expression over coordinates i,j,k (chain-file syntax) or NULL
 * for the constant fill_value; init (optional, alloc-sized) overrides both. */
int ooc_rt_declare(ooc_runtime* rt, const char* name, int ndim, const int64_t lo[3],
                   const int64_t hi[3], const int64_t halo[3], int64_t elem_bytes,
                   const char* fill_expr, double fill_value, const double* init, int* id_out);

/* One par_loop. Per argument a: dataset[a], mode[a], noffsets[a] stencil points
 * taken consecutively (3 ints each) from `offsets`. write_exprs[w] is the prefix
 * expression stored into argument write_args[w]. */
int ooc_rt_enqueue_loop(ooc_runtime* rt, int ndim, const int64_t lo[3], const int64_t hi[3],
                        int nargs, const int* dataset, const int* mode, const int* noffsets,
                        const int64_t* offsets, int nwrites, const int* write_args,
                        const char* const* write_exprs, int reduce_op, const char* reduce_expr,
                        const char* reduce_name);

int ooc_rt_flush(ooc_runtime* rt);
int ooc_rt_finish(ooc_runtime* rt);
int ooc_rt_sync(ooc_runtime* rt);
int ooc_rt_set_cyclic(ooc_runtime* rt, int on);
int ooc_rt_fetch_dataset(ooc_runtime* rt, int dataset, double* out, int64_t n);
int ooc_rt_fetch_reduction(ooc_runtime* rt, const char* name, double* out);

int ooc_rt_num_datasets(ooc_runtime* rt);
int ooc_rt_dataset_info(ooc_runtime* rt, int dataset, int64_t* len, int* stale, int* ndim,
                        int64_t lo[3], int64_t hi[3]);
int ooc_rt_find_dataset(ooc_runtime* rt, const char* name);
/* Direct pointer to the pinned host storage (no flush, no copy-back). */
int ooc_rt_host_data(ooc_runtime* rt, int dataset, double** data, int64_t* len);

int ooc_rt_run_app(ooc_runtime* rt, const char* name, int64_t nx, int64_t ny, int64_t nz,
                   int iters, int span, int cyclic);
int ooc_rt_declare_app(ooc_runtime* rt, const char* name, int64_t nx, int64_t ny, int64_t nz,
                       int span);
/* Step-wise driving: iterations [it0, it1) of an app declared with ooc_rt_declare_app. */
int ooc_rt_app_iterations(ooc_runtime* rt, const char* name, int64_t nx, int64_t ny, int64_t nz,
                          int span, int cyclic, int it0, int it1);
int64_t ooc_app_problem_bytes(const char* name, int64_t nx, int64_t ny, int64_t nz, int span);

/* Timing marks: a CUDA event recorded on the compute queue (after everything the
 * runtime issued so far); ooc_rt_mark_elapsed syncs and returns seconds between marks. */
int ooc_rt_mark(ooc_runtime* rt);
int ooc_rt_mark_elapsed(ooc_runtime* rt, int a, int b, double* seconds);

const char* ooc_rt_flush_log_json(ooc_runtime* rt);
const char* ooc_rt_audit_json(ooc_runtime* rt);
const char* ooc_rt_report_json(ooc_runtime* rt);
const char* ooc_rt_chain_timings_json(ooc_runtime* rt);
const char* ooc_rt_loop_metrics_json(ooc_runtime* rt);
const char* ooc_rt_device_json(ooc_runtime* rt);
/* profile_loops runs: every launch since the last call as [first_loop, nloops, bytes, s]. */
const char* ooc_rt_launch_log_json(ooc_runtime* rt);
int ooc_rt_num_chains(ooc_runtime* rt);
/* CSV exports in the reference's schemas; NULL on error (see ooc_rt_last_error).
 * report: proj/src/metrics.cpp:46-60 (report_csv_header + report_csv_row)
 * loops:  proj/src/metrics.cpp:62-70 (loops_csv; with timeline=1 loop times come
 *         from the real timeline, attributed as attribute_loop_times, metrics.cpp:14-32)
 * audit:  proj/src/metrics.cpp:72-79 (audit_csv)
 * timeline: proj/src/command.cpp:160-168 (timeline_csv; rows are measured CUDA
 *         events, seconds from the first recorded command, not a simulation) */
const char* ooc_rt_report_csv(ooc_runtime* rt, const char* app, const char* size, int iters);
const char* ooc_rt_loops_csv(ooc_runtime* rt);
const char* ooc_rt_audit_csv(ooc_runtime* rt);
const char* ooc_rt_timeline_csv(ooc_runtime* rt);
/* Full plan of recorded chain `chain`: tiles>0 plans with that count, else
 * choose_tile_count(budget). `dump` = 1 returns the reference plan_dump_json
 * schema instead of the full footprint record. */
const char* ooc_rt_chain_plan_json(ooc_runtime* rt, int chain, int tiles, int64_t budget,
                                   int dump);
const char* ooc_rt_chain_plan_text(ooc_runtime* rt, int chain, int tiles);
/* Slab decomposition: join the NCCL communicator (id from ooc_comm_unique_id in
 * ooc_device.h); export a recorded chain's (window-clipped) loops; its ghost depth
 * and the ghost-band exchange it triggers. */
/* Chain-description JSON (proj/include/ooc/chain_file.hpp:22-23 load_chain_json): declares
 * the datasets and enqueues the loops; "ops" lists may interleave flush / finish / cyclic. */
int ooc_rt_load_chain_json(ooc_runtime* rt, const char* json_text, int* loops_enqueued);
int ooc_rt_comm_init(ooc_runtime* rt, const void* unique_id128);
/* Join the CUDA-IPC transport instead of NCCL: the ranks of one node rendezvous in a
 * shared-memory segment named `name` (same on every rank), ghost bands move by
 * cudaMemcpyAsync out of the neighbours' IPC-mapped outboxes (NVLink peer copies; ranks
 * may also share one GPU). */
int ooc_rt_comm_init_ipc(ooc_runtime* rt, const char* name);
const char* ooc_rt_chain_export_json(ooc_runtime* rt, int chain);
const char* ooc_rt_dist_plan_json(ooc_runtime* rt, int chain);
/* Group recorded chain `chain` as the engine would (fuse = 1: loop fusion) and
 * generate + NVRTC-compile each group's specialised sm_100a kernel (no GPU needed). */
const char* ooc_rt_chain_jit_check(ooc_runtime* rt, int chain, int fuse);
/* Row-sweep partition of a recorded chain (resident, untiled): JSON list of runs with
 * their sweep plans; compile = 1 builds each run's kernel with NVRTC (no GPU). */
const char* ooc_rt_chain_sweep_check(ooc_runtime* rt, int chain, int compile);
/* Process-wide fusion policy: 1 (default; env OOC_ROW_RECOMPUTE=0 turns it off) admits
 * row-recompute groups (neighbour reads along the row dimension of values written
 * earlier in the launch, re-evaluated in-thread). */
void ooc_rt_set_row_recompute(int on);
/* Process-wide: row-sweep kernels for resident untiled 2-D chains (default on; OOC_SWEEP=0). */
void ooc_rt_set_sweep(int on);
/* Exact reductions for the chains executed from now on (debug; default off): every
 * reduction is folded by one thread in the reference's sequential row-major order
 * (proj/src/kernel_exec.cpp:193-197), so fetch_reduction is bitwise equal to the
 * reference's instead of within 1e-12. Reducing loops launch alone, graphs are off. */
int ooc_rt_set_exact_reductions(ooc_runtime* rt, int on);
/* dependency_oracle over recorded chain `chain` planned with `tiles`. */
const char* ooc_rt_chain_oracle_json(ooc_runtime* rt, int chain, int tiles);

#ifdef __cplusplus
}
#endif

#endif /* OOC_STENCIL_H */
