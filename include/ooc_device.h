/* ooc_device.h — C ABI of the B200 device layer (liboocdev.so, built by nvcc for sm_100a).
 *
 * This is the seam between the host C++ engine (planner, lazy runtime, streaming
 * executor) and CUDA. It replaces the parts of the reference that pretend to be a
 * device — all host-only in /root/reference/proj:
 *
 *   ooc_host_alloc / ooc_host_free    Dataset::host pageable std::vector
 *                                     (proj/include/ooc/dataset.hpp:28) -> pinned memory
 *   ooc_mem_*                         explicit-mode arenas std::vector<double>
 *                                     (proj/src/explicit_exec.cpp:32-35, 73-84) -> HBM pool
 *   ooc_event_* / ooc_queue_*         simulated CommandQueueProgram / push_wait / simulate_timeline
 *                                     (proj/include/ooc/command.hpp:32-128,
 *                                      proj/src/command.cpp:35-126) -> CUDA streams + events
 *   ooc_copy_box                      copy_box row memcpy (proj/src/explicit_exec.cpp:13-30)
 *                                     -> cudaMemcpy2D/3DAsync on the H2D / D2H / compute queues
 *   ooc_launch_loop                   apply_loop (proj/include/ooc/kernel_exec.hpp:29-30,
 *                                     proj/src/kernel_exec.cpp:133-198) -> sm_100a kernels
 *   ooc_reduce_*                      per-chain reduction accumulators
 *                                     (proj/src/explicit_exec.cpp:159-162, 275-276)
 *
 * Conventions: every call returns int (0 = OK, negative = error, message in
 * ooc_dev_last_error()). No call takes ownership of host memory. One context per
 * GPU; a context is driven by one host thread. Plain C types only.
 */
#ifndef OOC_DEVICE_H
#define OOC_DEVICE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OOC_OK 0
#define OOC_ERR_CUDA (-10)
#define OOC_ERR_ARG (-11)
#define OOC_ERR_NODEV (-12)
#define OOC_ERR_CAPACITY (-13)
#define OOC_ERR_UNSUPPORTED (-14)

#define OOC_MAX_ARGS 16   /* kernel_exec.cpp:163-164 */
#define OOC_MAX_WRITES 8  /* kernel_exec.cpp:171-172 */
#define OOC_MAX_STACK 32  /* kernel_exec.cpp:23 */
#define OOC_MAX_TAPE 512  /* total instructions of one loop (all tapes) */
#define OOC_REDUCE_SLOTS 1024

const char* ooc_dev_last_error(void);
int ooc_dev_count(int* n);
/* Library build id (sm arch, git-less version string). */
const char* ooc_dev_build_info(void);

/* ------------------------------------------------------------ host memory */
int ooc_host_alloc(size_t bytes, void** out); /* page-locked, portable */
int ooc_host_free(void* p);
/* Preferred GPU for the page-locked allocations of the calling thread (-1: none): the
 * pages are placed on the CPUs local to that GPU (its NUMA node). */
int ooc_host_numa_device(int device);

/* ------------------------------------------------------------ context */
typedef struct ooc_ctx ooc_ctx;
typedef struct {
  int device;
  int sm_count;
  int cc_major, cc_minor;
  long long l2_bytes;
  long long hbm_bytes;
  long long free_bytes;
  char name[128];
} ooc_dev_props;

int ooc_ctx_create(int device, ooc_ctx** out);
int ooc_ctx_destroy(ooc_ctx* ctx);
int ooc_ctx_props(ooc_ctx* ctx, ooc_dev_props* out);
int ooc_ctx_sync(ooc_ctx* ctx);

/* ------------------------------------------------------------ device memory manager */
int ooc_mem_alloc(ooc_ctx* ctx, size_t bytes, void** out); /* 256-B aligned, tracked */
int ooc_mem_free(ooc_ctx* ctx, void* p);
int ooc_mem_usage(ooc_ctx* ctx, long long* in_use, long long* peak);

/* ------------------------------------------------------------ queues and events */
enum { OOC_Q_COMPUTE = 0, OOC_Q_H2D = 1, OOC_Q_D2H = 2, OOC_NUM_QUEUES = 3 };
typedef struct ooc_event ooc_event;
int ooc_event_create(ooc_ctx* ctx, int timing, ooc_event** out);
int ooc_event_destroy(ooc_ctx* ctx, ooc_event* ev);
int ooc_event_record(ooc_ctx* ctx, ooc_event* ev, int queue);
int ooc_queue_wait(ooc_ctx* ctx, int queue, ooc_event* ev); /* queue waits for ev */
int ooc_event_sync(ooc_ctx* ctx, ooc_event* ev);
int ooc_event_query(ooc_ctx* ctx, ooc_event* ev, int* done);
int ooc_event_elapsed_ms(ooc_event* start, ooc_event* end, float* ms);
int ooc_queue_sync(ooc_ctx* ctx, int queue);
/* Raw cudaStream_t of a queue (for callers that time on the launching stream). */
int ooc_queue_handle(ooc_ctx* ctx, int queue, void** stream);

/* ------------------------------------------------------------ CUDA graphs
 * Capture the work issued on a queue between begin and end into an executable graph
 * (relaxed capture: NVRTC compiles may happen inside), replay it with one launch.
 * `kernels` = launches the graph holds, added to the statistics on every replay. */
typedef struct ooc_graph ooc_graph;
int ooc_graph_begin(ooc_ctx* ctx, int queue);
int ooc_graph_end(ooc_ctx* ctx, int queue, long long kernels, ooc_graph** out);
int ooc_graph_launch(ooc_ctx* ctx, int queue, ooc_graph* g);
void ooc_graph_destroy(ooc_graph* g);
/* 1 when every specialised-kernel structure seen so far has finished tile-shape
 * tuning. */
int ooc_jit_settled(void);
/* freeze = 1: launches of structures still being tuned use the fastest shape measured
 * so far (no timing launches) — set while capturing a graph. */
void ooc_jit_freeze(int freeze);

/* ------------------------------------------------------------ box views and copies */
/* A strided window covering the box [lo, hi) in global index space: element p
 * lives at data[sum_d (p[d]-lo[d]) * stride[d]]. The last used dimension
 * (ndim-1) must have stride 1 (row-major, extent.hpp:115-129); the others may be
 * padded (arena rows are padded to 128 B). For 3-D views stride[0] must be a
 * multiple of stride[1]. Unused trailing dims keep the reference's [0,1). */
typedef struct {
  double* data;
  int64_t lo[3];
  int64_t hi[3];
  int64_t stride[3];
} ooc_view;

enum { OOC_COPY_H2D = 1, OOC_COPY_D2H = 2, OOC_COPY_D2D = 3 };
/* Copy `region` (contained in both views) from src to dst on `queue`. */
int ooc_copy_box(ooc_ctx* ctx, int queue, int kind, const ooc_view* src, const ooc_view* dst,
                 const int64_t region_lo[3], const int64_t region_hi[3]);
/* Set every element of a device view's box to value (arena initialisation). */
int ooc_fill_box(ooc_ctx* ctx, int queue, const ooc_view* dst, double value);

/* ------------------------------------------------------------ loop launch */
/* Opcodes equal ooc::ExprOp (proj/include/ooc/expr.hpp:12-22). */
enum {
  OOC_OP_CONST = 0,
  OOC_OP_READ = 1,
  OOC_OP_COORD = 2,
  OOC_OP_ADD = 3,
  OOC_OP_SUB = 4,
  OOC_OP_MUL = 5,
  OOC_OP_DIV = 6,
  OOC_OP_MIN = 7,
  OOC_OP_MAX = 8
};
enum { OOC_RED_NONE = 0, OOC_RED_SUM = 1, OOC_RED_MIN = 2, OOC_RED_MAX = 3 };

typedef struct {
  int32_t op;
  int32_t arg;
  double value;
  int64_t offset[3];
} ooc_ins;

/* One par_loop over one (sub-)range. Tapes are postfix programs
 * (proj/src/expr.cpp:13-23): write tapes first (write_len[w] each), then the
 * reduction tape (reduce_len). Semantics of apply_loop: per point, every tape
 * is evaluated before any write lands; the reduction value of the range is
 * combined into accumulator `reduce_slot`. */
typedef struct {
  int32_t ndim;
  int64_t lo[3];
  int64_t hi[3];
  int32_t nargs;
  ooc_view args[OOC_MAX_ARGS];
  int32_t nwrites;
  int32_t write_arg[OOC_MAX_WRITES];
  int32_t write_len[OOC_MAX_WRITES];
  int32_t reduce_op;
  int32_t reduce_len;
  int32_t reduce_slot;
  int32_t ntape;
  const ooc_ins* tape;
} ooc_loop;

int ooc_launch_loop(ooc_ctx* ctx, int queue, const ooc_loop* loop);
/* One launch running n consecutive loops per point, in order (loop fusion).
 * Legal only when every cross-loop access is point-wise: a dataset written by an
 * earlier loop of the group is read by later ones at offset 0 only, and a dataset
 * read by an earlier loop is written by later ones only if that read was at
 * offset 0 (the host engine checks this). Points outside a loop's own range skip
 * it. Reducing loops are launched alone. Same observable result as n launches. */
int ooc_launch_group(ooc_ctx* ctx, int queue, const ooc_loop* loops, int n);

/* Row-sweep fusion (2-D, new): a run of consecutive loops — any stencils, including
 * column-offset reads of values written earlier in the run — executed by one kernel
 * that streams the mesh through shared-memory rings (csrc/device/sweep.cu). A dataset
 * the run both reads from memory and writes ("out of place") is written to a
 * caller-provided buffer of identical layout; every element of its view inside the
 * run's bounding box is written there, so the caller swaps the two buffers after the
 * launch. Everything else is updated in place. Same observable result as launching
 * the loops one by one (plus the swap).
 * ooc_sweep_check: 1 = the run is sweepable, 0 = not. flags (may be NULL) receive, per
 * loop i and argument a, flags[i*OOC_MAX_ARGS + a] = 1 (out of place) | 2 (read from
 * memory by the run) | 4 (written by the run).
 * A redirect with dst = NULL marks a dataset whose values the run produces but nobody
 * reads before they are overwritten (the caller's dead-store analysis): not stored,
 * and for an out-of-place dataset no swap. */
typedef struct {
  const double* src; /* view data of the dataset before the launch */
  double* dst;       /* buffer receiving its new values (same box and strides); NULL: dead */
} ooc_redirect;
int ooc_sweep_check(const ooc_loop* loops, int n, int* flags);
/* 3-D chains as plane-tile sweeps (threads over a dim-1 x column tile of each plane,
 * rings of plane tiles): 1 enables, 0 disables (default on; OOC_SWEEP_3D=0 turns them off). */
void ooc_sweep_set_3d(int on);
int ooc_sweep_3d_enabled(void);
int ooc_launch_sweep(ooc_ctx* ctx, int queue, const ooc_loop* loops, int n, const ooc_redirect* redirects,
                     int nredirects);
/* JSON description of the sweep plan (lags, halos, rings, load mode) and its compulsory
 * DRAM bytes — every array the run loads read once, every live output written once
 * (redirects mark dead outputs as in ooc_launch_sweep; may be NULL); compile = 1 also
 * builds the kernel with NVRTC for sm_100a (no GPU needed). */
int ooc_sweep_describe(const ooc_loop* loops, int n, const ooc_redirect* redirects, int nredirects, char* log,
                       int len, int compile);
/* JSON: the prefetch depth chosen per sweep structure and the measured ms per candidate. */
int ooc_sweep_report(char* buf, int len);

/* Specialised kernels: the par_loop kernel template instantiated per loop body
 * (or fused group) with NVRTC at first use, cached per process. mode 0: never
 * (interpreter only), 1: for launches of >= min_points points (default 2^18),
 * 2: always (error if NVRTC is unavailable). Env: OOC_JIT, OOC_JIT_MIN_POINTS. */
int ooc_jit_config(int mode, long long min_points);
/* Current specialisation policy (mode, threshold) as set by ooc_jit_config / OOC_JIT. */
int ooc_jit_policy(int* mode, long long* min_points);
/* Generate + NVRTC-compile (no load, no GPU needed) the specialised kernel of a
 * group; `log` receives the generated body or the compiler log. */
int ooc_jit_compile_check(const ooc_loop* loops, int n, char* log, int len);
/* JSON summary of the tile-shape autotuning of every specialised kernel. */
int ooc_jit_report(char* buf, int len);
/* "ok" or why specialisation is unavailable (NVRTC / driver not found). */
int ooc_jit_status(char* buf, int len);

/* ------------------------------------------------------------ reductions */
int ooc_reduce_reset(ooc_ctx* ctx, int queue, int slot, int op);
/* Asynchronous device->host read of a slot into page-locked `dst` on `queue`. */
int ooc_reduce_fetch(ooc_ctx* ctx, int queue, int slot, double* dst);
/* Exact mode (debug; default 0): a reducing launch writes one contribution per point
 * (row-major over its box) and one thread folds them into the slot in that order —
 * the reference's sequential fold (proj/src/kernel_exec.cpp:156-159, 193-197), bitwise.
 * Reducing groups then run loop by loop through the interpreter; ooc_launch_sweep
 * refuses reducing runs. The contribution buffer grows outside graph captures only. */
int ooc_set_reduce_exact(ooc_ctx* ctx, int on);

/* ------------------------------------------------------------ multi-GPU (NCCL) */
/* Slab decomposition plumbing (new; the reference is single-device).
 * ooc_comm_unique_id fills 128 opaque bytes on one rank; every rank passes them to
 * ooc_comm_init. Exchanges are grouped NCCL send/recv of contiguous device ranges
 * (whole rows of the outermost dimension), enqueued on `queue`. */
typedef struct {
  int peer;
  const double* send;
  int64_t send_count; /* doubles */
  double* recv;
  int64_t recv_count;
} ooc_xfer;
int ooc_comm_unique_id(void* out128);
int ooc_comm_init(ooc_ctx* ctx, int rank, int world, const void* id128);
/* CUDA-IPC transport (new): the ranks of one node rendezvous in a POSIX shared-memory
 * segment named by `name` (same string on every rank, unique per job); exchanges pack
 * the sends into a device outbox the peers map with cudaIpcOpenMemHandle and pull from
 * after a host barrier (peer-to-peer over NVLink; a device copy when ranks share a GPU).
 * Collective: every rank makes the same sequence of exchange / all-reduce calls. */
int ooc_comm_init_ipc(ooc_ctx* ctx, int rank, int world, const char* name);
/* Host barrier of the IPC transport (OOC_ERR_UNSUPPORTED for NCCL communicators). */
int ooc_comm_barrier(ooc_ctx* ctx);
int ooc_comm_exchange(ooc_ctx* ctx, int queue, const ooc_xfer* xfers, int n);
/* All-reduce of one reduction accumulator across the communicator (sum/min/max). */
int ooc_reduce_allreduce(ooc_ctx* ctx, int queue, int slot, int op);
void ooc_comm_release(ooc_ctx* ctx);

/* ------------------------------------------------------------ statistics */
typedef struct {
  long long kernel_launches;
  long long interp_launches;
  long long special_launches;
  long long h2d_bytes, d2h_bytes, d2d_bytes;
  long long copy_calls;
  long long jit_launches, jit_compiles, jit_compile_ms;
  long long comm_bytes;
  long long jit_host_us;  /* host time spent preparing specialised launches */
  long long graph_launches;
  long long jit_unsettled;  /* specialised launches made while their shape was still being tuned */
  long long sweep_launches; /* row-sweep launches (ooc_launch_sweep) */
  long long sweep_host_us;  /* host time spent inside ooc_launch_sweep (plan lookup, parameters, launch) */
} ooc_dev_stats;
int ooc_stats(ooc_ctx* ctx, ooc_dev_stats* out);
int ooc_stats_reset(ooc_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* OOC_DEVICE_H */
