// Device layer: contexts, pinned host memory, HBM memory manager, queues/events,
// strided box copies. Implements include/ooc_device.h (except loop launch /
// reductions, in loop_kernels.cu).
#include <sched.h>

#include <cctype>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <mutex>
#include <string>
#include <unordered_set>

#include "internal.cuh"

namespace oocdev {

namespace {
thread_local std::string g_error;
std::mutex g_host_mu;
std::unordered_set<void*>* g_pinned = nullptr;  // pointers from ooc_host_alloc
}  // namespace

void set_error(const std::string& msg) { g_error = msg; }

}  // namespace oocdev

using namespace oocdev;

namespace {

// canonical (a, b, c) dims of a rank: c = ndim-1 contiguous, b = ndim-2, a = ndim-3
void canon_dims(int ndim, int& a, int& b, int& c) {
  c = ndim - 1;
  b = ndim >= 2 ? ndim - 2 : -1;
  a = ndim >= 3 ? ndim - 3 : -1;
}

int view_rank(const ooc_view& v) {
  // rank = highest dim whose box is not the trailing [0,1) convention
  for (int d = 2; d >= 1; --d)
    if (!(v.lo[d] == 0 && v.hi[d] == 1)) return d + 1;
  return 1;
}

bool box_contains(const ooc_view& v, const int64_t lo[3], const int64_t hi[3]) {
  for (int d = 0; d < 3; ++d)
    if (lo[d] < v.lo[d] || hi[d] > v.hi[d]) return false;
  return true;
}

}  // namespace

extern "C" {

const char* ooc_dev_last_error(void) { return g_error.c_str(); }

const char* ooc_dev_build_info(void) {
  return "ooc-b200 device layer; sm_100a; interpreter+stream engine; " __DATE__;
}

int ooc_dev_count(int* n) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *n = 0;
    set_error(cudaGetErrorString(e));
    return OOC_ERR_NODEV;
  }
  *n = c;
  return OOC_OK;
}

// NUMA placement of page-locked memory: with a preferred device set for the calling
// thread, cudaHostAlloc runs with the thread bound to the CPUs local to that GPU
// (/sys/bus/pci/devices/<bus id>/local_cpulist), so the pinned pages — each rank's slab,
// streamed over its own link — live on the GPU's socket. A no-op on single-node hosts.
static thread_local int g_numa_dev = -1;

int ooc_host_numa_device(int device) {
  g_numa_dev = device;
  return OOC_OK;
}

static bool local_cpus(int device, cpu_set_t* set) {
  char bus[64] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  std::string id(bus);
  for (char& ch : id) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
  std::ifstream in("/sys/bus/pci/devices/" + id + "/local_cpulist");
  std::string list;
  if (!in || !std::getline(in, list) || list.empty()) return false;
  CPU_ZERO(set);
  std::size_t i = 0;
  int n = 0;
  while (i < list.size()) {
    std::size_t j = list.find(',', i);
    if (j == std::string::npos) j = list.size();
    const std::string part = list.substr(i, j - i);
    const std::size_t dash = part.find('-');
    const int a = std::atoi(part.c_str()), b = dash == std::string::npos ? a : std::atoi(part.c_str() + dash + 1);
    for (int c = a; c <= b && c < CPU_SETSIZE; ++c, ++n) CPU_SET(c, set);
    i = j + 1;
  }
  return n > 0;
}

int ooc_host_alloc(size_t bytes, void** out) {
  static int has_dev = -1;
  if (has_dev < 0) {
    int n = 0;
    has_dev = (ooc_dev_count(&n) == OOC_OK && n > 0) ? 1 : 0;
  }
  if (!has_dev) {
    set_error("no CUDA device: cannot allocate page-locked memory");
    return OOC_ERR_NODEV;
  }
  void* p = nullptr;
  cpu_set_t old_set, want;
  const bool bind = g_numa_dev >= 0 && sched_getaffinity(0, sizeof old_set, &old_set) == 0 && local_cpus(g_numa_dev, &want) &&
                    sched_setaffinity(0, sizeof want, &want) == 0;
  cudaError_t e = cudaHostAlloc(&p, bytes, cudaHostAllocPortable);
  if (bind) sched_setaffinity(0, sizeof old_set, &old_set);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error(std::string("cudaHostAlloc: ") + cudaGetErrorString(e));
    return OOC_ERR_CUDA;
  }
  std::lock_guard<std::mutex> lk(g_host_mu);
  if (!g_pinned) g_pinned = new std::unordered_set<void*>();
  g_pinned->insert(p);
  *out = p;
  return OOC_OK;
}

int ooc_host_free(void* p) {
  {
    std::lock_guard<std::mutex> lk(g_host_mu);
    if (!g_pinned || !g_pinned->erase(p)) {
      set_error("ooc_host_free: pointer not from ooc_host_alloc");
      return OOC_ERR_ARG;
    }
  }
  OOC_CUDA_TRY(cudaFreeHost(p));
  return OOC_OK;
}

int ooc_ctx_create(int device, ooc_ctx** out) {
  int n = 0;
  if (ooc_dev_count(&n) != OOC_OK || device < 0 || device >= n) {
    set_error("ooc_ctx_create: no CUDA device " + std::to_string(device));
    return OOC_ERR_NODEV;
  }
  auto* c = new ooc_ctx;
  c->device = device;
  OOC_CUDA_TRY(cudaSetDevice(device));
  OOC_CUDA_TRY(cudaGetDeviceProperties(&c->prop, device));
  for (int q = 0; q < OOC_NUM_QUEUES; ++q)
    OOC_CUDA_TRY(cudaStreamCreateWithFlags(&c->q[q], cudaStreamNonBlocking));
  OOC_CUDA_TRY(cudaMalloc(&c->red_acc, OOC_REDUCE_SLOTS * sizeof(double)));
  OOC_CUDA_TRY(cudaMemset(c->red_acc, 0, OOC_REDUCE_SLOTS * sizeof(double)));
  c->red_part_cap = 8192;
  for (int q = 0; q < OOC_NUM_QUEUES; ++q)
    OOC_CUDA_TRY(cudaMalloc(&c->red_part[q], c->red_part_cap * sizeof(double)));
  *out = c;
  return OOC_OK;
}

int ooc_ctx_destroy(ooc_ctx* c) {
  if (!c) return OOC_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  ooc_comm_release(c);
  for (auto& [p, sz] : c->allocs) cudaFree(p);
  cudaFree(c->red_acc);
  for (int q = 0; q < OOC_NUM_QUEUES; ++q) {
    cudaFree(c->red_part[q]);
    cudaFree(c->red_scratch[q]);
    cudaStreamDestroy(c->q[q]);
  }
  delete c;
  return OOC_OK;
}

int ooc_ctx_props(ooc_ctx* c, ooc_dev_props* o) {
  OOC_ARG_CHECK(c && o, "ooc_ctx_props: null");
  std::memset(o, 0, sizeof *o);
  o->device = c->device;
  o->sm_count = c->prop.multiProcessorCount;
  o->cc_major = c->prop.major;
  o->cc_minor = c->prop.minor;
  o->l2_bytes = c->prop.l2CacheSize;
  o->hbm_bytes = static_cast<long long>(c->prop.totalGlobalMem);
  size_t fr = 0, tot = 0;
  OOC_CUDA_TRY(cudaSetDevice(c->device));
  OOC_CUDA_TRY(cudaMemGetInfo(&fr, &tot));
  o->free_bytes = static_cast<long long>(fr);
  std::snprintf(o->name, sizeof o->name, "%s", c->prop.name);
  return OOC_OK;
}

int ooc_ctx_sync(ooc_ctx* c) {
  OOC_ARG_CHECK(c, "ooc_ctx_sync: null");
  for (int q = 0; q < OOC_NUM_QUEUES; ++q) OOC_CUDA_TRY(cudaStreamSynchronize(c->q[q]));
  return OOC_OK;
}

// ------------------------------------------------------------ memory manager

int ooc_mem_alloc(ooc_ctx* c, size_t bytes, void** out) {
  OOC_ARG_CHECK(c && out, "ooc_mem_alloc: null");
  if (bytes == 0) bytes = 256;
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error("ooc_mem_alloc(" + std::to_string(bytes) + " B): " + cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? OOC_ERR_CAPACITY : OOC_ERR_CUDA;
  }
  c->allocs[p] = bytes;
  c->in_use += static_cast<long long>(bytes);
  if (c->in_use > c->peak) c->peak = c->in_use;
  *out = p;
  return OOC_OK;
}

int ooc_mem_free(ooc_ctx* c, void* p) {
  OOC_ARG_CHECK(c, "ooc_mem_free: null ctx");
  if (!p) return OOC_OK;
  auto it = c->allocs.find(p);
  OOC_ARG_CHECK(it != c->allocs.end(), "ooc_mem_free: unknown pointer");
  c->in_use -= static_cast<long long>(it->second);
  c->allocs.erase(it);
  OOC_CUDA_TRY(cudaFree(p));
  return OOC_OK;
}

int ooc_mem_usage(ooc_ctx* c, long long* in_use, long long* peak) {
  OOC_ARG_CHECK(c, "ooc_mem_usage: null");
  if (in_use) *in_use = c->in_use;
  if (peak) *peak = c->peak;
  return OOC_OK;
}

// ------------------------------------------------------------ queues and events

int ooc_event_create(ooc_ctx* c, int timing, ooc_event** out) {
  OOC_ARG_CHECK(c && out, "ooc_event_create: null");
  auto* e = new ooc_event;
  OOC_CUDA_TRY(cudaEventCreateWithFlags(&e->ev, timing ? cudaEventDefault : cudaEventDisableTiming));
  *out = e;
  return OOC_OK;
}

int ooc_event_destroy(ooc_ctx*, ooc_event* e) {
  if (!e) return OOC_OK;
  cudaEventDestroy(e->ev);
  delete e;
  return OOC_OK;
}

int ooc_event_record(ooc_ctx* c, ooc_event* e, int q) {
  OOC_ARG_CHECK(c && e && q >= 0 && q < OOC_NUM_QUEUES, "ooc_event_record: bad args");
  OOC_CUDA_TRY(cudaEventRecord(e->ev, c->q[q]));
  return OOC_OK;
}

int ooc_queue_wait(ooc_ctx* c, int q, ooc_event* e) {
  OOC_ARG_CHECK(c && e && q >= 0 && q < OOC_NUM_QUEUES, "ooc_queue_wait: bad args");
  OOC_CUDA_TRY(cudaStreamWaitEvent(c->q[q], e->ev, 0));
  return OOC_OK;
}

int ooc_event_sync(ooc_ctx*, ooc_event* e) {
  OOC_ARG_CHECK(e, "ooc_event_sync: null");
  OOC_CUDA_TRY(cudaEventSynchronize(e->ev));
  return OOC_OK;
}

int ooc_event_query(ooc_ctx*, ooc_event* e, int* done) {
  OOC_ARG_CHECK(e && done, "ooc_event_query: null");
  cudaError_t r = cudaEventQuery(e->ev);
  if (r == cudaErrorNotReady) {
    *done = 0;
    return OOC_OK;
  }
  OOC_CUDA_TRY(r);
  *done = 1;
  return OOC_OK;
}

int ooc_event_elapsed_ms(ooc_event* a, ooc_event* b, float* ms) {
  OOC_ARG_CHECK(a && b && ms, "ooc_event_elapsed_ms: null");
  OOC_CUDA_TRY(cudaEventElapsedTime(ms, a->ev, b->ev));
  return OOC_OK;
}

int ooc_queue_sync(ooc_ctx* c, int q) {
  OOC_ARG_CHECK(c && q >= 0 && q < OOC_NUM_QUEUES, "ooc_queue_sync: bad args");
  OOC_CUDA_TRY(cudaStreamSynchronize(c->q[q]));
  return OOC_OK;
}

int ooc_queue_handle(ooc_ctx* c, int q, void** s) {
  OOC_ARG_CHECK(c && s && q >= 0 && q < OOC_NUM_QUEUES, "ooc_queue_handle: bad args");
  *s = c->q[q];
  return OOC_OK;
}

// ------------------------------------------------------------ strided box copies
// One cudaMemcpy{,2D,3D}Async per region (never the batched memcpy APIs).

int ooc_copy_box(ooc_ctx* c, int q, int kind, const ooc_view* src, const ooc_view* dst,
                 const int64_t lo[3], const int64_t hi[3]) {
  OOC_ARG_CHECK(c && src && dst && q >= 0 && q < OOC_NUM_QUEUES, "ooc_copy_box: bad args");
  for (int d = 0; d < 3; ++d)
    if (hi[d] <= lo[d]) return OOC_OK;  // empty region
  OOC_ARG_CHECK(box_contains(*src, lo, hi), "ooc_copy_box: region outside the source box");
  OOC_ARG_CHECK(box_contains(*dst, lo, hi), "ooc_copy_box: region outside the destination box");
  const int nd = std::max(view_rank(*src), view_rank(*dst));
  int A, B, C;
  canon_dims(nd, A, B, C);
  OOC_ARG_CHECK(src->stride[C] == 1 && dst->stride[C] == 1,
                "ooc_copy_box: innermost dimension must be contiguous");
  cudaMemcpyKind k = kind == OOC_COPY_H2D   ? cudaMemcpyHostToDevice
                     : kind == OOC_COPY_D2H ? cudaMemcpyDeviceToHost
                                            : cudaMemcpyDeviceToDevice;
  auto addr = [&](const ooc_view* v) {
    int64_t off = 0;
    for (int d = 0; d < 3; ++d) off += (lo[d] - v->lo[d]) * v->stride[d];
    return v->data + off;
  };
  double* s = addr(src);
  double* t = addr(dst);
  const size_t width = static_cast<size_t>(hi[C] - lo[C]) * sizeof(double);
  const size_t rows = B >= 0 ? static_cast<size_t>(hi[B] - lo[B]) : 1;
  const size_t planes = A >= 0 ? static_cast<size_t>(hi[A] - lo[A]) : 1;
  cudaStream_t st = c->q[q];
  // Collapse what is contiguous on both sides: one 1-D copy when the whole region is
  // (H2D pitched 3-D copies run at ~34 GB/s on B200 + PCIe 5, 1-D ones at ~55), one
  // 2-D copy of whole planes when each plane is.
  const int64_t w = hi[C] - lo[C];
  auto rows_dense = [&](const ooc_view* v) { return rows == 1 || v->stride[B] == w; };
  auto dense = [&](const ooc_view* v) {
    return rows_dense(v) && (planes == 1 || v->stride[A] == w * static_cast<int64_t>(rows));
  };
  if (dense(src) && dense(dst)) {
    OOC_CUDA_TRY(cudaMemcpyAsync(t, s, width * rows * planes, k, st));
  } else if (planes > 1 && rows_dense(src) && rows_dense(dst)) {
    OOC_CUDA_TRY(cudaMemcpy2DAsync(t, static_cast<size_t>(dst->stride[A]) * sizeof(double), s,
                                   static_cast<size_t>(src->stride[A]) * sizeof(double), width * rows, planes, k,
                                   st));
  } else if (planes == 1 && rows == 1) {
    OOC_CUDA_TRY(cudaMemcpyAsync(t, s, width, k, st));
  } else if (planes == 1) {
    OOC_CUDA_TRY(cudaMemcpy2DAsync(t, static_cast<size_t>(dst->stride[B]) * sizeof(double), s,
                                   static_cast<size_t>(src->stride[B]) * sizeof(double), width,
                                   rows, k, st));
  } else {
    OOC_ARG_CHECK(src->stride[A] % src->stride[B] == 0 && dst->stride[A] % dst->stride[B] == 0,
                  "ooc_copy_box: plane stride must be a multiple of the row stride");
    cudaMemcpy3DParms p{};
    p.srcPtr = make_cudaPitchedPtr(s, static_cast<size_t>(src->stride[B]) * sizeof(double), width,
                                   static_cast<size_t>(src->stride[A] / src->stride[B]));
    p.dstPtr = make_cudaPitchedPtr(t, static_cast<size_t>(dst->stride[B]) * sizeof(double), width,
                                   static_cast<size_t>(dst->stride[A] / dst->stride[B]));
    p.extent = make_cudaExtent(width, rows, planes);
    p.kind = k;
    OOC_CUDA_TRY(cudaMemcpy3DAsync(&p, st));
  }
  const long long bytes = static_cast<long long>(width * rows * planes);
  if (kind == OOC_COPY_H2D) c->stats.h2d_bytes += bytes;
  else if (kind == OOC_COPY_D2H) c->stats.d2h_bytes += bytes;
  else c->stats.d2d_bytes += bytes;
  ++c->stats.copy_calls;
  return OOC_OK;
}

int ooc_stats(ooc_ctx* c, ooc_dev_stats* o) {
  OOC_ARG_CHECK(c && o, "ooc_stats: null");
  *o = c->stats;
  return OOC_OK;
}

int ooc_stats_reset(ooc_ctx* c) {
  OOC_ARG_CHECK(c, "ooc_stats_reset: null");
  c->stats = ooc_dev_stats{};
  return OOC_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ CUDA graphs
struct ooc_graph {
  cudaGraphExec_t exec = nullptr;
  long long kernels = 0;
};

int ooc_graph_begin(ooc_ctx* c, int q) {
  OOC_ARG_CHECK(c && q >= 0 && q < OOC_NUM_QUEUES, "ooc_graph_begin: bad args");
  OOC_CUDA_TRY(cudaStreamBeginCapture(c->q[q], cudaStreamCaptureModeRelaxed));
  c->capture_launches0 = c->stats.kernel_launches;
  return OOC_OK;
}

int ooc_graph_end(ooc_ctx* c, int q, long long kernels, ooc_graph** out) {
  OOC_ARG_CHECK(c && out && q >= 0 && q < OOC_NUM_QUEUES, "ooc_graph_end: bad args");
  cudaGraph_t g = nullptr;
  OOC_CUDA_TRY(cudaStreamEndCapture(c->q[q], &g));
  auto* G = new ooc_graph;
  G->kernels = kernels >= 0 ? kernels : c->stats.kernel_launches - c->capture_launches0;
  cudaError_t e = cudaGraphInstantiate(&G->exec, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) {
    delete G;
    OOC_CUDA_TRY(e);
  }
  // captured launches did not run: the replay that follows counts them
  c->stats.kernel_launches = c->capture_launches0;
  *out = G;
  return OOC_OK;
}

int ooc_graph_launch(ooc_ctx* c, int q, ooc_graph* g) {
  OOC_ARG_CHECK(c && g && q >= 0 && q < OOC_NUM_QUEUES, "ooc_graph_launch: bad args");
  OOC_CUDA_TRY(cudaGraphLaunch(g->exec, c->q[q]));
  c->stats.kernel_launches += g->kernels;
  c->stats.graph_launches++;
  return OOC_OK;
}

void ooc_graph_destroy(ooc_graph* g) {
  if (!g) return;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  delete g;
}
