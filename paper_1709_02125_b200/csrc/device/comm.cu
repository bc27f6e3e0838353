// Multi-GPU plumbing of the device layer for the slab decomposition: ghost-band
// exchange between neighbouring ranks and all-reduce of reduction accumulators, both
// ordered on a queue of the context. Two transports:
//   NCCL  (opened lazily with dlopen): grouped point-to-point send/recv + ncclAllReduce,
//         enqueued without host syncs (one process per GPU, distinct GPUs).
//   IPC   (CUDA IPC + a POSIX shared-memory rendezvous between the ranks of one node):
//         each rank packs what it sends into a device "outbox" whose IPC handle the
//         peers map once; after a host barrier every rank pulls its ghost bands straight
//         out of the neighbours' outboxes with cudaMemcpyAsync — peer-to-peer over
//         NVLink between GPUs, a device copy when ranks share a GPU (which NCCL refuses,
//         so this is also how the multi-rank data path runs on a single GPU).
#include <dlfcn.h>
#include <nccl.h>

#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "internal.cuh"

using namespace oocdev;

namespace {

struct Nccl {
  bool tried = false, ok = false;
  std::string why;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
  static Nccl n;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (n.tried) return n;
  n.tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    n.why = "dlopen libnccl.so.2 failed";
    return n;
  }
#define BIND(field, name) *reinterpret_cast<void**>(&n.field) = dlsym(h, name)
  BIND(get_unique_id, "ncclGetUniqueId");
  BIND(comm_init_rank, "ncclCommInitRank");
  BIND(comm_destroy, "ncclCommDestroy");
  BIND(send, "ncclSend");
  BIND(recv, "ncclRecv");
  BIND(group_start, "ncclGroupStart");
  BIND(group_end, "ncclGroupEnd");
  BIND(all_reduce, "ncclAllReduce");
  BIND(error_string, "ncclGetErrorString");
#undef BIND
  n.ok = n.get_unique_id && n.comm_init_rank && n.comm_destroy && n.send && n.recv &&
         n.group_start && n.group_end && n.all_reduce;
  if (!n.ok) n.why = "libnccl.so.2 lacks required entry points";
  return n;
}

int nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return OOC_OK;
  const char* s = nccl().error_string ? nccl().error_string(r) : "?";
  set_error(std::string(what) + ": " + s);
  return OOC_ERR_CUDA;
}

}  // namespace


// ---------------------------------------------------------------- CUDA-IPC transport
namespace {

constexpr int kIpcMaxRanks = 64;
constexpr std::uint32_t kIpcMagic = 0x0c0c1709u;

struct IpcRankSlot {
  std::atomic<std::uint64_t> gen[2];       // outbox generation per exchange parity (0: none yet)
  cudaIpcMemHandle_t handle[2];
  std::int64_t off[2][kIpcMaxRanks];       // doubles: start of the segment destined to each rank
  double red[2];                           // reduction partial per all-reduce parity
  int device, pid;
};
struct IpcShm {
  std::atomic<std::uint32_t> magic, joined, count, sense;
  int world;
  IpcRankSlot r[kIpcMaxRanks];
};
struct IpcPeer {
  std::uint64_t gen[2] = {0, 0};
  double* base[2] = {nullptr, nullptr};
};
struct IpcComm {
  IpcShm* shm = nullptr;
  std::string name;
  int rank = 0, world = 1;
  std::uint32_t sense = 0;
  double* outbox[2] = {nullptr, nullptr};
  std::size_t cap[2] = {0, 0};  // doubles
  std::uint64_t gen[2] = {0, 0};
  long long exchanges = 0, reductions = 0;
  std::vector<IpcPeer> peers;
};

double ipc_timeout_s() {
  static const double t = [] {
    const char* e = std::getenv("OOC_IPC_TIMEOUT");
    return e ? std::atof(e) : 300.0;
  }();
  return t;
}

// Sense-reversing barrier over the shared segment (host threads only: no GPU work ever
// waits on another rank, so ranks sharing one GPU never block each other's kernels).
int ipc_barrier(IpcComm& m) {
  m.sense ^= 1u;
  if (m.shm->count.fetch_add(1, std::memory_order_acq_rel) + 1 == static_cast<std::uint32_t>(m.world)) {
    m.shm->count.store(0, std::memory_order_relaxed);
    m.shm->sense.store(m.sense, std::memory_order_release);
    return OOC_OK;
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (unsigned spin = 0; m.shm->sense.load(std::memory_order_acquire) != m.sense; ++spin) {
    if (spin > 256) {
      sched_yield();
      if ((spin & 1023) == 0 &&
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > ipc_timeout_s()) {
        set_error("ipc barrier: rank " + std::to_string(m.rank) + " timed out waiting for its peers");
        return OOC_ERR_CUDA;
      }
    }
  }
  return OOC_OK;
}

void ipc_close(ooc_ctx* c) {
  auto* m = static_cast<IpcComm*>(c->ipc);
  if (!m) return;
  cudaSetDevice(c->device);
  for (IpcPeer& p : m->peers)
    for (double* b : p.base)
      if (b) cudaIpcCloseMemHandle(b);
  for (double* o : m->outbox)
    if (o) cudaFree(o);
  if (m->shm) munmap(m->shm, sizeof(IpcShm));
  delete m;
  c->ipc = nullptr;
}

int ipc_exchange(ooc_ctx* c, int q, const ooc_xfer* x, int n) {
  IpcComm& m = *static_cast<IpcComm*>(c->ipc);
  const int par = static_cast<int>(m.exchanges++ & 1);
  // outbox layout: one segment per destination rank (ascending), each the concatenation
  // of this rank's sends to it in call order — the receiver finds its data by the same order
  std::vector<std::int64_t> seg(static_cast<std::size_t>(m.world), 0), cur(static_cast<std::size_t>(m.world), 0);
  for (int i = 0; i < n; ++i) {
    OOC_ARG_CHECK(x[i].peer >= 0 && x[i].peer < m.world && x[i].peer != m.rank, "ooc_comm_exchange: bad peer");
    seg[static_cast<std::size_t>(x[i].peer)] += x[i].send_count;
  }
  std::int64_t total = 0;
  for (int r = 0; r < m.world; ++r) {
    const std::int64_t len = seg[static_cast<std::size_t>(r)];
    seg[static_cast<std::size_t>(r)] = total;
    cur[static_cast<std::size_t>(r)] = total;
    total += len;
  }
  cudaStream_t st = c->q[q];
  if (static_cast<std::size_t>(total) > m.cap[par]) {
    // peers finished reading this parity's outbox before the previous barrier
    OOC_CUDA_TRY(cudaStreamSynchronize(st));
    if (m.outbox[par]) OOC_CUDA_TRY(cudaFree(m.outbox[par]));
    m.outbox[par] = nullptr;
    const std::size_t cap = static_cast<std::size_t>(total) + static_cast<std::size_t>(total) / 4 + 4096;
    OOC_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&m.outbox[par]), cap * sizeof(double)));
    m.cap[par] = cap;
    OOC_CUDA_TRY(cudaIpcGetMemHandle(&m.shm->r[m.rank].handle[par], m.outbox[par]));
    m.gen[par] += 1;
  }
  for (int i = 0; i < n; ++i)
    if (x[i].send_count > 0) {
      std::int64_t& o = cur[static_cast<std::size_t>(x[i].peer)];
      OOC_CUDA_TRY(cudaMemcpyAsync(m.outbox[par] + o, x[i].send, static_cast<std::size_t>(x[i].send_count) * 8,
                                   cudaMemcpyDeviceToDevice, st));
      o += x[i].send_count;
    }
  IpcRankSlot& me = m.shm->r[m.rank];
  for (int r = 0; r < m.world; ++r) me.off[par][r] = seg[static_cast<std::size_t>(r)];
  me.gen[par].store(m.gen[par], std::memory_order_release);
  OOC_CUDA_TRY(cudaStreamSynchronize(st));  // the outbox is complete before any peer reads it
  int rc = ipc_barrier(m);
  if (rc) return rc;
  std::vector<std::int64_t> taken(static_cast<std::size_t>(m.world), 0);
  for (int i = 0; i < n; ++i) {
    if (x[i].recv_count <= 0) continue;
    const int p = x[i].peer;
    const IpcRankSlot& ps = m.shm->r[p];
    IpcPeer& pc = m.peers[static_cast<std::size_t>(p)];
    const std::uint64_t g = ps.gen[par].load(std::memory_order_acquire);
    if (g == 0) {
      set_error("ooc_comm_exchange: peer " + std::to_string(p) + " published no outbox");
      return OOC_ERR_ARG;
    }
    if (g != pc.gen[par]) {  // first exchange, or the peer grew its outbox
      if (pc.base[par]) OOC_CUDA_TRY(cudaIpcCloseMemHandle(pc.base[par]));
      void* b = nullptr;
      OOC_CUDA_TRY(cudaIpcOpenMemHandle(&b, ps.handle[par], cudaIpcMemLazyEnablePeerAccess));
      pc.base[par] = static_cast<double*>(b);
      pc.gen[par] = g;
    }
    const double* src = pc.base[par] + ps.off[par][m.rank] + taken[static_cast<std::size_t>(p)];
    OOC_CUDA_TRY(cudaMemcpyAsync(x[i].recv, src, static_cast<std::size_t>(x[i].recv_count) * 8,
                                 cudaMemcpyDeviceToDevice, st));
    taken[static_cast<std::size_t>(p)] += x[i].recv_count;
  }
  for (int i = 0; i < n; ++i) c->stats.comm_bytes += 8 * (x[i].send_count + x[i].recv_count);
  return OOC_OK;
}

// All-reduce of one accumulator: every rank publishes its value, then folds all of them
// in rank order (the same order on every rank: identical results everywhere).
int ipc_allreduce(ooc_ctx* c, int q, int slot, int op) {
  IpcComm& m = *static_cast<IpcComm*>(c->ipc);
  const int par = static_cast<int>(m.reductions++ & 1);
  cudaStream_t st = c->q[q];
  double v = 0.0;
  OOC_CUDA_TRY(cudaMemcpyAsync(&v, c->red_acc + slot, sizeof v, cudaMemcpyDeviceToHost, st));
  OOC_CUDA_TRY(cudaStreamSynchronize(st));
  m.shm->r[m.rank].red[par] = v;
  int rc = ipc_barrier(m);
  if (rc) return rc;
  double acc = m.shm->r[0].red[par];
  for (int r = 1; r < m.world; ++r) {
    const double w = m.shm->r[r].red[par];
    acc = op == OOC_RED_MIN ? (w < acc ? w : acc) : op == OOC_RED_MAX ? (acc < w ? w : acc) : acc + w;
  }
  OOC_CUDA_TRY(cudaMemcpyAsync(c->red_acc + slot, &acc, sizeof acc, cudaMemcpyHostToDevice, st));
  OOC_CUDA_TRY(cudaStreamSynchronize(st));
  return OOC_OK;
}

}  // namespace

extern "C" {

int ooc_comm_unique_id(void* out) {
  OOC_ARG_CHECK(out, "ooc_comm_unique_id: null");
  Nccl& n = nccl();
  if (!n.ok) {
    set_error(n.why);
    return OOC_ERR_UNSUPPORTED;
  }
  ncclUniqueId id;
  int rc = nccl_check(n.get_unique_id(&id), "ncclGetUniqueId");
  if (rc) return rc;
  std::memcpy(out, &id, sizeof id);
  return OOC_OK;
}

int ooc_comm_init(ooc_ctx* c, int rank, int world, const void* id_bytes) {
  OOC_ARG_CHECK(c && id_bytes && world >= 1 && rank >= 0 && rank < world, "ooc_comm_init: bad args");
  Nccl& n = nccl();
  if (!n.ok) {
    set_error(n.why);
    return OOC_ERR_UNSUPPORTED;
  }
  ncclUniqueId id;
  std::memcpy(&id, id_bytes, sizeof id);
  OOC_CUDA_TRY(cudaSetDevice(c->device));
  ncclComm_t comm;
  int rc = nccl_check(n.comm_init_rank(&comm, world, id, rank), "ncclCommInitRank");
  if (rc) return rc;
  c->comm = comm;
  c->rank = rank;
  c->world = world;
  return OOC_OK;
}

int ooc_comm_init_ipc(ooc_ctx* c, int rank, int world, const char* name) {
  OOC_ARG_CHECK(c && name && name[0] && world >= 1 && world <= kIpcMaxRanks && rank >= 0 && rank < world,
                "ooc_comm_init_ipc: bad args");
  OOC_ARG_CHECK(!c->comm && !c->ipc, "ooc_comm_init_ipc: the context already has a communicator");
  OOC_CUDA_TRY(cudaSetDevice(c->device));
  const std::string nm = std::string("/ooc_") + name;
  int fd = -1;
  const auto t0 = std::chrono::steady_clock::now();
  auto late = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > ipc_timeout_s(); };
  if (rank == 0) {
    shm_unlink(nm.c_str());  // a leftover of a crashed run with the same name
    fd = shm_open(nm.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
    if (fd < 0 || ftruncate(fd, sizeof(IpcShm)) != 0) {
      set_error("ooc_comm_init_ipc: cannot create shared segment " + nm);
      if (fd >= 0) close(fd);
      return OOC_ERR_CUDA;
    }
  } else {
    struct stat sb {};
    for (;;) {  // wait until rank 0 has created and sized the segment
      fd = shm_open(nm.c_str(), O_RDWR, 0600);
      if (fd >= 0 && fstat(fd, &sb) == 0 && static_cast<std::size_t>(sb.st_size) >= sizeof(IpcShm)) break;
      if (fd >= 0) close(fd);
      fd = -1;
      if (late()) {
        set_error("ooc_comm_init_ipc: rank " + std::to_string(rank) + " found no segment " + nm);
        return OOC_ERR_CUDA;
      }
      usleep(1000);
    }
  }
  void* mem = mmap(nullptr, sizeof(IpcShm), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (mem == MAP_FAILED) {
    set_error("ooc_comm_init_ipc: mmap failed");
    return OOC_ERR_CUDA;
  }
  auto* shm = static_cast<IpcShm*>(mem);
  if (rank == 0) {
    shm->world = world;  // the segment arrives zero-filled (ftruncate)
    shm->magic.store(kIpcMagic, std::memory_order_release);
  } else {
    while (shm->magic.load(std::memory_order_acquire) != kIpcMagic) {
      if (late()) {
        munmap(mem, sizeof(IpcShm));
        set_error("ooc_comm_init_ipc: segment never initialised");
        return OOC_ERR_CUDA;
      }
      usleep(1000);
    }
    if (shm->world != world) {
      munmap(mem, sizeof(IpcShm));
      set_error("ooc_comm_init_ipc: world size differs from rank 0's");
      return OOC_ERR_ARG;
    }
  }
  auto* m = new IpcComm;
  m->shm = shm;
  m->name = nm;
  m->rank = rank;
  m->world = world;
  m->peers.resize(static_cast<std::size_t>(world));
  shm->r[rank].device = c->device;
  shm->r[rank].pid = static_cast<int>(getpid());
  shm->joined.fetch_add(1, std::memory_order_acq_rel);
  c->ipc = m;
  c->rank = rank;
  c->world = world;
  int rc = ipc_barrier(*m);  // everyone mapped the segment: its name can go
  if (rc) {
    ipc_close(c);
    return rc;
  }
  if (rank == 0) shm_unlink(nm.c_str());
  return OOC_OK;
}

int ooc_comm_barrier(ooc_ctx* c) {
  OOC_ARG_CHECK(c, "ooc_comm_barrier: null");
  if (c->ipc) return ipc_barrier(*static_cast<IpcComm*>(c->ipc));
  OOC_ARG_CHECK(c->comm, "ooc_comm_barrier: no communicator");
  return OOC_ERR_UNSUPPORTED;  // NCCL ranks order through their streams
}

int ooc_comm_exchange(ooc_ctx* c, int q, const ooc_xfer* x, int n) {
  OOC_ARG_CHECK(c && (x || n == 0) && q >= 0 && q < OOC_NUM_QUEUES, "ooc_comm_exchange: bad args");
  if (c->ipc) return ipc_exchange(c, q, x, n);
  OOC_ARG_CHECK(c->comm, "ooc_comm_exchange: no communicator (ooc_comm_init / ooc_comm_init_ipc)");
  Nccl& nc = nccl();
  auto comm = static_cast<ncclComm_t>(c->comm);
  int rc = nccl_check(nc.group_start(), "ncclGroupStart");
  if (rc) return rc;
  for (int i = 0; i < n; ++i) {
    if (x[i].send_count > 0)
      rc |= nccl_check(nc.send(x[i].send, static_cast<size_t>(x[i].send_count), ncclFloat64, x[i].peer,
                               comm, c->q[q]), "ncclSend");
    if (x[i].recv_count > 0)
      rc |= nccl_check(nc.recv(x[i].recv, static_cast<size_t>(x[i].recv_count), ncclFloat64, x[i].peer,
                               comm, c->q[q]), "ncclRecv");
    c->stats.comm_bytes += 8 * (x[i].send_count + x[i].recv_count);
  }
  int rc2 = nccl_check(nc.group_end(), "ncclGroupEnd");
  return rc ? OOC_ERR_CUDA : rc2;
}

int ooc_reduce_allreduce(ooc_ctx* c, int q, int slot, int op) {
  OOC_ARG_CHECK(c && slot >= 0 && slot < OOC_REDUCE_SLOTS && q >= 0 && q < OOC_NUM_QUEUES,
                "ooc_reduce_allreduce: bad args");
  if (c->ipc) return ipc_allreduce(c, q, slot, op);
  OOC_ARG_CHECK(c->comm, "ooc_reduce_allreduce: no communicator (ooc_comm_init / ooc_comm_init_ipc)");
  const ncclRedOp_t rop = op == OOC_RED_MIN ? ncclMin : op == OOC_RED_MAX ? ncclMax : ncclSum;
  return nccl_check(nccl().all_reduce(c->red_acc + slot, c->red_acc + slot, 1, ncclFloat64, rop,
                                      static_cast<ncclComm_t>(c->comm), c->q[q]),
                    "ncclAllReduce");
}

void ooc_comm_release(ooc_ctx* c) {
  if (c && c->comm && nccl().ok) nccl().comm_destroy(static_cast<ncclComm_t>(c->comm));
  if (c) c->comm = nullptr;
  if (c) ipc_close(c);
}

}  // extern "C"
