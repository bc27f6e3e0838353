// Multi-GPU plumbing of the device layer: NCCL (opened lazily with dlopen) for the
// slab decomposition — grouped point-to-point ghost-band exchange between
// neighbouring ranks and all-reduce of reduction accumulators, both enqueued on a
// queue of the context so they order with the chain's kernels without host syncs.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

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

int ooc_comm_exchange(ooc_ctx* c, int q, const ooc_xfer* x, int n) {
  OOC_ARG_CHECK(c && (x || n == 0) && q >= 0 && q < OOC_NUM_QUEUES, "ooc_comm_exchange: bad args");
  OOC_ARG_CHECK(c->comm, "ooc_comm_exchange: no communicator (ooc_comm_init)");
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
  OOC_ARG_CHECK(c->comm, "ooc_reduce_allreduce: no communicator (ooc_comm_init)");
  const ncclRedOp_t rop = op == OOC_RED_MIN ? ncclMin : op == OOC_RED_MAX ? ncclMax : ncclSum;
  return nccl_check(nccl().all_reduce(c->red_acc + slot, c->red_acc + slot, 1, ncclFloat64, rop,
                                      static_cast<ncclComm_t>(c->comm), c->q[q]),
                    "ncclAllReduce");
}

void ooc_comm_release(ooc_ctx* c) {
  if (c && c->comm && nccl().ok) nccl().comm_destroy(static_cast<ncclComm_t>(c->comm));
  if (c) c->comm = nullptr;
}

}  // extern "C"
