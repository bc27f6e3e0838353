// Internal state of the device layer (never exposed through include/ooc_device.h).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <string>
#include <unordered_map>

#include "ooc_device.h"

namespace oocdev {

void set_error(const std::string& msg);

#define OOC_CUDA_TRY(expr)                                                                  \
  do {                                                                                      \
    cudaError_t e_ = (expr);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      ::oocdev::set_error(std::string(#expr) + ": " + cudaGetErrorString(e_) + " (" +       \
                          __FILE__ + ":" + std::to_string(__LINE__) + ")");                 \
      return OOC_ERR_CUDA;                                                                  \
    }                                                                                       \
  } while (0)

#define OOC_ARG_CHECK(cond, msg)      \
  do {                                \
    if (!(cond)) {                    \
      ::oocdev::set_error(msg);       \
      return OOC_ERR_ARG;             \
    }                                 \
  } while (0)

}  // namespace oocdev

struct ooc_event {
  cudaEvent_t ev = nullptr;
};

struct ooc_ctx {
  int device = 0;
  cudaStream_t q[OOC_NUM_QUEUES] = {nullptr, nullptr, nullptr};
  cudaDeviceProp prop{};
  // device memory manager bookkeeping
  std::unordered_map<void*, size_t> allocs;
  long long in_use = 0, peak = 0;
  // reduction accumulators + per-queue block-partials scratch
  double* red_acc = nullptr;   // OOC_REDUCE_SLOTS
  double* red_part[OOC_NUM_QUEUES] = {nullptr, nullptr, nullptr};
  int red_part_cap = 0;
  // exact-reduction mode (ooc_set_reduce_exact): per-point contributions of a reducing
  // launch, folded by one thread in row-major order (the reference's sequential fold)
  int red_exact = 0;
  double* red_scratch[OOC_NUM_QUEUES] = {nullptr, nullptr, nullptr};
  long long red_scratch_elems[OOC_NUM_QUEUES] = {0, 0, 0};
  ooc_dev_stats stats{};
  // multi-GPU (comm.cu): NCCL communicator of the slab decomposition, or the CUDA-IPC
  // transport (shared-memory rendezvous + peer-mapped outboxes)
  void* comm = nullptr;
  void* ipc = nullptr;
  int rank = 0, world = 1;
  long long capture_launches0 = 0;  // kernel-launch count when a graph capture began
};
