// par_loop kernels for sm_100a: the generic tape interpreter (K0) and the
// reduction fold. Implements ooc_launch_loop / ooc_fill_box / ooc_reduce_*.
//
// Semantics are those of the reference's apply_loop (proj/src/kernel_exec.cpp:133-198):
// every point evaluates its write tapes (and the reduction tape) on the values
// present before any of its own writes, then stores. Points are independent by
// construction (writes only at offset 0, validated by loop.cpp:32-105), so any
// thread order gives bit-identical buffers. Arithmetic is IEEE binary64 with FMA
// contraction disabled at compile time (--fmad=false) and std::min/std::max
// tie/NaN behaviour reproduced exactly: min(a,b) = (b<a)?b:a, max(a,b) = (a<b)?b:a.
//
// Design (B200): the tape lives in the kernel's parameter space (constant bank,
// warp-uniform dispatch, no divergence). The evaluation stack is a register
// array: the host resolves, for every instruction, the stack slot it touches,
// so each (opcode, slot) pair is its own switch case with compile-time register
// indices — no local-memory stack. Each thread evaluates P points of one row,
// BLOCK apart, so every load instruction of a warp is a fully coalesced 256-B
// access and P independent loads are in flight per thread.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "internal.cuh"

using namespace oocdev;

namespace {

constexpr int kBlock = 128;

enum Kind : int { K_CONST = 0, K_READ, K_ADD, K_SUB, K_MUL, K_DIV, K_MIN, K_MAX, K_OUT, K_RED };
__host__ __device__ constexpr int kcode(int kind, int slot) { return kind * 32 + slot; }

struct KIns {
  union {
    const double* ptr;  // K_READ: address of (range.lo + offset) in the argument's view
    double value;       // K_CONST
  } u;
  long long sA, sB;     // K_READ: strides of canonical dims a, b in the argument's view
  int code;
  int pad;
};

template <int CAP>
struct KParams {
  long long nA, nB, nC;  // canonical extents; c is contiguous
  int ncode;
  int nwrites;
  int red_op;
  int pad;
  double* part;  // reduction block partials
  double* wptr[OOC_MAX_WRITES];
  long long wsA[OOC_MAX_WRITES], wsB[OOC_MAX_WRITES];
  KIns code[CAP];
};

__device__ __forceinline__ double red_identity(int op) {
  return op == OOC_RED_MIN ? INFINITY : op == OOC_RED_MAX ? -INFINITY : 0.0;
}
__device__ __forceinline__ double red_combine(int op, double acc, double v) {
  if (op == OOC_RED_SUM) return acc + v;
  if (op == OOC_RED_MIN) return v < acc ? v : acc;
  return acc < v ? v : acc;
}

// Per-(opcode, slot) cases; `r` is the slot pushed (const/read) or the result
// slot of a binary op (operands r, r+1).
#define OOC_SLOT_CASES(r)                                                              \
  case kcode(K_CONST, r):                                                              \
    if constexpr (r < S) {                                                             \
      _Pragma("unroll") for (int k = 0; k < P; ++k) s[r][k] = ins.u.value;             \
    }                                                                                  \
    break;                                                                             \
  case kcode(K_READ, r):                                                               \
    if constexpr (r < S) {                                                             \
      const double* a_ = ins.u.ptr + ia * ins.sA + ib * ins.sB + cx;                   \
      _Pragma("unroll") for (int k = 0; k < P; ++k) if (ok[k]) s[r][k] =               \
          __ldg(a_ + k * kBlock);                                                      \
    }                                                                                  \
    break;                                                                             \
  case kcode(K_ADD, r):                                                                \
    if constexpr (r + 1 < S) {                                                         \
      _Pragma("unroll") for (int k = 0; k < P; ++k) s[r][k] = s[r][k] + s[r + 1][k];   \
    }                                                                                  \
    break;                                                                             \
  case kcode(K_SUB, r):                                                                \
    if constexpr (r + 1 < S) {                                                         \
      _Pragma("unroll") for (int k = 0; k < P; ++k) s[r][k] = s[r][k] - s[r + 1][k];   \
    }                                                                                  \
    break;                                                                             \
  case kcode(K_MUL, r):                                                                \
    if constexpr (r + 1 < S) {                                                         \
      _Pragma("unroll") for (int k = 0; k < P; ++k) s[r][k] = s[r][k] * s[r + 1][k];   \
    }                                                                                  \
    break;                                                                             \
  case kcode(K_DIV, r):                                                                \
    if constexpr (r + 1 < S) {                                                         \
      _Pragma("unroll") for (int k = 0; k < P; ++k) s[r][k] = s[r][k] / s[r + 1][k];   \
    }                                                                                  \
    break;                                                                             \
  case kcode(K_MIN, r):                                                                \
    if constexpr (r + 1 < S) {                                                         \
      _Pragma("unroll") for (int k = 0; k < P; ++k) s[r][k] =                          \
          s[r + 1][k] < s[r][k] ? s[r + 1][k] : s[r][k];                               \
    }                                                                                  \
    break;                                                                             \
  case kcode(K_MAX, r):                                                                \
    if constexpr (r + 1 < S) {                                                         \
      _Pragma("unroll") for (int k = 0; k < P; ++k) s[r][k] =                          \
          s[r][k] < s[r + 1][k] ? s[r + 1][k] : s[r][k];                               \
    }                                                                                  \
    break;

#define OOC_OUT_CASE(w)                                                                \
  case kcode(K_OUT, w):                                                                \
    if constexpr (w < W) {                                                             \
      _Pragma("unroll") for (int k = 0; k < P; ++k) out[w][k] = s[0][k];               \
    }                                                                                  \
    break;

template <int CAP, int P, int S, int W, bool RED>
__global__ void __launch_bounds__(kBlock) k_interp(const __grid_constant__ KParams<CAP> p) {
  const long long rows = p.nA * p.nB;
  const long long xblocks = (p.nC + kBlock * P - 1) / (kBlock * P);
  double acc = 0.0;
  if constexpr (RED) acc = red_identity(p.red_op);
  for (long long row = blockIdx.y; row < rows; row += gridDim.y) {
    const long long ia = row / p.nB;
    const long long ib = row - ia * p.nB;
    for (long long xb = blockIdx.x; xb < xblocks; xb += gridDim.x) {
      const long long cx = xb * (kBlock * P) + threadIdx.x;
      bool ok[P];
#pragma unroll
      for (int k = 0; k < P; ++k) ok[k] = cx + k * kBlock < p.nC;
      double s[S][P];
      double out[W][P];
      double rv[P];
      for (int pc = 0; pc < p.ncode; ++pc) {
        const KIns& ins = p.code[pc];
        switch (ins.code) {
          OOC_SLOT_CASES(0)
          OOC_SLOT_CASES(1)
          OOC_SLOT_CASES(2)
          OOC_SLOT_CASES(3)
          OOC_SLOT_CASES(4)
          OOC_SLOT_CASES(5)
          OOC_SLOT_CASES(6)
          OOC_SLOT_CASES(7)
          OOC_SLOT_CASES(8)
          OOC_SLOT_CASES(9)
          OOC_SLOT_CASES(10)
          OOC_SLOT_CASES(11)
          OOC_SLOT_CASES(12)
          OOC_SLOT_CASES(13)
          OOC_SLOT_CASES(14)
          OOC_SLOT_CASES(15)
          OOC_SLOT_CASES(16)
          OOC_SLOT_CASES(17)
          OOC_SLOT_CASES(18)
          OOC_SLOT_CASES(19)
          OOC_SLOT_CASES(20)
          OOC_SLOT_CASES(21)
          OOC_SLOT_CASES(22)
          OOC_SLOT_CASES(23)
          OOC_SLOT_CASES(24)
          OOC_SLOT_CASES(25)
          OOC_SLOT_CASES(26)
          OOC_SLOT_CASES(27)
          OOC_SLOT_CASES(28)
          OOC_SLOT_CASES(29)
          OOC_SLOT_CASES(30)
          OOC_SLOT_CASES(31)
          OOC_OUT_CASE(0)
          OOC_OUT_CASE(1)
          OOC_OUT_CASE(2)
          OOC_OUT_CASE(3)
          OOC_OUT_CASE(4)
          OOC_OUT_CASE(5)
          OOC_OUT_CASE(6)
          OOC_OUT_CASE(7)
          case kcode(K_RED, 0):
#pragma unroll
            for (int k = 0; k < P; ++k) rv[k] = s[0][k];
            break;
          default:
            __trap();
        }
      }
      // all tapes evaluated: the point's writes land now (kernel_exec.cpp:173-179)
#pragma unroll
      for (int w = 0; w < W; ++w) {
        if (w < p.nwrites) {
          double* q = p.wptr[w] + ia * p.wsA[w] + ib * p.wsB[w] + cx;
#pragma unroll
          for (int k = 0; k < P; ++k)
            if (ok[k]) q[k * kBlock] = out[w][k];
        }
      }
      if constexpr (RED) {
#pragma unroll
        for (int k = 0; k < P; ++k)
          if (ok[k]) acc = red_combine(p.red_op, acc, rv[k]);
      }
    }
  }
  if constexpr (RED) {
    // warp shuffle, then across the block's 4 warps, in a fixed order
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = red_combine(p.red_op, acc, __shfl_down_sync(~0u, acc, o));
    __shared__ double warp_part[kBlock / 32];
    if ((threadIdx.x & 31) == 0) warp_part[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = warp_part[0];
      for (int i = 1; i < kBlock / 32; ++i) b = red_combine(p.red_op, b, warp_part[i]);
      p.part[blockIdx.y * gridDim.x + blockIdx.x] = b;
    }
  }
}

// Fold block partials in a fixed order and combine into the chain accumulator:
// acc = combine(acc, fold(partials)). Launched on the same queue, so tiles fold
// in tile order like the reference's red_acc (explicit_exec.cpp:159-162).
__global__ void __launch_bounds__(1024) k_fold(const double* part, int n, double* acc, int op) {
  __shared__ double sm[1024];
  double v = red_identity(op);
  for (int i = threadIdx.x; i < n; i += blockDim.x) v = red_combine(op, v, part[i]);
  sm[threadIdx.x] = v;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sm[threadIdx.x] = red_combine(op, sm[threadIdx.x], sm[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *acc = red_combine(op, *acc, sm[0]);
}

__global__ void k_set(double* dst, double v) { *dst = v; }

__global__ void k_fill(double* base, long long nA, long long nB, long long nC, long long sA,
                       long long sB, double v) {
  const long long total = nA * nB * nC;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    long long c = i % nC;
    long long r = i / nC;
    long long b = r % nB;
    long long a = r / nB;
    base[a * sA + b * sB + c] = v;
  }
}

// ------------------------------------------------------------ host-side lowering

struct Canon {
  int A, B, C;  // canonical dims (−1 when absent)
};
Canon canon(int ndim) {
  return Canon{ndim >= 3 ? ndim - 3 : -1, ndim >= 2 ? ndim - 2 : -1, ndim - 1};
}

template <int CAP>
int lower(const ooc_loop& L, KParams<CAP>& kp, int& max_slot) {
  const Canon cn = canon(L.ndim);
  auto ext = [&](int d) { return d < 0 ? 1LL : static_cast<long long>(L.hi[d] - L.lo[d]); };
  kp.nA = ext(cn.A);
  kp.nB = ext(cn.B);
  kp.nC = ext(cn.C);
  kp.nwrites = L.nwrites;
  kp.red_op = L.reduce_op;
  auto stride = [&](const ooc_view& v, int d) { return d < 0 ? 0LL : static_cast<long long>(v.stride[d]); };
  auto at_lo = [&](const ooc_view& v) {
    long long off = 0;
    for (int d = 0; d < 3; ++d) off += (L.lo[d] - v.lo[d]) * v.stride[d];
    return v.data + off;
  };
  for (int a = 0; a < L.nargs; ++a) {
    OOC_ARG_CHECK(L.args[a].stride[cn.C] == 1, "ooc_launch_loop: argument view not contiguous");
  }
  for (int w = 0; w < L.nwrites; ++w) {
    const ooc_view& v = L.args[L.write_arg[w]];
    kp.wptr[w] = at_lo(v);
    kp.wsA[w] = stride(v, cn.A);
    kp.wsB[w] = stride(v, cn.B);
  }
  int n = 0, sp = 0;
  max_slot = 0;
  auto emit_tape = [&](const ooc_ins* t, int len) -> int {
    for (int i = 0; i < len; ++i) {
      OOC_ARG_CHECK(n < CAP, "ooc_launch_loop: tape too long");
      KIns& k = kp.code[n++];
      k.sA = k.sB = 0;
      k.pad = 0;
      switch (t[i].op) {
        case OOC_OP_CONST:
          k.u.value = t[i].value;
          k.code = kcode(K_CONST, sp);
          max_slot = std::max(max_slot, sp + 1);
          ++sp;
          break;
        case OOC_OP_READ: {
          OOC_ARG_CHECK(t[i].arg >= 0 && t[i].arg < L.nargs, "ooc_launch_loop: bad read argument");
          const ooc_view& v = L.args[t[i].arg];
          long long delta = 0;
          for (int d = 0; d < 3; ++d) delta += t[i].offset[d] * v.stride[d];
          k.u.ptr = at_lo(v) + delta;
          k.sA = stride(v, cn.A);
          k.sB = stride(v, cn.B);
          k.code = kcode(K_READ, sp);
          max_slot = std::max(max_slot, sp + 1);
          ++sp;
          break;
        }
        case OOC_OP_ADD:
        case OOC_OP_SUB:
        case OOC_OP_MUL:
        case OOC_OP_DIV:
        case OOC_OP_MIN:
        case OOC_OP_MAX: {
          OOC_ARG_CHECK(sp >= 2, "ooc_launch_loop: malformed tape (stack underflow)");
          static const int kind[] = {K_ADD, K_SUB, K_MUL, K_DIV, K_MIN, K_MAX};
          k.u.value = 0.0;
          k.code = kcode(kind[t[i].op - OOC_OP_ADD], sp - 2);
          --sp;
          break;
        }
        default:
          OOC_ARG_CHECK(false, "ooc_launch_loop: unsupported opcode (coord outside fills?)");
      }
    }
    return OOC_OK;
  };
  const ooc_ins* t = L.tape;
  for (int w = 0; w < L.nwrites; ++w) {
    sp = 0;
    int rc = emit_tape(t, L.write_len[w]);
    if (rc) return rc;
    t += L.write_len[w];
    OOC_ARG_CHECK(sp == 1, "ooc_launch_loop: malformed write tape");
    OOC_ARG_CHECK(n < CAP, "ooc_launch_loop: tape too long");
    KIns& o = kp.code[n++];
    o = KIns{};
    o.code = kcode(K_OUT, w);
  }
  if (L.reduce_op != OOC_RED_NONE) {
    sp = 0;
    int rc = emit_tape(t, L.reduce_len);
    if (rc) return rc;
    OOC_ARG_CHECK(sp == 1, "ooc_launch_loop: malformed reduction tape");
    OOC_ARG_CHECK(n < CAP, "ooc_launch_loop: tape too long");
    KIns& o = kp.code[n++];
    o = KIns{};
    o.code = kcode(K_RED, 0);
  }
  kp.ncode = n;
  return OOC_OK;
}

template <int CAP, int P, int S, int W>
int launch_variant(ooc_ctx* c, int q, const KParams<CAP>& kp, bool red) {
  const long long rows = kp.nA * kp.nB;
  const long long xblocks = (kp.nC + kBlock * P - 1) / (kBlock * P);
  dim3 grid;
  grid.x = static_cast<unsigned>(std::min<long long>(xblocks, 1 << 20));
  if (red) {
    grid.x = static_cast<unsigned>(std::min<long long>(xblocks, c->red_part_cap));
    long long gy = std::max<long long>(1, c->red_part_cap / grid.x);
    gy = std::min<long long>(gy, std::max<long long>(1, 4 * 148 * 8 / grid.x));
    grid.y = static_cast<unsigned>(std::min<long long>(rows, gy));
  } else {
    grid.y = static_cast<unsigned>(std::min<long long>(rows, 65535));
  }
  cudaStream_t st = c->q[q];
  if (red) {
    KParams<CAP> kr = kp;
    kr.part = c->red_part[q];
    k_interp<CAP, P, S, W, true><<<grid, kBlock, 0, st>>>(kr);
  } else {
    k_interp<CAP, P, S, W, false><<<grid, kBlock, 0, st>>>(kp);
  }
  OOC_CUDA_TRY(cudaGetLastError());
  return static_cast<int>(grid.x * grid.y);
}

template <int CAP>
int launch_cap(ooc_ctx* c, int q, const ooc_loop& L) {
  auto* kp = new KParams<CAP>();  // large struct: keep it off the host stack
  int max_slot = 0;
  int rc = lower<CAP>(L, *kp, max_slot);
  if (rc) {
    delete kp;
    return rc;
  }
  const bool red = L.reduce_op != OOC_RED_NONE;
  int blocks;
  if (max_slot <= 4 && L.nwrites <= 1)
    blocks = launch_variant<CAP, 4, 4, 1>(c, q, *kp, red);
  else if (max_slot <= 8 && L.nwrites <= 2)
    blocks = launch_variant<CAP, 2, 8, 2>(c, q, *kp, red);
  else
    blocks = launch_variant<CAP, 1, 32, OOC_MAX_WRITES>(c, q, *kp, red);
  delete kp;
  if (blocks < 0) return blocks;
  if (red) {
    k_fold<<<1, 1024, 0, c->q[q]>>>(c->red_part[q], blocks, c->red_acc + L.reduce_slot,
                                    L.reduce_op);
    OOC_CUDA_TRY(cudaGetLastError());
    ++c->stats.kernel_launches;
  }
  ++c->stats.kernel_launches;
  ++c->stats.interp_launches;
  return OOC_OK;
}

}  // namespace

extern "C" {

int ooc_launch_loop(ooc_ctx* c, int q, const ooc_loop* L) {
  OOC_ARG_CHECK(c && L && q >= 0 && q < OOC_NUM_QUEUES, "ooc_launch_loop: bad args");
  OOC_ARG_CHECK(L->ndim >= 1 && L->ndim <= 3, "ooc_launch_loop: bad rank");
  OOC_ARG_CHECK(L->nargs >= 0 && L->nargs <= OOC_MAX_ARGS, "ooc_launch_loop: too many args");
  OOC_ARG_CHECK(L->nwrites >= 0 && L->nwrites <= OOC_MAX_WRITES, "ooc_launch_loop: too many writes");
  OOC_ARG_CHECK(L->reduce_op == OOC_RED_NONE ||
                    (L->reduce_slot >= 0 && L->reduce_slot < OOC_REDUCE_SLOTS),
                "ooc_launch_loop: bad reduction slot");
  for (int d = 0; d < 3; ++d)
    if (L->hi[d] <= L->lo[d]) return OOC_OK;  // empty sub-range: nothing to do
  if (L->nwrites == 0 && L->reduce_op == OOC_RED_NONE) return OOC_OK;
  // total instructions incl. one OUT per write and one RED
  const int n = L->ntape + L->nwrites + (L->reduce_op != OOC_RED_NONE ? 1 : 0);
  if (n <= 64) return launch_cap<64>(c, q, *L);
  OOC_ARG_CHECK(n <= OOC_MAX_TAPE + OOC_MAX_WRITES + 1, "ooc_launch_loop: tape too long");
  return launch_cap<OOC_MAX_TAPE + 16>(c, q, *L);
}

int ooc_fill_box(ooc_ctx* c, int q, const ooc_view* v, double value) {
  OOC_ARG_CHECK(c && v && q >= 0 && q < OOC_NUM_QUEUES, "ooc_fill_box: bad args");
  long long n[3];
  for (int d = 0; d < 3; ++d) {
    n[d] = v->hi[d] - v->lo[d];
    if (n[d] <= 0) return OOC_OK;
  }
  const long long total = n[0] * n[1] * n[2];
  const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 148 * 16));
  k_fill<<<blocks, 256, 0, c->q[q]>>>(v->data, n[0], n[1], n[2], v->stride[0], v->stride[1], value);
  OOC_CUDA_TRY(cudaGetLastError());
  ++c->stats.kernel_launches;
  return OOC_OK;
}

int ooc_reduce_reset(ooc_ctx* c, int q, int slot, int op) {
  OOC_ARG_CHECK(c && slot >= 0 && slot < OOC_REDUCE_SLOTS && q >= 0 && q < OOC_NUM_QUEUES,
                "ooc_reduce_reset: bad args");
  double v = op == OOC_RED_MIN ? INFINITY : op == OOC_RED_MAX ? -INFINITY : 0.0;
  k_set<<<1, 1, 0, c->q[q]>>>(c->red_acc + slot, v);
  OOC_CUDA_TRY(cudaGetLastError());
  ++c->stats.kernel_launches;
  return OOC_OK;
}

int ooc_reduce_fetch(ooc_ctx* c, int q, int slot, double* dst) {
  OOC_ARG_CHECK(c && dst && slot >= 0 && slot < OOC_REDUCE_SLOTS && q >= 0 && q < OOC_NUM_QUEUES,
                "ooc_reduce_fetch: bad args");
  OOC_CUDA_TRY(cudaMemcpyAsync(dst, c->red_acc + slot, sizeof(double), cudaMemcpyDeviceToHost,
                               c->q[q]));
  return OOC_OK;
}

}  // extern "C"
