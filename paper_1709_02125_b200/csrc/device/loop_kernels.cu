// par_loop kernels for sm_100a: the loop-program interpreter (K0, also running
// fused groups of loops) and the reduction fold. Implements ooc_launch_loop /
// ooc_launch_group / ooc_fill_box / ooc_reduce_*.
//
// Semantics are those of the reference's apply_loop (proj/src/kernel_exec.cpp:133-198):
// every point evaluates its write tapes (and the reduction tape) on the values
// present before any of its own writes, then stores. Points are independent by
// construction (writes only at offset 0, validated by loop.cpp:32-105), so any
// thread order gives bit-identical buffers. Arithmetic is IEEE binary64 with FMA
// contraction disabled at compile time (--fmad=false) and std::min/std::max
// tie/NaN behaviour reproduced exactly: min(a,b) = (b<a)?b:a, max(a,b) = (a<b)?b:a.
//
// Design (B200, HBM-bound):
//  * The loop program lives in the kernel's parameter space (constant bank):
//    warp-uniform dispatch, no divergence.
//  * Every distinct (argument, offset) read of a loop is hoisted into a LOAD at
//    the top of the loop's program, so all of a point's HBM loads are in flight
//    together (memory-level parallelism = reads x points per thread). The host
//    resolves each instruction's stack slot, so every (opcode, slot) pair is its
//    own switch case with compile-time register indices: no local-memory stack.
//  * Each thread evaluates P points of one row, BLOCK apart: every warp-level
//    load is a fully coalesced 256-B access.
//  * A fused group runs several consecutive loops per point (ooc_launch_group);
//    RANGE instructions mask points outside a loop's own range, and reads of data
//    written earlier in the same launch use coherent loads. The host only fuses
//    loops whose cross-loop accesses are point-wise (same thread), so per-point
//    program order reproduces the sequential loop order exactly.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "internal.cuh"
#include "jit.cuh"

using namespace oocdev;

namespace {

constexpr int kBlock = 128;
constexpr int kMaxReads = 8;  // hoisted reads per loop (more: in-place READ instructions)

enum Kind : int {
  K_CONST = 0,
  K_READ,    // s[r] = ld.nc            (in-place read, no hoisting)
  K_READC,   // s[r] = ld (coherent)    (in-place read of data written earlier in the launch)
  K_ADD,
  K_SUB,
  K_MUL,
  K_DIV,
  K_MIN,
  K_MAX,
  K_LOAD,    // rd[j] = ld.nc
  K_LOADC,   // rd[j] = ld (coherent)
  K_OUT,     // out[w] = s[0]
  K_STORE,   // *dst_w = out[w] (active lanes)
  K_RED,     // rv = s[0]
  K_RANGE,   // act = point inside [lo, hi) of the current loop
  K_PUSHR0,  // s[r] = rd[0] ... K_PUSHR0 + 7: s[r] = rd[7]
};
__host__ __device__ constexpr int kcode(int kind, int slot) { return kind * 32 + slot; }

struct KIns {
  union {
    const double* ptr;  // READ / LOAD / STORE: address at the launch origin (+ offset)
    double value;       // CONST
    int lohi_a[2];      // RANGE: canonical-a bounds relative to the launch origin
  } u;
  union {
    long long sA;  // strides of canonical dims a, b in the argument's view
    int lohi_b[2];
  } x;
  union {
    long long sB;
    int lohi_c[2];
  } y;
  int code;
  int pad;
};
static_assert(sizeof(KIns) == 32, "KIns layout");

template <int CAP>
struct KParams {
  long long nA, nB, nC;  // canonical extents of the launch box; c is contiguous
  int ncode;
  int red_op;
  double* part;     // reduction block partials
  double* scratch;  // exact mode: one contribution per point of the launch box
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
__device__ __forceinline__ double ld_coherent(const double* p) {
  double v;
  asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

#define OOC_UNROLL _Pragma("unroll")

#define OOC_PUSHR(r, j)                                                                \
  case kcode(K_PUSHR0 + j, r):                                                         \
    if constexpr (r < S && j < R) {                                                    \
      OOC_UNROLL for (int k = 0; k < P; ++k) s[r][k] = rd[j][k];                       \
    }                                                                                  \
    break;

#define OOC_BINOP(KIND, r, EXPR)                                                       \
  case kcode(KIND, r):                                                                 \
    if constexpr (r + 1 < S) {                                                         \
      OOC_UNROLL for (int k = 0; k < P; ++k) {                                         \
        const double a_ = s[r][k], b_ = s[r + 1][k];                                   \
        s[r][k] = (EXPR);                                                              \
      }                                                                                \
    }                                                                                  \
    break;

// Per-(opcode, slot) cases; `r` is the slot pushed (const / read / pushr) or the
// result slot of a binary op (operands r, r+1).
#define OOC_SLOT_CASES(r)                                                              \
  case kcode(K_CONST, r):                                                              \
    if constexpr (r < S) {                                                             \
      OOC_UNROLL for (int k = 0; k < P; ++k) s[r][k] = ins.u.value;                    \
    }                                                                                  \
    break;                                                                             \
  case kcode(K_READ, r):                                                               \
    if constexpr (r < S) {                                                             \
      const double* a_ = ins.u.ptr + ia * ins.x.sA + ib * ins.y.sB + cx;               \
      OOC_UNROLL for (int k = 0; k < P; ++k) if (act[k]) s[r][k] = __ldg(a_ + k * kBlock); \
    }                                                                                  \
    break;                                                                             \
  case kcode(K_READC, r):                                                              \
    if constexpr (r < S) {                                                             \
      const double* a_ = ins.u.ptr + ia * ins.x.sA + ib * ins.y.sB + cx;               \
      OOC_UNROLL for (int k = 0; k < P; ++k) if (act[k]) s[r][k] =                     \
          ld_coherent(a_ + k * kBlock);                                                \
    }                                                                                  \
    break;                                                                             \
  OOC_BINOP(K_ADD, r, a_ + b_)                                                         \
  OOC_BINOP(K_SUB, r, a_ - b_)                                                         \
  OOC_BINOP(K_MUL, r, a_ * b_)                                                         \
  OOC_BINOP(K_DIV, r, a_ / b_)                                                         \
  OOC_BINOP(K_MIN, r, b_ < a_ ? b_ : a_)                                               \
  OOC_BINOP(K_MAX, r, a_ < b_ ? b_ : a_)                                               \
  OOC_PUSHR(r, 0)                                                                      \
  OOC_PUSHR(r, 1)                                                                      \
  OOC_PUSHR(r, 2)                                                                      \
  OOC_PUSHR(r, 3)                                                                      \
  OOC_PUSHR(r, 4)                                                                      \
  OOC_PUSHR(r, 5)                                                                      \
  OOC_PUSHR(r, 6)                                                                      \
  OOC_PUSHR(r, 7)

#define OOC_LOAD_CASES(j)                                                              \
  case kcode(K_LOAD, j):                                                               \
    if constexpr (j < R) {                                                             \
      const double* a_ = ins.u.ptr + ia * ins.x.sA + ib * ins.y.sB + cx;               \
      OOC_UNROLL for (int k = 0; k < P; ++k) if (act[k]) rd[j][k] = __ldg(a_ + k * kBlock); \
    }                                                                                  \
    break;                                                                             \
  case kcode(K_LOADC, j):                                                              \
    if constexpr (j < R) {                                                             \
      const double* a_ = ins.u.ptr + ia * ins.x.sA + ib * ins.y.sB + cx;               \
      OOC_UNROLL for (int k = 0; k < P; ++k) if (act[k]) rd[j][k] =                    \
          ld_coherent(a_ + k * kBlock);                                                \
    }                                                                                  \
    break;

#define OOC_OUT_CASES(w)                                                               \
  case kcode(K_OUT, w):                                                                \
    if constexpr (w < W) {                                                             \
      OOC_UNROLL for (int k = 0; k < P; ++k) out[w][k] = s[0][k];                      \
    }                                                                                  \
    break;                                                                             \
  case kcode(K_STORE, w):                                                              \
    if constexpr (w < W) {                                                             \
      double* q_ = const_cast<double*>(ins.u.ptr) + ia * ins.x.sA + ib * ins.y.sB + cx; \
      OOC_UNROLL for (int k = 0; k < P; ++k) if (act[k]) q_[k * kBlock] = out[w][k];   \
    }                                                                                  \
    break;

template <int CAP, int P, int S, int W, int R, bool RED>
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
      bool ok[P], act[P];
#pragma unroll
      for (int k = 0; k < P; ++k) act[k] = ok[k] = cx + k * kBlock < p.nC;
      double s[S][P];
      double rd[R > 0 ? R : 1][P];
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
          OOC_LOAD_CASES(0)
          OOC_LOAD_CASES(1)
          OOC_LOAD_CASES(2)
          OOC_LOAD_CASES(3)
          OOC_LOAD_CASES(4)
          OOC_LOAD_CASES(5)
          OOC_LOAD_CASES(6)
          OOC_LOAD_CASES(7)
          OOC_OUT_CASES(0)
          OOC_OUT_CASES(1)
          OOC_OUT_CASES(2)
          OOC_OUT_CASES(3)
          OOC_OUT_CASES(4)
          OOC_OUT_CASES(5)
          OOC_OUT_CASES(6)
          OOC_OUT_CASES(7)
          case kcode(K_RED, 0):
#pragma unroll
            for (int k = 0; k < P; ++k) rv[k] = s[0][k];
            break;
          case kcode(K_RANGE, 0): {
            const bool in_ab = ia >= ins.u.lohi_a[0] && ia < ins.u.lohi_a[1] &&
                               ib >= ins.x.lohi_b[0] && ib < ins.x.lohi_b[1];
#pragma unroll
            for (int k = 0; k < P; ++k) {
              const long long c = cx + k * kBlock;
              act[k] = ok[k] && in_ab && c >= ins.y.lohi_c[0] && c < ins.y.lohi_c[1];
            }
            break;
          }
          default:
            __trap();
        }
      }
      if constexpr (RED) {
        if (p.scratch) {
          // exact mode: the contribution of every point of the launch box in row-major
          // order, the identity where the point is outside the loop's range
          double* dst = p.scratch + row * p.nC + cx;
#pragma unroll
          for (int k = 0; k < P; ++k)
            if (ok[k]) dst[k * kBlock] = act[k] ? rv[k] : red_identity(p.red_op);
        } else {
#pragma unroll
          for (int k = 0; k < P; ++k)
            if (act[k]) acc = red_combine(p.red_op, acc, rv[k]);
        }
      }
    }
  }
  if constexpr (RED) {
    if (p.scratch) return;
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

// Exact mode: acc = fold of the per-point contributions in row-major order by one
// thread — the reference's sequential fold (kernel_exec.cpp:193-197), identity entries
// being exact no-ops. The dependent add chain is the bound: warps 1.. stage the next
// tile of contributions into shared memory (coalesced) while thread 0 folds the current
// one from shared memory, so the folding thread never waits on HBM latency.
constexpr int kSeqTile = 2048;
__global__ void __launch_bounds__(256) k_fold_seq(const double* __restrict__ v, long long n,
                                                  double* acc, int op) {
  __shared__ __align__(16) double buf[2][kSeqTile];
  const long long tiles = (n + kSeqTile - 1) / kSeqTile;
  auto stage = [&](long long t) {
    const long long base = t * kSeqTile;
    const int len = static_cast<int>(n - base < kSeqTile ? n - base : kSeqTile);
    double* dst = buf[t & 1];
    for (int i = threadIdx.x - 32; i < len; i += blockDim.x - 32) dst[i] = __ldg(v + base + i);
  };
  double a = 0.0;
  if (threadIdx.x == 0) a = *acc;
  if (threadIdx.x >= 32 && tiles > 0) stage(0);
  __syncthreads();
  for (long long t = 0; t < tiles; ++t) {
    if (threadIdx.x >= 32) {
      if (t + 1 < tiles) stage(t + 1);
    } else if (threadIdx.x == 0) {
      const long long base = t * kSeqTile;
      const int len = static_cast<int>(n - base < kSeqTile ? n - base : kSeqTile);
      const double* src = buf[t & 1];
      int i = 0;
      for (; i + 16 <= len; i += 16) {
        double x[16];
#pragma unroll
        for (int k = 0; k < 16; k += 2) {
          const double2 p = *reinterpret_cast<const double2*>(src + i + k);
          x[k] = p.x;
          x[k + 1] = p.y;
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) a = red_combine(op, a, x[k]);
      }
      for (; i < len; ++i) a = red_combine(op, a, src[i]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *acc = a;
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
Canon canon(int ndim) { return Canon{ndim >= 3 ? ndim - 3 : -1, ndim >= 2 ? ndim - 2 : -1, ndim - 1}; }

struct Shape {
  int max_slot = 0;  // stack depth
  int max_out = 0;   // writes of one loop
  int max_reads = 0; // hoisted reads of one loop
};

// Lower a group of loops (n == 1: a plain par_loop) into one kernel program.
template <int CAP>
int lower_group(const ooc_loop* Ls, int n, int read_cap, KParams<CAP>& kp, Shape& sh) {
  const Canon cn = canon(Ls[0].ndim);
  int64_t lo[3], hi[3];  // hull of the loops' ranges = the launch box
  for (int d = 0; d < 3; ++d) {
    lo[d] = Ls[0].lo[d];
    hi[d] = Ls[0].hi[d];
    for (int i = 1; i < n; ++i) {
      lo[d] = std::min(lo[d], Ls[i].lo[d]);
      hi[d] = std::max(hi[d], Ls[i].hi[d]);
    }
  }
  auto ext = [&](int d) { return d < 0 ? 1LL : static_cast<long long>(hi[d] - lo[d]); };
  kp.nA = ext(cn.A);
  kp.nB = ext(cn.B);
  kp.nC = ext(cn.C);
  kp.red_op = n == 1 ? Ls[0].reduce_op : OOC_RED_NONE;
  auto stride = [&](const ooc_view& v, int d) { return d < 0 ? 0LL : static_cast<long long>(v.stride[d]); };
  auto at_origin = [&](const ooc_view& v) {
    long long off = 0;
    for (int d = 0; d < 3; ++d) off += (lo[d] - v.lo[d]) * v.stride[d];
    return v.data + off;
  };
  int nc = 0;
  auto push = [&]() -> KIns* {
    if (nc >= CAP) return nullptr;
    KIns* k = &kp.code[nc++];
    std::memset(k, 0, sizeof *k);
    return k;
  };
  std::vector<const double*> written;  // data pointers written by earlier loops of the group
  sh = Shape{};
  for (int i = 0; i < n; ++i) {
    const ooc_loop& L = Ls[i];
    OOC_ARG_CHECK(L.ndim == Ls[0].ndim, "ooc_launch_group: mixed ranks");
    for (int a = 0; a < L.nargs; ++a)
      OOC_ARG_CHECK(L.args[a].stride[cn.C] == 1, "ooc_launch_loop: argument view not contiguous");
    auto coherent = [&](int arg) {
      return std::find(written.begin(), written.end(), L.args[arg].data) != written.end();
    };
    if (n > 1) {
      KIns* k = push();
      OOC_ARG_CHECK(k, "ooc_launch_loop: program too long");
      k->code = kcode(K_RANGE, 0);
      auto rel = [&](int d, int which) -> int {
        if (d < 0) return which == 0 ? 0 : 1;
        return static_cast<int>((which == 0 ? L.lo[d] : L.hi[d]) - lo[d]);
      };
      k->u.lohi_a[0] = rel(cn.A, 0);
      k->u.lohi_a[1] = rel(cn.A, 1);
      k->x.lohi_b[0] = rel(cn.B, 0);
      k->x.lohi_b[1] = rel(cn.B, 1);
      k->y.lohi_c[0] = rel(cn.C, 0);
      k->y.lohi_c[1] = rel(cn.C, 1);
    }
    // distinct reads of the loop (all tapes) -> hoisted LOADs
    struct Rd {
      int arg;
      int64_t off[3];
    };
    std::vector<Rd> reads;
    for (int t = 0; t < L.ntape; ++t)
      if (L.tape[t].op == OOC_OP_READ) {
        OOC_ARG_CHECK(L.tape[t].arg >= 0 && L.tape[t].arg < L.nargs, "ooc_launch_loop: bad read argument");
        bool seen = false;
        for (const Rd& r : reads)
          seen |= r.arg == L.tape[t].arg && r.off[0] == L.tape[t].offset[0] &&
                  r.off[1] == L.tape[t].offset[1] && r.off[2] == L.tape[t].offset[2];
        if (!seen) reads.push_back({L.tape[t].arg, {L.tape[t].offset[0], L.tape[t].offset[1], L.tape[t].offset[2]}});
      }
    const bool hoist = static_cast<int>(reads.size()) <= read_cap;
    auto read_ptr = [&](int arg, const int64_t* off) {
      const ooc_view& v = L.args[arg];
      long long delta = 0;
      for (int d = 0; d < 3; ++d) delta += off[d] * v.stride[d];
      return at_origin(v) + delta;
    };
    if (hoist) {
      sh.max_reads = std::max(sh.max_reads, static_cast<int>(reads.size()));
      for (std::size_t j = 0; j < reads.size(); ++j) {
        KIns* k = push();
        OOC_ARG_CHECK(k, "ooc_launch_loop: program too long");
        k->u.ptr = read_ptr(reads[j].arg, reads[j].off);
        k->x.sA = stride(L.args[reads[j].arg], cn.A);
        k->y.sB = stride(L.args[reads[j].arg], cn.B);
        k->code = kcode(coherent(reads[j].arg) ? K_LOADC : K_LOAD, static_cast<int>(j));
      }
    }
    auto read_slot = [&](const ooc_ins& in) {
      for (std::size_t j = 0; j < reads.size(); ++j)
        if (reads[j].arg == in.arg && reads[j].off[0] == in.offset[0] &&
            reads[j].off[1] == in.offset[1] && reads[j].off[2] == in.offset[2])
          return static_cast<int>(j);
      return -1;
    };
    int sp = 0;
    auto emit_tape = [&](const ooc_ins* t, int len) -> int {
      for (int q = 0; q < len; ++q) {
        KIns* k = push();
        OOC_ARG_CHECK(k, "ooc_launch_loop: program too long");
        switch (t[q].op) {
          case OOC_OP_CONST:
            k->u.value = t[q].value;
            k->code = kcode(K_CONST, sp);
            sh.max_slot = std::max(sh.max_slot, ++sp);
            break;
          case OOC_OP_READ:
            if (hoist) {
              k->code = kcode(K_PUSHR0 + read_slot(t[q]), sp);
            } else {
              k->u.ptr = read_ptr(t[q].arg, t[q].offset);
              k->x.sA = stride(L.args[t[q].arg], cn.A);
              k->y.sB = stride(L.args[t[q].arg], cn.B);
              k->code = kcode(coherent(t[q].arg) ? K_READC : K_READ, sp);
            }
            sh.max_slot = std::max(sh.max_slot, ++sp);
            break;
          case OOC_OP_ADD:
          case OOC_OP_SUB:
          case OOC_OP_MUL:
          case OOC_OP_DIV:
          case OOC_OP_MIN:
          case OOC_OP_MAX: {
            OOC_ARG_CHECK(sp >= 2, "ooc_launch_loop: malformed tape (stack underflow)");
            static const int kind[] = {K_ADD, K_SUB, K_MUL, K_DIV, K_MIN, K_MAX};
            k->code = kcode(kind[t[q].op - OOC_OP_ADD], sp - 2);
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
      KIns* o = push();
      OOC_ARG_CHECK(o, "ooc_launch_loop: program too long");
      o->code = kcode(K_OUT, w);
    }
    sh.max_out = std::max(sh.max_out, static_cast<int>(L.nwrites));
    if (L.reduce_op != OOC_RED_NONE) {
      OOC_ARG_CHECK(n == 1, "ooc_launch_group: reducing loops are launched alone");
      sp = 0;
      int rc = emit_tape(t, L.reduce_len);
      if (rc) return rc;
      OOC_ARG_CHECK(sp == 1, "ooc_launch_loop: malformed reduction tape");
      KIns* o = push();
      OOC_ARG_CHECK(o, "ooc_launch_loop: program too long");
      o->code = kcode(K_RED, 0);
    }
    // stores after every tape of the loop (writes land after all reads)
    for (int w = 0; w < L.nwrites; ++w) {
      const ooc_view& v = L.args[L.write_arg[w]];
      KIns* k = push();
      OOC_ARG_CHECK(k, "ooc_launch_loop: program too long");
      k->u.ptr = at_origin(v);
      k->x.sA = stride(v, cn.A);
      k->y.sB = stride(v, cn.B);
      k->code = kcode(K_STORE, w);
      written.push_back(v.data);
    }
  }
  kp.ncode = nc;
  return OOC_OK;
}

template <int CAP, int P, int S, int W, int R>
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
  if (red && c->red_exact) {
    const long long pts = rows * kp.nC;
    if (pts > c->red_scratch_elems[q]) {
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      OOC_CUDA_TRY(cudaStreamIsCapturing(st, &cs));
      if (cs != cudaStreamCaptureStatusNone) {
        set_error("exact reductions: the contribution buffer cannot grow inside a graph capture");
        return OOC_ERR_ARG;
      }
      OOC_CUDA_TRY(cudaStreamSynchronize(st));
      OOC_CUDA_TRY(cudaFree(c->red_scratch[q]));
      c->red_scratch[q] = nullptr;
      c->red_scratch_elems[q] = 0;
      OOC_CUDA_TRY(cudaMalloc(&c->red_scratch[q], pts * sizeof(double)));
      c->red_scratch_elems[q] = pts;
    }
    grid.x = static_cast<unsigned>(std::min<long long>(xblocks, 1 << 20));
    grid.y = static_cast<unsigned>(std::min<long long>(rows, 65535));
    KParams<CAP> kr = kp;
    kr.scratch = c->red_scratch[q];
    k_interp<CAP, P, S, W, R, true><<<grid, kBlock, 0, st>>>(kr);
    OOC_CUDA_TRY(cudaGetLastError());
    return 0;  // no block partials: the caller folds the contributions
  }
  if (red) {
    KParams<CAP> kr = kp;
    kr.part = c->red_part[q];
    k_interp<CAP, P, S, W, R, true><<<grid, kBlock, 0, st>>>(kr);
  } else {
    k_interp<CAP, P, S, W, R, false><<<grid, kBlock, 0, st>>>(kp);
  }
  OOC_CUDA_TRY(cudaGetLastError());
  return static_cast<int>(grid.x * grid.y);
}

template <int CAP>
int launch_cap(ooc_ctx* c, int q, const ooc_loop* Ls, int n) {
  auto* kp = new KParams<CAP>();  // large struct: keep it off the host stack
  Shape sh;
  int rc = lower_group<CAP>(Ls, n, kMaxReads, *kp, sh);
  if (rc) {
    delete kp;
    return rc;
  }
  const bool red = kp->red_op != OOC_RED_NONE;
  // register-shape variants (P points/thread, S stack slots, W outputs, R hoisted
  // reads); OOC_KVARIANT forces one for experiments when the loop fits it
  static const char* force = std::getenv("OOC_KVARIANT");
  const char v = force && *force ? *force : 0;
  const bool fitsA = sh.max_slot <= 4 && sh.max_out <= 1 && sh.max_reads <= 4;
  const bool fitsB = sh.max_slot <= 8 && sh.max_out <= 2 && sh.max_reads <= 8;
  int blocks;
  if (v == 'E' && fitsA)
    blocks = launch_variant<CAP, 2, 4, 1, 4>(c, q, *kp, red);
  else if (v == 'F' && fitsA)
    blocks = launch_variant<CAP, 8, 4, 1, 4>(c, q, *kp, red);
  else if (v == 'D' && fitsA)
    blocks = launch_variant<CAP, 4, 4, 1, 8>(c, q, *kp, red);
  else if (v == 'C')
    blocks = launch_variant<CAP, 1, 32, OOC_MAX_WRITES, kMaxReads>(c, q, *kp, red);
  else if (v != 'B' && fitsA)
    blocks = launch_variant<CAP, 4, 4, 1, 4>(c, q, *kp, red);
  else if (fitsB)
    blocks = launch_variant<CAP, 2, 8, 2, kMaxReads>(c, q, *kp, red);
  else
    blocks = launch_variant<CAP, 1, 32, OOC_MAX_WRITES, kMaxReads>(c, q, *kp, red);
  const int red_op = kp->red_op;
  const long long pts = kp->nA * kp->nB * kp->nC;
  delete kp;
  if (blocks < 0) return blocks;
  if (red && c->red_exact) {
    k_fold_seq<<<1, 256, 0, c->q[q]>>>(c->red_scratch[q], pts, c->red_acc + Ls[0].reduce_slot, red_op);
    OOC_CUDA_TRY(cudaGetLastError());
    ++c->stats.kernel_launches;
  } else if (red) {
    k_fold<<<1, 1024, 0, c->q[q]>>>(c->red_part[q], blocks, c->red_acc + Ls[0].reduce_slot, red_op);
    OOC_CUDA_TRY(cudaGetLastError());
    ++c->stats.kernel_launches;
  }
  ++c->stats.kernel_launches;
  ++c->stats.interp_launches;
  if (n > 1) ++c->stats.special_launches;
  return OOC_OK;
}

int check_loop(const ooc_loop* L) {
  OOC_ARG_CHECK(L->ndim >= 1 && L->ndim <= 3, "ooc_launch_loop: bad rank");
  OOC_ARG_CHECK(L->nargs >= 0 && L->nargs <= OOC_MAX_ARGS, "ooc_launch_loop: too many args");
  OOC_ARG_CHECK(L->nwrites >= 0 && L->nwrites <= OOC_MAX_WRITES, "ooc_launch_loop: too many writes");
  OOC_ARG_CHECK(L->reduce_op == OOC_RED_NONE ||
                    (L->reduce_slot >= 0 && L->reduce_slot < OOC_REDUCE_SLOTS),
                "ooc_launch_loop: bad reduction slot");
  return OOC_OK;
}

bool loop_empty(const ooc_loop* L) {
  for (int d = 0; d < 3; ++d)
    if (L->hi[d] <= L->lo[d]) return true;
  return L->nwrites == 0 && L->reduce_op == OOC_RED_NONE;
}

}  // namespace

extern "C" {

int ooc_launch_group(ooc_ctx* c, int q, const ooc_loop* loops, int n) {
  OOC_ARG_CHECK(c && loops && n >= 1 && q >= 0 && q < OOC_NUM_QUEUES, "ooc_launch_group: bad args");
  std::vector<ooc_loop> live;
  int total = 0;
  for (int i = 0; i < n; ++i) {
    int rc = check_loop(&loops[i]);
    if (rc) return rc;
    if (loop_empty(&loops[i])) continue;
    live.push_back(loops[i]);
    // program size: range + reads + tape + out + stores (+ red)
    total += 1 + 2 * loops[i].ntape + 2 * loops[i].nwrites + 1;
  }
  if (live.empty()) return OOC_OK;
  if (c->red_exact && live.back().reduce_op != OOC_RED_NONE) {
    // exact reductions: the loops run one by one (the sequential semantics every fused
    // launch reproduces) and the reducing one through the interpreter's contribution path
    if (live.size() > 1) {
      for (const ooc_loop& L : live) {
        int rc = ooc_launch_group(c, q, &L, 1);
        if (rc) return rc;
      }
      return OOC_OK;
    }
    return launch_cap<1000>(c, q, live.data(), 1);
  }
  int blocks = 0;
  int jr = oocdev::jit_launch_group(c, q, live.data(), static_cast<int>(live.size()), &blocks);
  if (jr < 0) return jr;
  if (jr == OOC_OK) {
    if (live.size() == 1 && live[0].reduce_op != OOC_RED_NONE) {
      k_fold<<<1, 1024, 0, c->q[q]>>>(c->red_part[q], blocks, c->red_acc + live[0].reduce_slot,
                                      live[0].reduce_op);
      OOC_CUDA_TRY(cudaGetLastError());
      ++c->stats.kernel_launches;
    }
    ++c->stats.kernel_launches;
    if (live.size() > 1) ++c->stats.special_launches;
    return OOC_OK;
  }
  // The interpreter forwards values only at the point itself: a group that relies on
  // row recompute (a neighbour read of a value written earlier in the group) runs
  // loop by loop — the sequential semantics the fused launch reproduces.
  for (std::size_t j = 1; j < live.size(); ++j)
    for (int t = 0; t < live[j].ntape; ++t) {
      const ooc_ins& in = live[j].tape[t];
      if (in.op != OOC_OP_READ || (in.offset[0] == 0 && in.offset[1] == 0 && in.offset[2] == 0)) continue;
      const double* d = live[j].args[in.arg].data;
      for (std::size_t i = 0; i < j; ++i)
        for (int w = 0; w < live[i].nwrites; ++w)
          if (live[i].args[live[i].write_arg[w]].data == d) {
            for (const ooc_loop& L : live) {
              int rc = ooc_launch_group(c, q, &L, 1);
              if (rc) return rc;
            }
            return OOC_OK;
          }
    }
  if (total <= 64) return launch_cap<64>(c, q, live.data(), static_cast<int>(live.size()));
  OOC_ARG_CHECK(total <= 1000, "ooc_launch_group: program too long");
  return launch_cap<1000>(c, q, live.data(), static_cast<int>(live.size()));
}

int ooc_launch_loop(ooc_ctx* c, int q, const ooc_loop* L) {
  OOC_ARG_CHECK(c && L, "ooc_launch_loop: bad args");
  return ooc_launch_group(c, q, L, 1);
}

int ooc_set_reduce_exact(ooc_ctx* c, int on) {
  OOC_ARG_CHECK(c, "ooc_set_reduce_exact: null ctx");
  c->red_exact = on ? 1 : 0;
  return OOC_OK;
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


namespace oocdev {
int launch_fold(ooc_ctx* c, int q, int blocks, int slot, int op) {
  k_fold<<<1, 1024, 0, c->q[q]>>>(c->red_part[q], blocks, c->red_acc + slot, op);
  OOC_CUDA_TRY(cudaGetLastError());
  ++c->stats.kernel_launches;
  return OOC_OK;
}
}  // namespace oocdev
