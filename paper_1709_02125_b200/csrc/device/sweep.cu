// Row-sweep fusion: a whole run of 2-D par_loops — typically one or more complete
// timesteps of an app — executed by ONE kernel that streams the mesh through shared
// memory once.
//
// The register and TMA templates (jit.cu) fuse loops only while every value a point
// consumes is either in memory or produced at the same point (or recomputable along
// the row dimension); a read of an in-launch value at a column offset ends the group.
// miniflow2d's iteration therefore needs two launches and 22 arrays of DRAM traffic.
// The sweep kernel lifts that restriction the B200 way: each CTA owns a strip of
// TC columns and walks its rows top to bottom (a 2.5-D streaming sweep). Every dataset
// the group touches lives in a ring of W_d rows x 128 columns of shared memory; loop i
// runs `lag_i` rows behind the loads, so when it evaluates row r every value it reads —
// loaded from HBM, or produced by an earlier loop of the group at any (row, column)
// offset within the halo — is already in its ring. Per step a CTA:
//   1. waits for the cp.async loads of this step (issued P steps earlier) and syncs,
//   2. issues the loads of step s+P (8-byte cp.async, zero-filled outside the view),
//   3. evaluates the loops in order (one point per thread per loop; a barrier only
//      between loops that touch a common dataset),
//   4. stores the final rows of every written dataset to HBM (coalesced, 1 KB rows).
// DRAM traffic is one read of every input and one write of every output per group,
// however many loops and timesteps the group spans: miniflow2d goes from 22 arrays
// per iteration to 13 (one iteration per group) or fewer (several).
//
// Correctness constraints, all resolved at generation time from the loops' stencils:
//  * lags: RAW  lag_reader >= lag_writer + max row offset of the read;
//          WAR  lag_writer >= lag_reader - min row offset (the ring row is rewritten
//               only after every earlier loop has read the old value);
//          WAW  later writers never run ahead of earlier ones;
//  * column halos: loop j computes h_j extra columns each side, h_j >= h_k + |dc| for
//    every later loop k reading j's output at column offset dc, so a strip's owned
//    columns are exact (the halo is recomputed redundantly, never exchanged);
//  * warm-up rows: a CTA owning rows [r0, r1) starts its sweep `warm` rows earlier —
//    the depth of the dependency cone — and stores only its own rows;
//  * out-of-place outputs: a dataset the group both loads and writes is written to a
//    shadow buffer (the host engine flips the two after the launch), so a neighbouring
//    CTA's halo / warm-up rows always read the values from before the launch. Datasets
//    first written in the group (temporaries) are stored in place, only where a loop of
//    the group writes them.
// Arithmetic is the same tape order, IEEE binary64, --fmad=false, std::min/max
// semantics as every other kernel: results are bit-identical to the reference.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>
#include <mutex>
#include <sstream>
#include <string>
#include <unordered_map>
#include <vector>

#include "internal.cuh"
#include "jit.cuh"

using namespace oocdev;

#define SW_MAXL 48
#define SW_MAXD 16
#define SW_MAXC 384

namespace {

// ring row width in columns (TC owned + 2*HC halo) = threads per CTA; OOC_SWEEP_RC
int ring_cols() {
  static int rc = [] {
    const char* e = std::getenv("OOC_SWEEP_RC");
    const int v = e ? std::atoi(e) : 256;  // measured: 256 > 128 (+3 %) > 64
    return v == 64 || v == 128 || v == 256 || v == 512 ? v : 256;
  }();
  return rc;
}
// 3-D plane tiles: RB rows (dim 1) x RC columns; measured choices, OOC_SWEEP_RB / OOC_SWEEP_RC3
int ring_rows3() {
  static int rb = [] {
    const char* e = std::getenv("OOC_SWEEP_RB");
    const int v = e ? std::atoi(e) : 16;
    return v >= 4 && v <= 32 ? v : 16;
  }();
  return rb;
}
int ring_cols3() {
  static int rc = [] {
    const char* e = std::getenv("OOC_SWEEP_RC3");
    const int v = e ? std::atoi(e) : 32;
    return v == 32 || v == 64 ? v : 32;
  }();
  return rc;
}

// Parameter block; the kernel source declares an identical struct.
struct SweepParams {
  double* part;              // reduction: one partial per CTA
  long long R0, R1, C0, C1;  // launch box: rows (dim 0) [R0,R1) x columns (last dim) [C0,C1), absolute
  long long B0, B1;          // 3-D: launch box along dim 1 (2-D: [0,1))
  long long ntc;             // CTA tiles along the columns (blockIdx.x = tile_b * ntc + tile_c)
  long long seg_rows;        // rows owned per CTA row-segment
  long long edge_first;      // 1: the column-edge strips' CTAs dispatch first (see the prologue)
  unsigned long long* trace; // debug (OOC_SWEEP_TRACE): per CTA SM id, start, end
  long long rng[SW_MAXL][6];  // per loop: rows [0,1), columns [2,3), dim 1 [4,5), absolute
  const double* src[SW_MAXD];
  double* dst[SW_MAXD];
  long long s0[SW_MAXD];      // dim-0 stride (elements)
  long long s1[SW_MAXD];      // 3-D: dim-1 stride
  long long box[SW_MAXD][6];  // view box: rows [0,1), columns [2,3), dim 1 [4,5)
  double cst[SW_MAXC];
};

const char* kSweepDecl = R"CUDA(
struct SweepParams {
  double* part;
  long long R0, R1, C0, C1;
  long long B0, B1;
  long long ntc;
  long long seg_rows;
  long long edge_first;
  unsigned long long* trace;
  long long rng[SW_MAXL][6];
  const double* src[SW_MAXD];
  double* dst[SW_MAXD];
  long long s0[SW_MAXD];
  long long s1[SW_MAXD];
  long long box[SW_MAXD][6];
  double cst[SW_MAXC];
};
__device__ __forceinline__ double ooc_min(double a, double b) { return b < a ? b : a; }
__device__ __forceinline__ double ooc_max(double a, double b) { return a < b ? b : a; }
__device__ __forceinline__ double ooc_red(int op, double acc, double v) {
  if (op == 1) return acc + v;
  if (op == 2) return v < acc ? v : acc;
  return acc < v ? v : acc;
}
__device__ __forceinline__ long long sw_floordiv(long long a, long long k) {
  return a >= 0 ? a / k : -((-a + k - 1) / k);
}
// TMA (bulk async copy) loads: one thread arms an mbarrier with the step's byte count and
// issues one row copy per loaded dataset; every thread waits on the barrier's phase.
__device__ __forceinline__ unsigned sw_saddr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void sw_wait(unsigned bar, unsigned parity) {
  for (unsigned tries = 0;; ++tries) {
    unsigned done;
    asm volatile("{\n .reg .pred P1;\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
                 " selp.u32 %0, 1, 0, P1;\n}\n" : "=r"(done) : "r"(bar), "r"(parity) : "memory");
    if (done) return;
    if (tries > (1u << 28)) asm volatile("trap;");  // a byte count that never completes: a loud launch error, not a hang
  }
}
__device__ __forceinline__ void sw_bulk(unsigned dst, const double* src, unsigned bytes, unsigned bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
// 3-D: one tiled tensor copy per dataset and step — the whole RB x RCp plane tile, out-of-
// bounds elements zero-filled (innermost coordinate even: 16-byte aligned; negative is fine)
struct __align__(64) SwMaps { unsigned long long t[SW_MAXD][16]; };
__device__ __forceinline__ void sw_tensor3(unsigned dst, const void* map, int x, int y, int z, unsigned bar) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
               :: "r"(dst), "l"(map), "r"(x), "r"(y), "r"(z), "r"(bar) : "memory");
}
__device__ __forceinline__ int sw_slot(int x, int w) {  // x mod w, for rings of any length
  const int r = x % w;
  return r < 0 ? r + w : r;
}
__device__ __forceinline__ void sw_cp8(double* dst, const double* src, bool ok) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" :: "r"(s), "l"(src), "r"(ok ? 8 : 0) : "memory");
}
)CUDA";

struct Rd {
  long long omin = LLONG_MAX, omax = LLONG_MIN, oc = 0;  // row offsets range, max |column offset|
  long long ob = 0;                                      // 3-D: max |dim-1 offset|
};

struct SwLoop {
  long long lag = 0, h = 0, hb = 0;  // hb: 3-D halo along dim 1
  std::vector<int> wds;        // dataset of each write
  std::map<int, Rd> rd;        // dataset -> read offsets
  bool barrier = false;        // barrier before this loop (within a step)
};

struct SwDs {
  const ooc_view* v = nullptr;
  bool loaded = false, written = false, oop = false;
  bool store = false;  // written and still live after the group (not a dead store)
  long long lagL = 0, lagS = 0, W = 0, off = 0, need = 0;
  std::vector<int> writers;
};

struct SwPlan {
  int n = 0, K = 2, P = 2, NT = 256, RC = 128;
  int nd = 2;                      // 2: thread per ring column; 3: thread per (dim-1, column) of a plane tile
  int RB = 1;                      // 3-D: tile rows along dim 1 (ring "row" = RB x RCp plane tile)
  long long HB = 0, TB = 1;        // 3-D: dim-1 halo and owned tile rows
  long long pad = 32;              // doubles before/after the rings (edge neighbour reads)
  bool tma = false;  // loads: bulk async copies (one thread, mbarrier ring) instead of per-thread cp.async
  bool bulk_st = false;  // 2-D TMA: interior rows stored by the producer with bulk copies (smem -> global)
  bool trace = false;    // debug (OOC_SWEEP_TRACE=file): per-CTA SM id + start / end times
  long long U = 8;   // ring period: every ring length divides it (0: none small enough, no unrolling)
  int NB = 8;        // load barriers (a multiple of U's steps: constant indices in unrolled steps)
  int RCp = 128;     // ring row pitch in doubles (RC, or RC + 2 with TMA: even-column row copies)
  long long SP = 128;  // ring slot pitch in doubles: RB x RCp, 3-D rounded up to 128 bytes (tensor-copy destinations)
  long long HC = 0, TC = 0, warm = 0, lagS_max = 0, smem = 0;
  int red_op = OOC_RED_NONE;  // the run's last loop reduces (no writes): folded per CTA
  long long red_lag = 0;
  long long box[6] = {0, 0, 0, 0, 0, 1};  // launch box rows [0,1) / cols [2,3) / dim 1 [4,5)
  std::vector<SwLoop> L;
  std::vector<SwDs> D;
};

// 3-D plane-tile sweeps: on by default (measured 1.9x / 1.5x over the fused 3-D launches
// on miniflow3d / rk3chain3d, profiles/r02_summary.md); ooc_sweep_set_3d(0) / OOC_SWEEP_3D=0
// turns them off
int g_sweep3d = -1;
bool sweep_3d_enabled() {
  if (g_sweep3d < 0) g_sweep3d = std::getenv("OOC_SWEEP_3D") && std::atoi(std::getenv("OOC_SWEEP_3D")) == 0 ? 0 : 1;
  return g_sweep3d == 1;
}
long long smem_budget3() {  // 3-D rings of plane tiles: one CTA per SM
  static long long b = [] {
    // measured: 225 000 B lets rk3chain3d's 8-loop stage run fit one sweep (33.2 vs 36.2 ms
    // per ten 9-loop runs at 512^3), miniflow3d unchanged (profiles/r02_summary.md)
    const char* e = std::getenv("OOC_SWEEP_SMEM3");
    return e ? std::atoll(e) : 225000LL;
  }();
  return b;
}
long long smem_budget() {
  static long long b = [] {
    const char* e = std::getenv("OOC_SWEEP_SMEM");
    // measured: occupancy beats fewer DRAM passes (56 KB per 128 ring columns)
    return e ? std::atoll(e) : std::min<long long>(56LL * 1024 * ring_cols() / 128, 220LL * 1024);
  }();
  return b;
}

bool fail(std::string* why, const std::string& m) {
  if (why) *why = m;
  return false;
}

// Analyse a group for the sweep template with K rows per step (NT = 128*K threads)
// and a P-step load prefetch. Fills the plan (lags, halos, rings, barriers).
bool analyze(const ooc_loop* Ls, int n, int K, int P, SwPlan& pl, std::string* why,
             const std::vector<const double*>* dead = nullptr, bool tma = false) {
  pl = SwPlan{};
  pl.n = n;
  pl.K = K;
  pl.P = P;
  if (n < 1 || n > SW_MAXL) return fail(why, "group size");
  pl.nd = Ls[0].ndim;
  if (pl.nd != 2 && pl.nd != 3) return fail(why, "not 2-D / 3-D");
  if (pl.nd == 3 && !sweep_3d_enabled()) return fail(why, "3-D sweeps disabled (ooc_sweep_set_3d)");
  if (pl.nd == 3 && !tma) return fail(why, "3-D sweeps load with TMA only");
  pl.RC = pl.nd == 2 ? ring_cols() : ring_cols3();
  pl.RB = pl.nd == 2 ? 1 : ring_rows3();
  pl.NT = pl.RB * pl.RC;
  pl.tma = tma;
  // bulk-copy stores of the interior rows by the producer (OOC_SWEEP_BULKST=1): parity-
  // tested, measured no faster on the timestep runs (2.70 ms either way) and slower on the
  // chain's last run, which stores nine datasets (6.1 vs 5.1 ms): off by default
  static const bool bulk_env = std::getenv("OOC_SWEEP_BULKST") && std::atoi(std::getenv("OOC_SWEEP_BULKST")) == 1;
  pl.bulk_st = tma && pl.nd == 2 && bulk_env;
  static const bool trace_env = std::getenv("OOC_SWEEP_TRACE") != nullptr;
  pl.trace = trace_env;
  pl.RCp = tma ? pl.RC + 2 : pl.RC;
  if (tma) pl.NT += 32;  // + one producer warp issuing the bulk-copy loads
  pl.L.resize(static_cast<std::size_t>(n));
  int ncst = 0;
  auto ds_of = [&](const ooc_view& v) -> int {
    for (std::size_t d = 0; d < pl.D.size(); ++d) {
      const ooc_view& w = *pl.D[d].v;
      if (w.data != v.data) continue;
      for (int k = 0; k < 3; ++k)
        if (w.lo[k] != v.lo[k] || w.hi[k] != v.hi[k] || w.stride[k] != v.stride[k]) return -2;
      return static_cast<int>(d);
    }
    if (pl.nd == 2 && (v.stride[1] != 1 || v.lo[2] != 0 || v.hi[2] != 1)) return -2;
    if (pl.nd == 3 && v.stride[2] != 1) return -2;
    if (pl.D.size() >= SW_MAXD) return -3;
    SwDs D;
    D.v = &v;
    pl.D.push_back(D);
    return static_cast<int>(pl.D.size()) - 1;
  };
  long long tape_total = 0;
  for (int i = 0; i < n; ++i) {
    const ooc_loop& L = Ls[i];
    SwLoop& S = pl.L[static_cast<std::size_t>(i)];
    if (L.ndim != pl.nd) return fail(why, "mixed ranks");
    if (L.reduce_op != OOC_RED_NONE && (i != n - 1 || L.nwrites != 0 || n < 2))
      return fail(why, "reduction (only as the last, write-free loop of a run)");
    if (L.hi[0] <= L.lo[0] || L.hi[1] <= L.lo[1]) return fail(why, "range");
    if (pl.nd == 2 ? (L.lo[2] != 0 || L.hi[2] != 1) : L.hi[2] <= L.lo[2]) return fail(why, "range");
    tape_total += L.ntape;
    for (int t = 0; t < L.ntape; ++t) {
      const ooc_ins& in = L.tape[t];
      if (in.op == OOC_OP_CONST) {
        ++ncst;
      } else if (in.op == OOC_OP_READ) {
        if (in.arg < 0 || in.arg >= L.nargs) return fail(why, "bad arg");
        const int d = ds_of(L.args[in.arg]);
        if (d < 0) return fail(why, "dataset views differ / too many datasets");
        if ((pl.nd == 2 && in.offset[2] != 0) || std::llabs(in.offset[0]) > 8 || std::llabs(in.offset[1]) > 8 ||
            std::llabs(in.offset[2]) > 8)
          return fail(why, "offset");
        Rd& r = S.rd[d];
        r.omin = std::min<long long>(r.omin, in.offset[0]);
        r.omax = std::max<long long>(r.omax, in.offset[0]);
        r.oc = std::max<long long>(r.oc, std::llabs(in.offset[pl.nd - 1]));
        if (pl.nd == 3) r.ob = std::max<long long>(r.ob, std::llabs(in.offset[1]));
      } else if (in.op < OOC_OP_ADD || in.op > OOC_OP_MAX) {
        return fail(why, "opcode");
      }
    }
    for (int w = 0; w < L.nwrites; ++w) {
      const int d = ds_of(L.args[L.write_arg[w]]);
      if (d < 0) return fail(why, "dataset views differ / too many datasets");
      S.wds.push_back(d);
      auto it = S.rd.find(d);
      if (it != S.rd.end() && (it->second.omin != 0 || it->second.omax != 0 || it->second.oc != 0 || it->second.ob != 0))
        return fail(why, "loop reads its own output at an offset");
    }
  }
  if (ncst > SW_MAXC) return fail(why, "constants");
  if (tape_total > 1600) return fail(why, "tape length");
  const long long nd = static_cast<long long>(pl.D.size());
  auto writes = [&](int j, int d) {
    for (int x : pl.L[static_cast<std::size_t>(j)].wds)
      if (x == d) return true;
    return false;
  };
  auto reads = [&](int j, int d) { return pl.L[static_cast<std::size_t>(j)].rd.count(d) > 0; };
  for (int d = 0; d < nd; ++d)
    for (int j = 0; j < n; ++j)
      if (writes(j, d)) pl.D[static_cast<std::size_t>(d)].writers.push_back(j);
  // ---- column halos (backward), and along dim 1 for 3-D plane tiles
  for (int k = n - 1; k >= 0; --k)
    for (const auto& [d, r] : pl.L[static_cast<std::size_t>(k)].rd)
      for (int j = 0; j < k; ++j)
        if (writes(j, d)) {
          SwLoop& J = pl.L[static_cast<std::size_t>(j)];
          const SwLoop& Kl = pl.L[static_cast<std::size_t>(k)];
          J.h = std::max(J.h, Kl.h + r.oc);
          J.hb = std::max(J.hb, Kl.hb + r.ob);
        }
  long long HC = 0, HB = 0;
  for (const SwLoop& S : pl.L) {
    HC = std::max(HC, S.h);
    HB = std::max(HB, S.hb);
    for (const auto& [d, r] : S.rd) {
      HC = std::max(HC, S.h + r.oc);
      HB = std::max(HB, S.hb + r.ob);
    }
  }
  if (HC > 16 || 2 * HC >= pl.RC / 2) return fail(why, "column halo");
  if (pl.nd == 3 && 2 * HB > pl.RB / 2) return fail(why, "dim-1 halo");
  pl.HC = HC;
  pl.TC = pl.RC - 2 * HC;
  pl.HB = pl.nd == 3 ? HB : 0;
  pl.TB = pl.RB - 2 * pl.HB;
  // shared memory around the rings: the farthest neighbour read of an edge lane
  // (a multiple of 16 doubles: 3-D tensor copies land on 128-byte aligned plane slots)
  pl.pad = (std::max<long long>(32, pl.HB * pl.RCp + pl.HC + 4) + 15) / 16 * 16;
  pl.SP = static_cast<long long>(pl.RB) * pl.RCp;
  if (pl.nd == 3) pl.SP = (pl.SP + 15) / 16 * 16;  // every plane slot starts 128-byte aligned
  // ---- loaded / written / out-of-place
  for (int d = 0; d < nd; ++d) {
    SwDs& D = pl.D[static_cast<std::size_t>(d)];
    D.written = !D.writers.empty();
    for (int k = 0; k < n && !D.loaded; ++k) {
      if (!reads(k, d)) continue;
      const ooc_loop& L = Ls[k];
      const Rd& r = pl.L[static_cast<std::size_t>(k)].rd.at(d);
      const int dc = pl.nd - 1;  // column dimension
      const long long b0 = L.lo[0] + r.omin, b1 = L.hi[0] + r.omax, c0 = L.lo[dc] - r.oc, c1 = L.hi[dc] + r.oc;
      const long long y0 = pl.nd == 3 ? L.lo[1] - r.ob : 0, y1 = pl.nd == 3 ? L.hi[1] + r.ob : 1;
      bool covered = false;
      for (int j = 0; j < k && !covered; ++j)
        if (writes(j, d))
          covered = Ls[j].lo[0] <= b0 && Ls[j].hi[0] >= b1 && Ls[j].lo[dc] <= c0 && Ls[j].hi[dc] >= c1 &&
                    (pl.nd == 2 || (Ls[j].lo[1] <= y0 && Ls[j].hi[1] >= y1));
      if (!covered) D.loaded = true;
    }
    D.oop = D.loaded && D.written;
    D.store = D.written && !(dead && std::find(dead->begin(), dead->end(), D.v->data) != dead->end());
  }
  // ---- lags (forward). Default: the tightest lags, with a barrier inside the step where
  // a region's column-offset access conflicts. OOC_SWEEP_SKEW=1 instead delays every
  // access that crosses threads (a column offset) by one step (K rows): a reader takes
  // the writer's rows of the PREVIOUS step, a writer overwrites rows its column-offset
  // readers finished in the previous step — the step barrier then orders every
  // cross-thread dependency and no barrier is left inside a step (measured slower on
  // miniflow2d: 3.35 vs 3.06 ms per timestep, the larger rings cost more than the barrier).
  static const bool skew = std::getenv("OOC_SWEEP_SKEW") && std::atoi(std::getenv("OOC_SWEEP_SKEW")) == 1;
  for (int i = 0; i < n; ++i) {
    SwLoop& S = pl.L[static_cast<std::size_t>(i)];
    long long lag = LLONG_MIN;
    for (const auto& [d, r] : S.rd)
      for (int j = 0; j < i; ++j)
        if (writes(j, d))
          lag = std::max(lag, pl.L[static_cast<std::size_t>(j)].lag + r.omax + (skew && r.oc != 0 ? K : 0));
    for (int d : S.wds)
      for (int j = 0; j < i; ++j) {
        const SwLoop& J = pl.L[static_cast<std::size_t>(j)];
        if (reads(j, d)) lag = std::max(lag, J.lag - J.rd.at(d).omin + (skew && J.rd.at(d).oc != 0 ? K : 0));
        if (writes(j, d)) lag = std::max(lag, J.lag);
      }
    S.lag = lag == LLONG_MIN ? 0 : lag;
  }
  for (int d = 0; d < nd; ++d) {
    SwDs& D = pl.D[static_cast<std::size_t>(d)];
    if (!D.loaded) continue;
    long long l = LLONG_MAX;
    for (int k = 0; k < n; ++k) {
      if (reads(k, d)) l = std::min(l, pl.L[static_cast<std::size_t>(k)].lag - pl.L[static_cast<std::size_t>(k)].rd.at(d).omax);
      if (writes(k, d)) l = std::min(l, pl.L[static_cast<std::size_t>(k)].lag);
    }
    D.lagL = l;
  }
  long long m = LLONG_MAX;
  for (const SwLoop& S : pl.L) m = std::min(m, S.lag);
  for (const SwDs& D : pl.D)
    if (D.loaded) m = std::min(m, D.lagL);
  for (SwLoop& S : pl.L) S.lag -= m;
  for (SwDs& D : pl.D)
    if (D.loaded) D.lagL -= m;
  for (SwDs& D : pl.D)
    for (int j : D.writers) D.lagS = std::max(D.lagS, pl.L[static_cast<std::size_t>(j)].lag);
  // ---- ring windows: rows live at step s are [sK - A, sK + B]
  long long off = 0;
  for (int d = 0; d < nd; ++d) {
    SwDs& D = pl.D[static_cast<std::size_t>(d)];
    long long A = LLONG_MIN, B = LLONG_MIN;
    if (D.loaded) {
      A = std::max(A, D.lagL);
      B = std::max(B, (P + 1) * K - 1 - D.lagL);
    }
    if (D.written) A = std::max(A, D.lagS);
    if (pl.bulk_st && D.store) A = std::max(A, D.lagS + K);  // read by the producer's bulk store one step later
    for (int k = 0; k < n; ++k) {
      const SwLoop& S = pl.L[static_cast<std::size_t>(k)];
      if (reads(k, d)) {
        A = std::max(A, S.lag - S.rd.at(d).omin);
        B = std::max(B, K - 1 - S.lag + S.rd.at(d).omax);
      }
      if (writes(k, d)) {
        A = std::max(A, S.lag);
        B = std::max(B, K - 1 - S.lag);
      }
    }
    D.need = std::max<long long>(A + B + 1, K);
  }
  // ring lengths: powers of two (default), or with OOC_SWEEP_RING=period the smallest
  // divisor of a common period U >= each ring's live rows, U among 8, 12, 16, 24 for the
  // fewest rows in total. Either way every ring length divides U, so the interior steps
  // unroll U times with constant slots. Period rings save shared memory (3 CTAs per SM
  // instead of 2 on miniflow2d) but measured slower: 3.3-3.6 ms per timestep against
  // 2.64-2.68 ms with power-of-two rings (round-2 record in profiles/).
  {
    static const bool pow2_only = !(std::getenv("OOC_SWEEP_RING") && std::string(std::getenv("OOC_SWEEP_RING")) == "period");
    long long bestU = 0, bestRows = LLONG_MAX;
    for (long long Uc : {8LL, 12LL, 16LL, 24LL}) {
      if (pow2_only && (Uc & (Uc - 1))) continue;
      long long rows = 0;
      bool okU = true;
      for (const SwDs& D : pl.D) {
        long long w = D.need;
        while (w <= Uc && Uc % w) ++w;
        if (w > Uc) {
          okU = false;
          break;
        }
        rows += w;
      }
      if (okU && rows < bestRows) {
        bestRows = rows;
        bestU = Uc;
      }
    }
    pl.U = bestU;
    pl.NB = bestU > 0 ? static_cast<int>(bestU) : 8;
    for (SwDs& D : pl.D) {
      if (bestU > 0) {
        D.W = D.need;
        while (bestU % D.W) ++D.W;
      } else {  // rings longer than 24 rows: powers of two, no unrolled steps
        D.W = 1;
        while (D.W < D.need) D.W *= 2;
      }
      D.off = off;
      off += D.W * pl.SP;
    }
  }
  pl.smem = (off + 2 * pl.pad) * 8;
  if (pl.smem > (pl.nd == 2 ? smem_budget() : smem_budget3())) return fail(why, "shared memory");
  // ---- warm-up depth: first correct row of every version (relative to the sweep start)
  const long long NONE = LLONG_MIN / 4;
  std::vector<long long> F(static_cast<std::size_t>(nd), NONE);
  for (int d = 0; d < nd; ++d)
    if (pl.D[static_cast<std::size_t>(d)].loaded) F[static_cast<std::size_t>(d)] = -pl.D[static_cast<std::size_t>(d)].lagL;
  long long F_red = NONE;
  for (int i = 0; i < n; ++i) {
    const SwLoop& S = pl.L[static_cast<std::size_t>(i)];
    long long Fi = -S.lag;
    for (const auto& [d, r] : S.rd) {
      if (F[static_cast<std::size_t>(d)] == NONE) return fail(why, "read of an unwritten, unloaded dataset");
      Fi = std::max(Fi, F[static_cast<std::size_t>(d)] - r.omin);
    }
    for (int d : S.wds) F[static_cast<std::size_t>(d)] = F[static_cast<std::size_t>(d)] == NONE ? Fi : std::max(F[static_cast<std::size_t>(d)], Fi);
    if (Ls[i].reduce_op != OOC_RED_NONE) {
      F_red = Fi;
      pl.red_op = Ls[i].reduce_op;
      pl.red_lag = S.lag;
    }
  }
  pl.warm = 0;
  pl.lagS_max = 0;
  if (pl.red_op != OOC_RED_NONE) {  // the reduction counts owned rows only: they must be exact
    pl.warm = std::max(pl.warm, F_red);
    pl.lagS_max = std::max(pl.lagS_max, pl.red_lag);
  }
  for (int d = 0; d < nd; ++d)
    if (pl.D[static_cast<std::size_t>(d)].store) {
      pl.warm = std::max(pl.warm, F[static_cast<std::size_t>(d)]);
      pl.lagS_max = std::max(pl.lagS_max, pl.D[static_cast<std::size_t>(d)].lagS);
    }
  // ---- barriers: a thread owns one ring column for every row, so only column-offset
  // accesses cross threads. A loop starts a new region (barrier) when it reads at a
  // column offset a dataset the current region wrote, or writes a dataset the region
  // read at a column offset; row-offset and point accesses stay in program order.
  std::vector<char> rc(static_cast<std::size_t>(nd), 0), ww(static_cast<std::size_t>(nd), 0);
  for (int i = 0; i < n && !skew; ++i) {
    SwLoop& S = pl.L[static_cast<std::size_t>(i)];
    bool conflict = false;
    for (const auto& [d, r] : S.rd) conflict = conflict || ((r.oc != 0 || r.ob != 0) && ww[static_cast<std::size_t>(d)]);
    for (int d : S.wds) conflict = conflict || rc[static_cast<std::size_t>(d)];
    if (conflict && i > 0) {
      S.barrier = true;
      std::fill(rc.begin(), rc.end(), 0);
      std::fill(ww.begin(), ww.end(), 0);
    }
    for (const auto& [d, r] : S.rd)
      if (r.oc != 0 || r.ob != 0) rc[static_cast<std::size_t>(d)] = 1;
    for (int d : S.wds) ww[static_cast<std::size_t>(d)] = 1;
  }
  // ---- launch box: loop ranges plus the allocations of out-of-place outputs (their
  // shadow must receive every element, written or not)
  const int dc = pl.nd - 1;  // column (contiguous) dimension
  long long bx[6] = {LLONG_MAX, LLONG_MIN, LLONG_MAX, LLONG_MIN, 0, 1};
  if (pl.nd == 3) {
    bx[4] = LLONG_MAX;
    bx[5] = LLONG_MIN;
  }
  auto grow = [&](const int64_t* lo, const int64_t* hi) {
    bx[0] = std::min<long long>(bx[0], lo[0]);
    bx[1] = std::max<long long>(bx[1], hi[0]);
    bx[2] = std::min<long long>(bx[2], lo[dc]);
    bx[3] = std::max<long long>(bx[3], hi[dc]);
    if (pl.nd == 3) {
      bx[4] = std::min<long long>(bx[4], lo[1]);
      bx[5] = std::max<long long>(bx[5], hi[1]);
    }
  };
  auto npts = [&] {
    return static_cast<double>(bx[1] - bx[0]) * static_cast<double>(bx[3] - bx[2]) * static_cast<double>(bx[5] - bx[4]);
  };
  for (int i = 0; i < n; ++i) grow(Ls[i].lo, Ls[i].hi);
  const double pts_loops = npts();
  for (const SwDs& D : pl.D)
    if (D.oop) grow(D.v->lo, D.v->hi);
  const double pts = npts();
  if (pts > 1.25 * pts_loops + 4096) return fail(why, "out-of-place allocation much larger than the loops");
  for (int k = 0; k < 6; ++k) pl.box[k] = bx[k];
  // a reducing run writes one partial per CTA into the queue's partial buffer (8192)
  if (pl.red_op != OOC_RED_NONE &&
      (bx[3] - bx[2] + pl.TC - 1) / pl.TC * ((bx[5] - bx[4] + pl.TB - 1) / pl.TB) > 4096)
    return fail(why, "reduction over too many strips");
  return true;
}

// Kernel source of an analysed group (structure only: ranges, pointers and
// constants are parameters). Fills the constant table in tape order.
std::string generate(const ooc_loop* Ls, const SwPlan& pl, std::vector<double>* cst) {
  // One thread per ring column (NT = 128); each thread evaluates K consecutive rows of
  // every loop per step. Ring sizes are powers of two and every thread of the CTA works
  // on the same rows, so ring slot offsets are CTA-uniform and every shared-memory
  // access is [thread base + uniform slot + immediate]. Steps whose rows lie inside
  // every loop range, store window and load box (all but a few at the ends of a
  // segment) run a body without any row predicate.
  std::ostringstream o;
  const int nd = static_cast<int>(pl.D.size());
  const int K = pl.K;
  // barrier among the ring threads (the TMA producer warp only joins the step barriers)
  const int NTc = pl.RB * pl.RC;  // consumer (ring) threads
  const bool d3 = pl.nd == 3;
  const std::string cbar = pl.tma ? "asm volatile(\"bar.sync 1, " + std::to_string(NTc) + ";\" ::: \"memory\");"
                                  : std::string("__syncthreads();");
  o << "#define SW_MAXL " << SW_MAXL << "\n#define SW_MAXD " << SW_MAXD << "\n#define SW_MAXC " << SW_MAXC << "\n";
  o << kSweepDecl;
  static const int min_blocks = [] {
    const char* e = std::getenv("OOC_SWEEP_MINB");
    return e ? std::atoi(e) : 0;
  }();
  // resident CTAs the shared memory allows (228 KB per SM, 1 KB reserved per CTA): ask
  // ptxas to fit that many in the register file too
  const long long smem_occ = std::min<long long>(8, 233472 / (pl.smem + 1024 + 256));
  o << "extern \"C\" __global__ void __launch_bounds__(" << pl.NT;
  if (min_blocks > 0) o << ", " << min_blocks;
  else if (smem_occ > 1) o << ", " << smem_occ;
  o << ") ooc_sweep_kernel(const __grid_constant__ SweepParams p" << (d3 ? ", const __grid_constant__ SwMaps m" : "")
    << ") {\n";
  o << "  extern __shared__ __align__(128) double sw_sm[];\n";
  if (pl.tma) o << "  __shared__ __align__(8) unsigned long long sw_bar[" << pl.NB << "];\n";
  // thread -> ring column lc (and, 3-D, tile row lb); CTA tile origin (c0, b0)
  o << "  const int lc = threadIdx.x % " << pl.RC << ", lb = threadIdx.x / " << pl.RC << ";\n";
  o << "  double* const B = sw_sm + " << pl.pad << " + lb * " << pl.RCp << " + lc;\n";
  // CTA -> (strip, row segment). The column-edge strips run the masked step body (their
  // halo columns leave some loop's range), ~3x longer than an interior strip's CTA: with
  // p.edge_first their CTAs take the first linear block indices — the block scheduler
  // dispatches in that order — so they start in the first wave instead of forming the
  // kernel's tail (measured: 58 edge CTAs of 905 us ending 550 us after the rest).
  o << "  long long sw_tx, sw_ty;\n  {\n"
       "    const long long lin = static_cast<long long>(blockIdx.y) * gridDim.x + blockIdx.x;\n"
       "    const long long nx = gridDim.x, ny = gridDim.y, ne = p.edge_first ? 2 * (nx / p.ntc) : 0;\n"
       "    if (lin < ne * ny) {\n"
       "      const long long k = lin % ne;\n"
       "      sw_ty = lin / ne;\n"
       "      sw_tx = (k >> 1) * p.ntc + ((k & 1) ? p.ntc - 1 : 0);\n"
       "    } else {\n"
       "      const long long l = lin - ne * ny, ni = nx - ne, i = l % ni;\n"
       "      sw_ty = l / ni;\n"
       "      sw_tx = p.edge_first ? (i / (p.ntc - 2)) * p.ntc + 1 + i % (p.ntc - 2) : i;\n"
       "    }\n  }\n";
  o << "  const long long c0 = p.C0 + (sw_tx % p.ntc) * " << pl.TC << ";\n";
  if (d3) {
    o << "  const long long b0 = p.B0 + (sw_tx / p.ntc) * " << pl.TB << ";\n";
    o << "  const long long b = b0 - " << pl.HB << " + lb;\n";
  }
  // one restrict-qualified base per ring: rings never overlap, so the compiler may move
  // a ring's loads across another ring's stores (instruction-level parallelism)
  static const bool restrict_rings = !(std::getenv("OOC_SWEEP_RESTRICT") && std::atoi(std::getenv("OOC_SWEEP_RESTRICT")) == 0);
  // TMA: a loaded dataset's ring rows start at the even view column at or below the
  // CTA's first ring column (16-byte aligned row copies); lanes read one element further
  // when that column is odd
  for (int d = 0; d < nd; ++d) {
    const SwDs& D = pl.D[static_cast<std::size_t>(d)];
    o << "  double* " << (restrict_rings ? "__restrict__ " : "") << "const R" << d << " = B + " << D.off;
    if (pl.tma && (D.loaded || (pl.bulk_st && D.store)))
      o << " + static_cast<int>((c0 - " << pl.HC << " - p.box[" << d << "][2]) & 1)";
    o << ";\n";
  }
  o << "  const long long r_own0 = p.R0 + sw_ty * p.seg_rows;\n";
  o << "  const long long r_own1 = min(p.R1, r_own0 + p.seg_rows);\n";
  o << "  const long long rbase = r_own0 - " << pl.warm << ";\n";
  o << "  const long long c = c0 - " << pl.HC << " + lc;\n";
  o << "  const int nsteps = static_cast<int>((r_own1 - rbase + " << pl.lagS_max << " + " << K - 1 << ") / " << K << ");\n";
  // fast steps: every row predicate true for all K rows
  o << "  long long s_lo = 0, s_hi = nsteps;\n";
  auto fast_rows = [&](long long q, const std::string& A, const std::string& Bs) {
    o << "  s_lo = max(s_lo, -sw_floordiv(-((" << A << ") - rbase - (" << q << ")), " << K << "));\n";
    o << "  s_hi = min(s_hi, sw_floordiv((" << Bs << ") - rbase - (" << q << ") - " << K << ", " << K << ") + 1);\n";
  };
  for (int i = 0; i < pl.n; ++i)
    fast_rows(-pl.L[static_cast<std::size_t>(i)].lag, "p.rng[" + std::to_string(i) + "][0]",
              "p.rng[" + std::to_string(i) + "][1]");
  for (int d = 0; d < nd; ++d) {
    const SwDs& D = pl.D[static_cast<std::size_t>(d)];
    const std::string ds = std::to_string(d);
    if (D.loaded) fast_rows(static_cast<long long>(pl.P) * K - D.lagL, "p.box[" + ds + "][0]", "p.box[" + ds + "][1]");
    if (D.store) {
      fast_rows(-D.lagS, "max(r_own0, p.box[" + ds + "][0])", "min(r_own1, p.box[" + ds + "][1])");
      if (!D.oop)
        for (int j : D.writers)
          fast_rows(-D.lagS, "p.rng[" + std::to_string(j) + "][0]", "p.rng[" + std::to_string(j) + "][1]");
    }
  }
  if (pl.red_op != OOC_RED_NONE) {
    const std::string ri = std::to_string(pl.n - 1);
    fast_rows(-pl.red_lag, "max(r_own0, p.rng[" + ri + "][0])", "min(r_own1, p.rng[" + ri + "][1])");
    o << "  double racc = " << (pl.red_op == OOC_RED_SUM ? "0.0" : pl.red_op == OOC_RED_MIN ? "__longlong_as_double(0x7ff0000000000000LL)"
                                                                                           : "__longlong_as_double(0xfff0000000000000LL)")
      << ";\n";
  }
  // column predicates of every loop / store, once per thread, as bit masks
  o << "  unsigned long long colmask = 0ull;\n  unsigned stmask = 0u;\n";
  for (int i = 0; i < pl.n; ++i) {
    const SwLoop& S = pl.L[static_cast<std::size_t>(i)];
    o << "  if (lc >= " << pl.HC - S.h << " && lc < " << pl.HC + pl.TC + S.h << " && c >= p.rng[" << i
      << "][2] && c < p.rng[" << i << "][3]";
    if (d3)
      o << " && lb >= " << pl.HB - S.hb << " && lb < " << pl.HB + pl.TB + S.hb << " && b >= p.rng[" << i << "][4] && b < p.rng["
        << i << "][5]";
    o << ") colmask |= 1ull << " << i << ";\n";
  }
  o << "  const bool own_col = lc >= " << pl.HC << " && lc < " << pl.HC + pl.TC << " && c < p.C1";
  if (d3) o << " && lb >= " << pl.HB << " && lb < " << pl.HB + pl.TB << " && b < p.B1";
  o << ";\n";
  // bulk stores cover the owned columns from the first 16-byte aligned one to the last; the
  // (at most two) edge columns outside are stored by their threads (stedge)
  if (pl.bulk_st) {
    o << "  unsigned stedge = 0u;\n";
    for (int d = 0; d < nd; ++d) {
      const SwDs& D = pl.D[static_cast<std::size_t>(d)];
      if (!D.store) continue;
      const std::string ds = std::to_string(d);
      o << "  if (own_col && (c < c0 + ((c0 - p.box[" << ds << "][2]) & 1) || c >= c0 + " << pl.TC << " - ((c0 + " << pl.TC
        << " - p.box[" << ds << "][2]) & 1))) stedge |= 1u << " << d << ";\n";
    }
  }
  // interior strip: all 128 ring columns inside every loop range and load box, every
  // owned column inside the launch box — the fast steps then evaluate every loop on
  // every lane without predicates (lanes outside a loop's halo produce values nobody
  // reads; their neighbour reads stay inside the padded shared-memory window)
  o << "  const long long cl = c0 - " << pl.HC << ", ch = cl + " << pl.RC << ";\n";
  o << "  bool strip_in = c0 + " << pl.TC << " <= p.C1;\n";
  for (int i = 0; i < pl.n; ++i)
    o << "  strip_in = strip_in && p.rng[" << i << "][2] <= cl && p.rng[" << i << "][3] >= ch;\n";
  for (int d = 0; d < nd; ++d) {
    const SwDs& D = pl.D[static_cast<std::size_t>(d)];
    if (D.loaded || D.store)
      o << "  strip_in = strip_in && p.box[" << d << "][2] <= cl && p.box[" << d << "][3] >= ch;\n";
  }
  if (d3) {  // the whole plane tile inside every range and box along dim 1 too
    o << "  const long long bl = b0 - " << pl.HB << ", bh = bl + " << pl.RB << ";\n";
    o << "  strip_in = strip_in && b0 + " << pl.TB << " <= p.B1;\n";
    for (int i = 0; i < pl.n; ++i)
      o << "  strip_in = strip_in && p.rng[" << i << "][4] <= bl && p.rng[" << i << "][5] >= bh;\n";
    for (int d = 0; d < nd; ++d) {
      const SwDs& D = pl.D[static_cast<std::size_t>(d)];
      if (D.loaded || D.store)
        o << "  strip_in = strip_in && p.box[" << d << "][4] <= bl && p.box[" << d << "][5] >= bh;\n";
    }
  }
  for (int d = 0; d < nd; ++d) {
    const SwDs& D = pl.D[static_cast<std::size_t>(d)];
    if (D.loaded && !pl.tma)
      o << "  const bool colok" << d << " = c >= p.box[" << d << "][2] && c < p.box[" << d << "][3];\n";
    if (D.store) {
      o << "  if (own_col && c >= p.box[" << d << "][2] && c < p.box[" << d << "][3]";
      if (d3) o << " && b >= p.box[" << d << "][4] && b < p.box[" << d << "][5]";
      o << ") stmask |= 1u << " << d << ";\n";
    }
  }
  if (pl.tma) {
    o << "  if (threadIdx.x == " << NTc << ") {\n";
    o << "    for (int k = 0; k < " << pl.NB << "; ++k)\n";
    o << "      asm volatile(\"mbarrier.init.shared::cta.b64 [%0], 1;\" :: \"r\"(sw_saddr(&sw_bar[k])) : \"memory\");\n";
    o << "    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n";
    o << "  }\n  __syncthreads();\n";
  }
  o << "  asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");\n";
  o << "  asm volatile(\"griddepcontrol.launch_dependents;\" ::: \"memory\");\n";
  if (pl.trace)  // CTA schedule: SM id, start (ns), end (ns)
    o << "  if (threadIdx.x == 0) {\n    unsigned long long t_; unsigned sm_;\n"
         "    asm volatile(\"mov.u64 %0, %%globaltimer;\" : \"=l\"(t_));\n"
         "    asm volatile(\"mov.u32 %0, %%smid;\" : \"=r\"(sm_));\n"
         "    unsigned long long* tr_ = p.trace + 3 * (static_cast<long long>(blockIdx.y) * gridDim.x + blockIdx.x);\n"
         "    tr_[0] = sm_; tr_[1] = t_;\n  }\n";
  // element (dataset d, row u + q) of this thread's column; u, q relative to rbase
  // In an unrolled step (unroll_u >= 0: u = unroll_u modulo the ring period) the slot is a
  // constant; otherwise (u + q) mod W at run time (a mask for power-of-two lengths).
  long long unroll_u = -1;
  const long long PL = pl.SP;  // ring slot pitch ("row": a plane tile in 3-D)
  // a read's cross-thread offset in ring elements: dim-1 offset x pitch + column offset
  // (0: the thread's own element, so it can be forwarded / carried in registers)
  auto xoff = [&](const ooc_ins& in) -> long long {
    return (pl.nd == 3 ? in.offset[1] * pl.RCp : 0) + in.offset[pl.nd - 1];
  };
  auto at = [&](int d, const std::string& u, long long q, long long oc) {
    const SwDs& D = pl.D[static_cast<std::size_t>(d)];
    std::ostringstream e;
    long long extra = -1;
    if (unroll_u >= 0 && u == "u") extra = 0;
    if (unroll_u >= 0 && u == "u + " + std::to_string(K)) extra = K;
    if (extra >= 0) {
      const long long slot = (((unroll_u + extra + q) % D.W) + D.W) % D.W;
      e << "R" << d << "[" << slot * PL;
    } else if ((D.W & (D.W - 1)) == 0) {
      e << "R" << d << "[(((" << u << ") + (" << q << ")) & " << D.W - 1 << ") * " << PL;
    } else {
      e << "R" << d << "[sw_slot((" << u << ") + (" << q << "), " << D.W << ") * " << PL;
    }
    if (oc) e << " + (" << oc << ")";
    e << "]";
    return e.str();
  };
  // element offsets of this thread's column in the row a load (gl) / store (gs) of the
  // current step touches; advanced by K rows per step
  for (int d = 0; d < nd; ++d) {
    const SwDs& D = pl.D[static_cast<std::size_t>(d)];
    if (D.loaded && !pl.tma)
      o << "  long long gl" << d << " = (rbase + " << static_cast<long long>(pl.P) * K - D.lagL << " - p.box[" << d
        << "][0]) * p.s0[" << d << "] + (c - p.box[" << d << "][2]);\n";
    if (D.store)
      o << "  double* gs" << d << " = p.dst[" << d << "] + (rbase - " << D.lagS << " - p.box[" << d << "][0]) * p.s0[" << d
        << "] + (c - p.box[" << d << "][2])" << (d3 ? " + (b - p.box[" + std::to_string(d) + "][4]) * p.s1[" + std::to_string(d) + "]" : "")
        << ";\n";
  }
  auto loads = [&](const std::string& step, const char* ind, bool fast, bool running) {
    if (pl.tma) return;  // issued once per step by one thread (tma_issue)
    for (int d = 0; d < nd; ++d) {
      const SwDs& D = pl.D[static_cast<std::size_t>(d)];
      if (!D.loaded) continue;
      o << ind << "{\n" << ind << "  const int ul = (" << step << ") * " << K << " - " << D.lagL << ";\n";
      if (running)
        o << ind << "  const double* g = p.src[" << d << "] + gl" << d << ";\n";
      else
        o << ind << "  const double* g = p.src[" << d << "] + (rbase + ul - p.box[" << d << "][0]) * p.s0[" << d
          << "] + (c - p.box[" << d << "][2]);\n";
      o << ind << "#pragma unroll\n" << ind << "  for (int r = 0; r < " << K << "; ++r) {\n";
      if (fast) {
        o << ind << "    const bool ok = colok" << d << ";\n";
      } else {
        o << ind << "    const long long row = rbase + ul + r;\n";
        o << ind << "    const bool ok = colok" << d << " && row >= p.box[" << d << "][0] && row < p.box[" << d
          << "][1];\n";
      }
      o << ind << "    sw_cp8(&" << at(d, "ul + r", 0, 0) << ", ok ? g + r * p.s0[" << d << "] : p.src[" << d
        << "], ok);\n";
      o << ind << "  }\n" << ind << "}\n";
    }
    o << ind << "asm volatile(\"cp.async.commit_group;\" ::: \"memory\");\n";
  };
  // TMA issue of the rows of step `step` (thread 0): per loaded dataset and row, one bulk
  // copy of the ring's columns clipped to the view (even start and length: 16-byte
  // aligned), completing on mbarrier step & 7. Rows outside the view are not copied:
  // nothing in range reads them (validate_loop), so stale ring contents only reach
  // values that are never stored.
  // The producer warp (TMA): lane i streams the i-th loaded dataset. Per step, after the
  // consumers' step barrier (which frees the ring rows the next loads overwrite), each
  // lane issues one bulk copy per row of step s+P — the ring's columns clipped to the view
  // (even start and length: 16-byte aligned) — arming barrier (s+P) mod NB with its bytes;
  // lane 0 then arrives. Rows outside the view are not copied: nothing in range reads them
  // (validate_loop), so stale ring contents only reach values that are never stored. An
  // L2 bulk prefetch runs `l2_ahead` steps further, so the ring loads hit L2.
  int nload = 0;
  for (const SwDs& D : pl.D) nload += D.loaded ? 1 : 0;
  static const int l2_ahead = [] {  // steps between an L2 prefetch and the ring load of a row
    const char* e = std::getenv("OOC_SWEEP_L2AHEAD");  // measured neutral to slightly slower: off
    return e ? std::atoi(e) : 0;
  }();
  // copies per step: one per loaded dataset and plane-tile row (RB rows in 3-D); lane l
  // of the producer owns copies l, l + 32, ... (descriptors computed once, in registers)
  const int ncopy = d3 ? nload : nload * pl.RB, J = (ncopy + 31) / 32;
  auto tma_issue = [&](const std::string& step, const std::string& pf, const char* ind) {
    o << ind << "{\n" << ind << "  const int sn = " << step << ", pf = " << pf << ";\n";
    o << ind << "  if (sn >= 0 && sn < nsteps) {\n";
    o << ind << "    const unsigned bar = bar0 + static_cast<unsigned>((sn % " << pl.NB << ") * 8);\n";
    o << ind << "    asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n";
    for (int j = 0; j < J; ++j)
      for (int r = 0; r < K; ++r) {
        const std::string js = std::to_string(j);
        o << ind << "    {\n" << ind << "      const long long v = vr0_" << js << " + static_cast<long long>(sn) * " << K << " + " << r
          << ";\n";
        o << ind << "      if (tn_" << js << " && v >= 0 && v < nrows_" << js << ") {\n";
        o << ind << "        asm volatile(\"mbarrier.expect_tx.shared::cta.b64 [%0], %1;\" :: \"r\"(bar), \"r\"(tn_" << js
          << ") : \"memory\");\n";
        if (d3)
          o << ind << "        sw_tensor3(dst_" << js << " + static_cast<unsigned>(sw_slot(sn * " << K << " + " << r << " - lagL_"
            << js << ", wlen_" << js << ") * " << PL * 8 << "), &m.t[dd_" << js << "][0], tx_" << js << ", ty_" << js
            << ", static_cast<int>(v), bar);\n";
        else
          o << ind << "        sw_bulk(dst_" << js << " + static_cast<unsigned>(sw_slot(sn * " << K << " + " << r << " - lagL_" << js
            << ", wlen_" << js << ") * " << PL * 8 << "), src_" << js << " + v * s0_" << js << ", tn_" << js << ", bar);\n";
        o << ind << "      }\n" << ind << "    }\n";
      }
    o << ind << "    __syncwarp();\n";
    o << ind << "    if (lane == 0) asm volatile(\"mbarrier.arrive.shared::cta.b64 _, [%0];\" :: \"r\"(bar) : \"memory\");\n";
    o << ind << "  }\n";
    o << ind << "  if (pf >= 0 && pf < nsteps) {\n";
    for (int j = 0; j < J; ++j)
      for (int r = 0; r < K; ++r) {
        const std::string js = std::to_string(j);
        o << ind << "    {\n" << ind << "      const long long v = vr0_" << js << " + static_cast<long long>(pf) * " << K << " + " << r
          << ";\n";
        o << ind << "      if (tn_" << js << " && v >= 0 && v < nrows_" << js << ")\n";
        if (d3)  // the plane tile of a later step into L2 (tensor prefetch, same box as the ring load)
          o << ind << "        asm volatile(\"cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];\" :: \"l\"(&m.t[dd_"
            << js << "][0]), \"r\"(tx_" << js << "), \"r\"(ty_" << js << "), \"r\"(static_cast<int>(v)) : \"memory\");\n";
        else
          o << ind << "        asm volatile(\"cp.async.bulk.prefetch.L2.global [%0], %1;\" :: \"l\"(src_" << js << " + v * s0_" << js
            << "), \"r\"(tn_" << js << ") : \"memory\");\n";
        o << ind << "    }\n";
      }
    o << ind << "  }\n" << ind << "}\n";
  };
  if (pl.tma) {
    o << "  if (threadIdx.x >= " << NTc << ") {  // ---- producer warp\n";
    o << "    const int lane = threadIdx.x - " << NTc << ";\n";
    for (int j = 0; j < J; ++j) {
      const std::string js = std::to_string(j);
      o << "    const double* src_" << js << " = nullptr;\n    long long s0_" << js << " = 0, vr0_" << js << " = 0, nrows_" << js
        << " = 0;\n    unsigned dst_" << js << " = 0, tn_" << js << " = 0;\n    int lagL_" << js << " = 0, wlen_" << js << " = 1;\n";
      if (d3) o << "    int dd_" << js << " = 0, tx_" << js << " = 0, ty_" << js << " = 0;\n";
      if (d3)  // one tensor copy per dataset
        o << "    {\n      const int idx = lane + " << 32 * j << ", li = idx, rb = 0;\n";
      else  // one row copy per dataset and tile row
        o << "    {\n      const int idx = lane + " << 32 * j << ", li = idx / " << pl.RB << ", rb = idx % " << pl.RB << ";\n";
      o << "      int dd = -1;\n      long long roff = 0;\n";
      int i = 0;
      for (int d = 0; d < nd; ++d) {
        const SwDs& D = pl.D[static_cast<std::size_t>(d)];
        if (!D.loaded) continue;
        o << "      " << (i ? "else if" : "if") << " (idx < " << ncopy << " && li == " << i << ") { dd = " << d << "; lagL_" << js
          << " = " << D.lagL << "; wlen_" << js << " = " << D.W << "; roff = " << pl.pad + D.off << "; }\n";
        ++i;
      }
      o << "      if (dd >= 0 && " << (d3 ? "true" : "false") << ") {  // 3-D: the plane tile's tensor-copy origin\n";
      o << "        const long long cs = c0 - " << pl.HC << " - p.box[dd][2];\n";
      if (d3) {
        o << "        dd_" << js << " = dd;\n";
        o << "        tx_" << js << " = static_cast<int>(cs - (cs & 1));  // even (16-byte aligned) column at or below the tile\n";
        o << "        ty_" << js << " = static_cast<int>(b0 - " << pl.HB << " - p.box[dd][4]);\n";
        o << "        tn_" << js << " = " << static_cast<long long>(pl.RB) * pl.RCp * 8 << "u;  // the whole box, zero-filled out of bounds\n";
        o << "        vr0_" << js << " = rbase - p.box[dd][0] - lagL_" << js << ";\n";
        o << "        nrows_" << js << " = p.box[dd][1] - p.box[dd][0];\n";
        o << "        dst_" << js << " = sw_saddr(sw_sm) + static_cast<unsigned>(roff * 8);\n";
      }
      o << "      } else if (dd >= 0) {\n";
      o << "        const long long cs = c0 - " << pl.HC << " - p.box[dd][2];\n";
      o << "        const long long a0 = cs > 0 ? (cs & ~1LL) : 0LL;\n";
      o << "        const long long a1 = (min(cs + " << pl.RC << "LL, p.box[dd][3] - p.box[dd][2]) + 1) & ~1LL;\n";
      if (d3) {
        o << "        const long long yb = b0 - " << pl.HB << " + rb - p.box[dd][4];  // this copy's dim-1 row in the view\n";
        o << "        const bool yok = yb >= 0 && yb < p.box[dd][5] - p.box[dd][4];\n";
      } else {
        o << "        const bool yok = true;\n        const long long yb = 0;\n";
      }
      o << "        tn_" << js << " = yok && a1 > a0 ? static_cast<unsigned>(a1 - a0) * 8u : 0u;\n";
      o << "        src_" << js << " = p.src[dd] + a0" << (d3 ? " + yb * p.s1[dd]" : "") << ";\n";
      o << "        s0_" << js << " = p.s0[dd];\n";
      o << "        vr0_" << js << " = rbase - p.box[dd][0] - lagL_" << js << ";  // view row of step sn, row r: vr0 + sn*K + r\n";
      o << "        nrows_" << js << " = p.box[dd][1] - p.box[dd][0];\n";
      o << "        dst_" << js << " = sw_saddr(sw_sm) + static_cast<unsigned>((roff + rb * " << pl.RCp
        << " + a0 - (cs - (cs & 1))) * 8);\n";
      o << "        (void)yb;\n      }\n    }\n";
    }
    o << "    const unsigned bar0 = sw_saddr(sw_bar);\n";
    o << "    for (int t = 0; t < " << pl.P + std::max(l2_ahead, 0) << "; ++t)\n";
    tma_issue("t < " + std::to_string(pl.P) + " ? t : -1",
              l2_ahead > 0 ? "t >= " + std::to_string(pl.P) + " ? t : -1" : "-1", "      ");
    // bulk stores (2-D): lane i copies the aligned owned columns of the i-th stored
    // dataset's row(s) of the PREVIOUS fast step out of its ring slot (kept one step longer
    // for this); the copy has read its rows before the producer joins the next barrier
    int nstore = 0;
    for (const SwDs& D : pl.D) nstore += D.store ? 1 : 0;
    const bool bst = pl.bulk_st && nstore > 0;
    auto bulk_store = [&](const std::string& step, const char* ind) {
      o << ind << "if (sdd >= 0 && snb && strip_in && (" << step << ") >= s_lo && (" << step << ") < s_hi) {\n";
      for (int r = 0; r < K; ++r) {
        o << ind << "  {\n" << ind << "    const int v = (" << step << ") * " << K << " + " << r << ";\n";
        o << ind << "    asm volatile(\"cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\" :: \"l\"(sg + static_cast<long long>(v) * ss0), "
          << "\"r\"(ssrc + static_cast<unsigned>(sw_slot(v - slagS, swl) * " << pl.RCp * 8 << ")), \"r\"(snb) : \"memory\");\n";
        o << ind << "  }\n";
      }
      o << ind << "  asm volatile(\"cp.async.bulk.commit_group;\" ::: \"memory\");\n" << ind << "}\n";
    };
    if (bst) {
      o << "    int sdd = -1, slagS = 0, swl = 1;\n    long long sroff = 0;\n";
      int i = 0;
      for (int d = 0; d < nd; ++d) {
        const SwDs& D = pl.D[static_cast<std::size_t>(d)];
        if (!D.store) continue;
        o << "    " << (i ? "else if" : "if") << " (lane == " << i << ") { sdd = " << d << "; slagS = " << D.lagS << "; swl = " << D.W
          << "; sroff = " << pl.pad + D.off << "; }\n";
        ++i;
      }
      o << "    double* sg = nullptr;\n    long long ss0 = 0;\n    unsigned ssrc = 0, snb = 0;\n";
      o << "    if (sdd >= 0) {\n";
      o << "      const long long ce0 = c0 + ((c0 - p.box[sdd][2]) & 1), ce1 = c0 + " << pl.TC << " - ((c0 + " << pl.TC
        << " - p.box[sdd][2]) & 1);\n";
      o << "      sg = p.dst[sdd] + (rbase - slagS - p.box[sdd][0]) * p.s0[sdd] + (ce0 - p.box[sdd][2]);\n";
      o << "      ss0 = p.s0[sdd];\n";
      o << "      ssrc = sw_saddr(sw_sm) + static_cast<unsigned>((sroff + (ce0 - c0 + " << pl.HC << ") + ((c0 - " << pl.HC
        << " - p.box[sdd][2]) & 1)) * 8);\n";
      o << "      snb = ce1 > ce0 ? static_cast<unsigned>(ce1 - ce0) * 8u : 0u;\n";
      o << "    }\n";
    }
    o << "    for (int s = 0; s < nsteps; ++s) {\n";
    if (bst) o << "      asm volatile(\"cp.async.bulk.wait_group.read 0;\" ::: \"memory\");\n";
    o << "      __syncthreads();\n";
    tma_issue("s + " + std::to_string(pl.P), l2_ahead > 0 ? "s + " + std::to_string(pl.P + l2_ahead) : "-1", "      ");
    if (bst) bulk_store("s - 1", "      ");
    o << "    }\n";
    if (bst) {  // the consumers' last step: one more barrier, then its rows; drain before exit
      o << "    __syncthreads();\n";
      bulk_store("nsteps - 1", "    ");
      o << "    asm volatile(\"cp.async.bulk.wait_group 0;\" ::: \"memory\");\n";
    }
    o << "    return;\n  }\n";
  } else
    for (int t = 0; t < pl.P; ++t) loads(std::to_string(t), "  ", false, false);
  int ci0 = 0;
  // ---- fast steps: rows r = 0..K-1 unrolled at generation so values stay in named
  // registers across loops. A read of a value this thread produced earlier in the step
  // (same dataset version, same row, column offset 0) is forwarded from its register;
  // repeated reads of one ring element are loaded once; a write skips its shared-memory
  // store when every consumer is such a forwarded read (and a final row stored this
  // step takes the register too). Shared-memory bandwidth is the sweep's bound.
  std::vector<std::vector<int>> prevw(static_cast<std::size_t>(pl.n), std::vector<int>(static_cast<std::size_t>(nd), -1));
  for (int k = 0; k < pl.n; ++k)
    for (int d = 0; d < nd; ++d)
      for (int j = k - 1; j >= 0 && prevw[static_cast<std::size_t>(k)][static_cast<std::size_t>(d)] < 0; --j)
        for (int w : pl.L[static_cast<std::size_t>(j)].wds)
          if (w == d) prevw[static_cast<std::size_t>(k)][static_cast<std::size_t>(d)] = j;
  auto tape_reads = [&](int k, std::vector<std::tuple<int, long long, long long>>& out) {
    const ooc_loop& L = Ls[k];
    for (int t = 0; t < L.ntape; ++t)
      if (L.tape[t].op == OOC_OP_READ)
        for (int d = 0; d < nd; ++d)
          if (pl.D[static_cast<std::size_t>(d)].v->data == L.args[L.tape[t].arg].data)
            out.emplace_back(d, L.tape[t].offset[0], xoff(L.tape[t]));
  };
  std::vector<std::vector<char>> need_sts(static_cast<std::size_t>(pl.n), std::vector<char>(static_cast<std::size_t>(nd), 0));
  std::vector<int> last_writer(static_cast<std::size_t>(nd), -1);
  for (int j = 0; j < pl.n; ++j)
    for (int d : pl.L[static_cast<std::size_t>(j)].wds) last_writer[static_cast<std::size_t>(d)] = j;
  // A value may reach a consumer from ANY earlier writer of the dataset (loop ranges
  // differ: where the latest writer is inactive, an older one supplied the point), and
  // slow steps always read shared memory. So a write skips its store only if every later
  // read of the dataset, and the final-row store, happen in the same step at the same
  // row and column (forwardable in fast steps; a slow step re-stores what it writes).
  for (int k = 0; k < pl.n; ++k) {
    std::vector<std::tuple<int, long long, long long>> rs;
    tape_reads(k, rs);
    for (const auto& [d, orow, ocol] : rs)
      for (int j = 0; j < k; ++j)
        for (int w : pl.L[static_cast<std::size_t>(j)].wds)
          if (w == d && (ocol != 0 || orow - pl.L[static_cast<std::size_t>(k)].lag != -pl.L[static_cast<std::size_t>(j)].lag))
            need_sts[static_cast<std::size_t>(j)][static_cast<std::size_t>(d)] = 1;
  }
  for (int d = 0; d < nd; ++d) {
    const SwDs& D = pl.D[static_cast<std::size_t>(d)];
    if (!D.store) continue;
    for (int j : D.writers)
      if (pl.L[static_cast<std::size_t>(j)].lag != D.lagS) need_sts[static_cast<std::size_t>(j)][static_cast<std::size_t>(d)] = 1;
  }
  static const bool forward = !(std::getenv("OOC_SWEEP_FWD") && std::atoi(std::getenv("OOC_SWEEP_FWD")) == 0);
  if (!forward)
    for (auto& v : need_sts) std::fill(v.begin(), v.end(), 1);
  // Carries: a ring element this thread holds in a register at the end of a fast step
  // (row u+q+K, column offset 0) whose first access in the next step is a read of the
  // same element (now row u'+q) enters that step as a register — the row-offset reads of
  // stencils stop re-loading rows the column already read. Only this thread writes its
  // column and loads land in rows of later steps, so the value cannot change in between;
  // after a slow step the carries are reloaded from the rings.
  using Key = std::tuple<int, long long, long long>;
  struct FastInfo {
    std::vector<Key> first_read;    // keys whose first access in the step is a read
    std::vector<char> miss;         // per dataset: some fast-step value came from its ring
    std::map<Key, std::string> end; // register of each cached key at the end of the step
  };
  std::vector<std::pair<Key, std::string>> carries;  // (key at step start, register name)
  // datasets whose fast steps never read their ring (every value forwarded or carried):
  // their fast-step writes skip the shared-memory store, and the last fast step spills
  // the carries so the predicated steps after it find the rows in the ring
  std::vector<char> no_smem(static_cast<std::size_t>(nd), 0);
  auto fast_body = [&](FastInfo* info, const std::string& uexpr) {
    const char* ind = "      ";
    loads("s + " + std::to_string(pl.P), ind, true, true);
    o << ind << "const int u = " << uexpr << ";\n";
    std::map<std::tuple<int, long long, long long>, std::string> cache;  // (d, row, col) -> register
    std::set<Key> touched;
    if (info) info->miss.assign(static_cast<std::size_t>(nd), 0);
    if (!carries.empty()) {
      o << ind << "if (!prev_fast) {\n";
      for (const auto& [k, name] : carries)
        o << ind << "  " << name << " = " << at(std::get<0>(k), "u", std::get<1>(k), 0) << ";\n";
      o << ind << "}\n";
      for (const auto& [k, name] : carries) cache[k] = name;
    }
    int ci = ci0;
    for (int i = 0; i < pl.n; ++i) {
      const ooc_loop& L = Ls[i];
      const SwLoop& S = pl.L[static_cast<std::size_t>(i)];
      if (S.barrier) o << ind << cbar << "\n";
      o << ind << "// loop " << i << " (lag " << S.lag << ", halo " << S.h << ")\n";
      int dsof_arg[OOC_MAX_ARGS];
      for (int a = 0; a < L.nargs; ++a) {
        dsof_arg[a] = -1;
        for (int d = 0; d < nd; ++d)
          if (pl.D[static_cast<std::size_t>(d)].v->data == L.args[a].data) dsof_arg[a] = d;
      }
      std::vector<std::vector<std::string>> outs(static_cast<std::size_t>(K));
      const int ci_loop = ci;
      for (int r = 0; r < K; ++r) {
        ci = ci_loop;
        const long long q0 = r - S.lag;
        int tmp = 0;
        const ooc_ins* t = L.tape;
        const std::string pre = "f" + std::to_string(i) + "_" + std::to_string(r) + "_";
        for (int w = 0; w < L.nwrites + (L.reduce_op != OOC_RED_NONE ? 1 : 0); ++w) {
          std::vector<std::string> st;
          for (int k = 0; k < (w < L.nwrites ? L.write_len[w] : L.reduce_len); ++k, ++t) {
            const ooc_ins& in = *t;
            if (in.op == OOC_OP_CONST) {
              st.push_back("p.cst[" + std::to_string(ci++) + "]");
            } else if (in.op == OOC_OP_READ) {
              const int d = dsof_arg[in.arg];
              const auto key = std::make_tuple(d, q0 + in.offset[0], xoff(in));
              if (info && touched.insert(key).second && xoff(in) == 0) info->first_read.push_back(key);
              auto it = forward ? cache.find(key) : cache.end();
              if (it == cache.end()) {
                const std::string name = pre + std::to_string(tmp++);
                o << ind << "const double " << name << " = " << at(d, "u", q0 + in.offset[0], xoff(in)) << ";\n";
                it = cache.emplace(key, name).first;
                if (info) info->miss[static_cast<std::size_t>(d)] = 1;
              }
              st.push_back(it->second);
            } else {
              const std::string y = st.back();
              st.pop_back();
              const std::string x = st.back();
              st.pop_back();
              const std::string name = pre + std::to_string(tmp++);
              o << ind << "const double " << name << " = ";
              switch (in.op) {
                case OOC_OP_ADD: o << x << " + " << y; break;
                case OOC_OP_SUB: o << x << " - " << y; break;
                case OOC_OP_MUL: o << x << " * " << y; break;
                case OOC_OP_DIV: o << x << " / " << y; break;
                case OOC_OP_MIN: o << "ooc_min(" << x << ", " << y << ")"; break;
                default: o << "ooc_max(" << x << ", " << y << ")"; break;
              }
              o << ";\n";
              st.push_back(name);
            }
          }
          outs[static_cast<std::size_t>(r)].push_back(st.back());
        }
      }
      // writes land after every tape of the point (and of every row) has been evaluated
      for (int r = 0; r < K; ++r)
        for (int w = 0; w < L.nwrites; ++w) {
          const int d = S.wds[static_cast<std::size_t>(w)];
          const long long q = r - S.lag;
          const std::string& v = outs[static_cast<std::size_t>(r)][static_cast<std::size_t>(w)];
          for (auto it = cache.begin(); it != cache.end();)
            it = std::get<0>(it->first) == d && (std::get<1>(it->first) == q || std::get<2>(it->first) != 0)
                     ? cache.erase(it) : std::next(it);
          cache[std::make_tuple(d, q, 0LL)] = v;
          touched.insert(std::make_tuple(d, q, 0LL));
          if (need_sts[static_cast<std::size_t>(i)][static_cast<std::size_t>(d)] && !no_smem[static_cast<std::size_t>(d)])
            o << ind << at(d, "u", q, 0) << " = " << v << ";\n";
        }
      if (L.reduce_op != OOC_RED_NONE)  // fast rows are owned rows (see s_lo / s_hi)
        for (int r = 0; r < K; ++r)
          o << ind << "if (own_col) racc = ooc_red(" << L.reduce_op << ", racc, "
            << outs[static_cast<std::size_t>(r)][static_cast<std::size_t>(L.nwrites)] << ");\n";
    }
    for (int d = 0; d < nd; ++d) {
      const SwDs& D = pl.D[static_cast<std::size_t>(d)];
      if (!D.store) continue;
      const std::string ds = std::to_string(d);
      if (!pl.bulk_st) o << ind << "if (own_col) {\n";
      for (int r = 0; r < K; ++r) {
        auto it = forward && last_writer[static_cast<std::size_t>(d)] >= 0 &&
                          pl.L[static_cast<std::size_t>(last_writer[static_cast<std::size_t>(d)])].lag == D.lagS
                      ? cache.find(std::make_tuple(d, static_cast<long long>(r) - D.lagS, 0LL))
                      : cache.end();
        if (it == cache.end() && info) info->miss[static_cast<std::size_t>(d)] = 1;
        const std::string v = it != cache.end() ? it->second : at(d, "u", r - D.lagS, 0);
        if (pl.bulk_st) {
          // the final row goes to its ring slot (if only in a register); the producer copies
          // the aligned owned columns out after the next step barrier
          if (it != cache.end()) o << ind << at(d, "u", r - D.lagS, 0) << " = " << v << ";\n";
          o << ind << "if (stedge & (1u << " << d << ")) gs" << ds << "[" << r << " * p.s0[" << ds << "]] = " << v << ";\n";
        } else {
          o << ind << "  gs" << ds << "[" << r << " * p.s0[" << ds << "]] = " << v << ";\n";
        }
      }
      if (!pl.bulk_st) o << ind << "}\n";
    }
    bool any_store = false;
    for (const SwDs& D : pl.D) any_store = any_store || D.store;
    if (pl.bulk_st && any_store)  // generic-proxy ring writes before the producer's async-proxy reads
      o << ind << "asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n";
    if (info) info->end = cache;
    for (const auto& [k, name] : carries) {  // parallel assignment: sources may be carries
      auto it = cache.find(std::make_tuple(std::get<0>(k), std::get<1>(k) + K, 0LL));
      o << ind << "const double n" << name << " = " << it->second << ";\n";
    }
    for (const auto& [k, name] : carries) o << ind << name << " = n" << name << ";\n";
    bool spill = false;
    for (const auto& [k, name] : carries) spill = spill || no_smem[static_cast<std::size_t>(std::get<0>(k))];
    if (spill) {  // the next step is predicated: it reads these rows from the rings
      o << ind << "if (s + 1 == s_hi) {\n";
      for (const auto& [k, name] : carries)
        if (no_smem[static_cast<std::size_t>(std::get<0>(k))])
          o << ind << "  " << at(std::get<0>(k), "u + " + std::to_string(K), std::get<1>(k), 0) << " = " << name << ";\n";
      o << ind << "}\n";
    }
    o << ind << "prev_fast = true;\n";
  };
  static const bool skip_stores = !(std::getenv("OOC_SWEEP_NOSMEM") && std::atoi(std::getenv("OOC_SWEEP_NOSMEM")) == 0);
  if (forward) {  // discarded passes: carries to a fixpoint (a carried key stays cached, so
                  // it can feed the next step's carry), then the ring-free datasets
    FastInfo info;
    for (int iter = 0; iter < 8; ++iter) {
      info = FastInfo{};
      std::ostringstream keep;
      std::swap(o, keep);
      fast_body(&info, "s * " + std::to_string(K));
      std::swap(o, keep);
      std::vector<Key> next;
      for (const Key& k : info.first_read)
        if (info.end.count(std::make_tuple(std::get<0>(k), std::get<1>(k) + K, 0LL))) next.push_back(k);
      std::vector<Key> cur;
      for (const auto& [k, name] : carries) cur.push_back(k);
      if (next == cur) break;
      carries.clear();
      for (const Key& k : next) carries.push_back({k, "cr" + std::to_string(carries.size())});
    }
    if (skip_stores)
      for (int d = 0; d < nd; ++d)
        no_smem[static_cast<std::size_t>(d)] = pl.D[static_cast<std::size_t>(d)].written && !info.miss[static_cast<std::size_t>(d)];
  }
  for (const auto& [k, name] : carries) o << "  double " << name << " = 0.0;\n";
  o << "  bool prev_fast = false;\n";
  auto body = [&](bool fast) {
    const char* ind = "      ";
    loads("s + " + std::to_string(pl.P), ind, fast, true);
    o << ind << "const int u = s * " << K << ";\n";
    int ci = ci0;
    for (int i = 0; i < pl.n; ++i) {
      const ooc_loop& L = Ls[i];
      const SwLoop& S = pl.L[static_cast<std::size_t>(i)];
      if (S.barrier) o << ind << cbar << "\n";
      const std::string is = std::to_string(i);
      if (fast)
        o << ind << "{  // loop " << i << " (lag " << S.lag << ", halo " << S.h << ")\n";
      else
        o << ind << "if (colmask & (1ull << " << i << ")) {  // loop " << i << " (lag " << S.lag << ", halo " << S.h
          << ")\n";
      o << "#pragma unroll\n" << ind << "  for (int r = 0; r < " << K << "; ++r) {\n";
      if (!fast) {
        o << ind << "    const long long row = rbase + u + r - " << S.lag << ";\n";
        o << ind << "    if (row >= p.rng[" << is << "][0] && row < p.rng[" << is << "][1]) {\n";
      } else {
        o << ind << "    {\n";
      }
      int dsof_arg[OOC_MAX_ARGS];
      for (int a = 0; a < L.nargs; ++a) {
        dsof_arg[a] = -1;
        for (int d = 0; d < nd; ++d)
          if (pl.D[static_cast<std::size_t>(d)].v->data == L.args[a].data) dsof_arg[a] = d;
      }
      const std::string ur = "u + r - " + std::to_string(S.lag);
      int tmp = 0;
      std::vector<std::string> outs;
      const ooc_ins* t = L.tape;
      for (int w = 0; w < L.nwrites + (L.reduce_op != OOC_RED_NONE ? 1 : 0); ++w) {
        std::vector<std::string> st;
        for (int k = 0; k < (w < L.nwrites ? L.write_len[w] : L.reduce_len); ++k, ++t) {
          const ooc_ins& in = *t;
          if (in.op == OOC_OP_CONST) {
            if (cst && !fast) cst->push_back(in.value);
            st.push_back("p.cst[" + std::to_string(ci++) + "]");
          } else if (in.op == OOC_OP_READ) {
            const std::string name = "v" + is + "_" + std::to_string(tmp++);
            o << ind << "      const double " << name << " = " << at(dsof_arg[in.arg], ur, in.offset[0], xoff(in))
              << ";\n";
            st.push_back(name);
          } else {
            const std::string y = st.back();
            st.pop_back();
            const std::string x = st.back();
            st.pop_back();
            const std::string name = "v" + is + "_" + std::to_string(tmp++);
            o << ind << "      const double " << name << " = ";
            switch (in.op) {
              case OOC_OP_ADD: o << x << " + " << y; break;
              case OOC_OP_SUB: o << x << " - " << y; break;
              case OOC_OP_MUL: o << x << " * " << y; break;
              case OOC_OP_DIV: o << x << " / " << y; break;
              case OOC_OP_MIN: o << "ooc_min(" << x << ", " << y << ")"; break;
              default: o << "ooc_max(" << x << ", " << y << ")"; break;
            }
            o << ";\n";
            st.push_back(name);
          }
        }
        outs.push_back(st.back());
      }
      for (int w = 0; w < L.nwrites; ++w)
        o << ind << "      " << at(S.wds[static_cast<std::size_t>(w)], ur, 0, 0) << " = "
          << outs[static_cast<std::size_t>(w)] << ";\n";
      if (L.reduce_op != OOC_RED_NONE)
        o << ind << "      if (own_col && row >= r_own0 && row < r_own1) racc = ooc_red(" << L.reduce_op << ", racc, "
          << outs[static_cast<std::size_t>(L.nwrites)] << ");\n";
      o << ind << "    }\n" << ind << "  }\n" << ind << "}\n";
    }
    // stores of the final rows (each thread stores the elements it wrote: no barrier)
    for (int d = 0; d < nd; ++d) {
      const SwDs& D = pl.D[static_cast<std::size_t>(d)];
      if (!D.store) continue;
      const std::string ds = std::to_string(d);
      o << ind << "if (" << (fast ? std::string("own_col") : "stmask & (1u << " + ds + ")") << ") {\n#pragma unroll\n" << ind
        << "  for (int r = 0; r < " << K << "; ++r) {\n";
      if (!fast) {
        o << ind << "    const long long row = rbase + u + r - " << D.lagS << ";\n";
        o << ind << "    if (row >= r_own0 && row < r_own1 && row >= p.box[" << ds << "][0] && row < p.box[" << ds
          << "][1]";
        if (!D.oop) {
          o << " && (false";
          for (int j : D.writers)
            o << " || (row >= p.rng[" << j << "][0] && row < p.rng[" << j << "][1] && c >= p.rng[" << j
              << "][2] && c < p.rng[" << j << "][3]"
              << (d3 ? " && b >= p.rng[" + std::to_string(j) + "][4] && b < p.rng[" + std::to_string(j) + "][5]" : "") << ")";
          o << ")";
        }
        o << ")\n";
      }
      o << ind << "      gs" << ds << "[r * p.s0[" << ds << "]] = " << at(d, "u + r", -D.lagS, 0)
        << ";\n" << ind << "  }\n" << ind << "}\n";
    }
  };
  // Masked fast steps (column-edge strips, OOC_SWEEP_MASKED=0 disables): the general
  // body's semantics — every value through the rings, each loop under its column mask —
  // inside the fast row range, where every row predicate holds (s_lo / s_hi), with the K
  // rows unrolled at generation so an unrolled step's ring slots fold to constants.
  auto masked_body = [&](const std::string& uexpr) {
    const char* ind = "      ";
    o << ind << "const int u = " << uexpr << ";\n";
    int ci = ci0;
    for (int i = 0; i < pl.n; ++i) {
      const ooc_loop& L = Ls[i];
      const SwLoop& S = pl.L[static_cast<std::size_t>(i)];
      if (S.barrier) o << ind << cbar << "\n";
      const std::string is = std::to_string(i);
      o << ind << "if (colmask & (1ull << " << i << ")) {  // loop " << i << " (lag " << S.lag << ", halo " << S.h << ")\n";
      int dsof_arg[OOC_MAX_ARGS];
      for (int a = 0; a < L.nargs; ++a) {
        dsof_arg[a] = -1;
        for (int d = 0; d < nd; ++d)
          if (pl.D[static_cast<std::size_t>(d)].v->data == L.args[a].data) dsof_arg[a] = d;
      }
      std::vector<std::vector<std::string>> outs(static_cast<std::size_t>(K));
      const int ci_loop = ci;
      for (int r = 0; r < K; ++r) {
        ci = ci_loop;
        const long long q0 = r - S.lag;
        int tmp = 0;
        const ooc_ins* t = L.tape;
        const std::string pre = "m" + is + "_" + std::to_string(r) + "_";
        for (int w = 0; w < L.nwrites + (L.reduce_op != OOC_RED_NONE ? 1 : 0); ++w) {
          std::vector<std::string> st;
          for (int k = 0; k < (w < L.nwrites ? L.write_len[w] : L.reduce_len); ++k, ++t) {
            const ooc_ins& in = *t;
            if (in.op == OOC_OP_CONST) {
              st.push_back("p.cst[" + std::to_string(ci++) + "]");
            } else if (in.op == OOC_OP_READ) {
              const std::string name = pre + std::to_string(tmp++);
              o << ind << "  const double " << name << " = " << at(dsof_arg[in.arg], "u", q0 + in.offset[0], xoff(in)) << ";\n";
              st.push_back(name);
            } else {
              const std::string y = st.back();
              st.pop_back();
              const std::string x = st.back();
              st.pop_back();
              const std::string name = pre + std::to_string(tmp++);
              o << ind << "  const double " << name << " = ";
              switch (in.op) {
                case OOC_OP_ADD: o << x << " + " << y; break;
                case OOC_OP_SUB: o << x << " - " << y; break;
                case OOC_OP_MUL: o << x << " * " << y; break;
                case OOC_OP_DIV: o << x << " / " << y; break;
                case OOC_OP_MIN: o << "ooc_min(" << x << ", " << y << ")"; break;
                default: o << "ooc_max(" << x << ", " << y << ")"; break;
              }
              o << ";\n";
              st.push_back(name);
            }
          }
          outs[static_cast<std::size_t>(r)].push_back(st.back());
        }
      }
      for (int r = 0; r < K; ++r) {  // writes after every row's tapes (as in the general body)
        for (int w = 0; w < L.nwrites; ++w)
          o << ind << "  " << at(S.wds[static_cast<std::size_t>(w)], "u", r - S.lag, 0) << " = "
            << outs[static_cast<std::size_t>(r)][static_cast<std::size_t>(w)] << ";\n";
        if (L.reduce_op != OOC_RED_NONE)
          o << ind << "  if (own_col) racc = ooc_red(" << L.reduce_op << ", racc, "
            << outs[static_cast<std::size_t>(r)][static_cast<std::size_t>(L.nwrites)] << ");\n";
      }
      o << ind << "}\n";
    }
    for (int d = 0; d < nd; ++d) {  // final rows: owned, inside the box (fast row range)
      const SwDs& D = pl.D[static_cast<std::size_t>(d)];
      if (!D.store) continue;
      const std::string ds = std::to_string(d);
      o << ind << "if ((stmask & (1u << " << ds << "))";
      if (!D.oop) {
        o << " && (false";
        for (int j : D.writers)
          o << " || (c >= p.rng[" << j << "][2] && c < p.rng[" << j << "][3]"
            << (d3 ? " && b >= p.rng[" + std::to_string(j) + "][4] && b < p.rng[" + std::to_string(j) + "][5]" : "") << ")";
        o << ")";
      }
      o << ") {\n";
      for (int r = 0; r < K; ++r)
        o << ind << "  gs" << ds << "[" << r << " * p.s0[" << ds << "]] = " << at(d, "u", r - D.lagS, 0) << ";\n";
      o << ind << "}\n";
    }
    o << ind << "prev_fast = false;\n";
  };
  auto step_top = [&](const std::string& ind, long long j = -1) {
    if (pl.tma && j >= 0) {  // unrolled step j of a period block (U == NB): constant barrier
      o << ind << "sw_wait(sw_saddr(sw_bar) + " << (j % pl.NB) * 8 << "u, static_cast<unsigned>(sbl & 1));\n";
      o << ind << "__syncthreads();\n";
    } else if (pl.tma) {
      o << ind << "sw_wait(sw_saddr(sw_bar) + static_cast<unsigned>((s % " << pl.NB << ") * 8), static_cast<unsigned>((s / "
        << pl.NB << ") & 1));\n";
      o << ind << "__syncthreads();\n";
    } else {
      o << ind << "asm volatile(\"cp.async.wait_group " << pl.P - 1 << ";\" ::: \"memory\");\n";
      o << ind << "__syncthreads();\n";
    }
  };
  auto advance = [&](const std::string& ind) {
    for (int d = 0; d < nd; ++d) {
      const SwDs& D = pl.D[static_cast<std::size_t>(d)];
      if (D.loaded && !pl.tma) o << ind << "gl" << d << " += " << K << " * p.s0[" << d << "];\n";
      if (D.store) o << ind << "gs" << d << " += " << K << " * p.s0[" << d << "];\n";
    }
  };
  // Unrolled fast steps: U consecutive steps starting at a multiple of U, U a power of
  // two >= every ring length (and >= the 8 load barriers). Every ring slot
  // ((u + q) & (W - 1)) and barrier index then folds to a constant, so the interior
  // sweep addresses shared memory with immediate offsets instead of per-step slot
  // arithmetic (OOC_SWEEP_UNROLL=0 disables).
  static const int unroll_env = [] {
    const char* e = std::getenv("OOC_SWEEP_UNROLL");
    return e ? std::atoi(e) : 1;
  }();
  long long U = pl.U;  // ring period (every ring length divides it; == NB with TMA)
  if (unroll_env == 0 || U > 24 || (pl.tma && U != pl.NB)) U = 0;
  o << "  for (int s = 0; s < nsteps;) {\n";
  if (U > 1) {
    o << "    if (strip_in && s % " << U << " == 0 && s >= s_lo && s + " << U << " <= s_hi) {\n";
    o << "      const int sbl = s / " << U << ";\n";
    for (long long j = 0; j < U; ++j) {
      o << "      {  // unrolled fast step " << j << "\n";
      o << "        const int s = sbl * " << U << " + " << j << ";\n";
      step_top("        ", j);
      o << "        {\n";
      unroll_u = j * K;
      fast_body(nullptr, "(sbl * " + std::to_string(U) + " + " + std::to_string(j) + ") * " + std::to_string(K));
      unroll_u = -1;
      o << "        }\n";
      advance("        ");
      o << "      }\n";
    }
    o << "      s += " << U << ";\n      continue;\n    }\n";
    // OOC_SWEEP_MASKED: 0 general body on edge strips, 1 (default) unrolled masked steps
    // in 2-D and compact ones in 3-D, 2 compact masked steps in both
    static const int masked_mode = std::getenv("OOC_SWEEP_MASKED") ? std::atoi(std::getenv("OOC_SWEEP_MASKED")) : 1;
    const bool masked_env = masked_mode == 1;
    // 2-D only: on the 3-D plane tiles the extra unrolled body cost the interior CTAs
    // more than it saved on the edge tiles (miniflow3d 600^3: 4.61 vs 4.31 ms per timestep)
    if (masked_env && !pl.bulk_st && pl.nd == 2) {
      o << "    if (!strip_in && s % " << U << " == 0 && s >= s_lo && s + " << U << " <= s_hi) {\n";
      o << "      const int sbl = s / " << U << ";\n";
      for (long long j = 0; j < U; ++j) {
        o << "      {  // unrolled masked step " << j << "\n";
        o << "        const int s = sbl * " << U << " + " << j << ";\n";
        step_top("        ", j);
        o << "        {\n";
        unroll_u = j * K;
        masked_body("(sbl * " + std::to_string(U) + " + " + std::to_string(j) + ") * " + std::to_string(K));
        unroll_u = -1;
        o << "        }\n";
        advance("        ");
        o << "      }\n";
      }
      o << "      s += " << U << ";\n      continue;\n    }\n";
    }
  }
  step_top("    ");
  o << "    if (strip_in && s >= s_lo && s < s_hi) {\n";
  fast_body(nullptr, "s * " + std::to_string(K));
  // 3-D edge tiles: the masked steps without the unrolling (one compact copy of the loops,
  // dynamic ring slots, no row predicates) — the unrolled copy doubles the 3-D kernel's
  // code and slowed every CTA (OOC_SWEEP_MASKED=0 disables)
  static const int masked_mode1 = std::getenv("OOC_SWEEP_MASKED") ? std::atoi(std::getenv("OOC_SWEEP_MASKED")) : 1;
  if (((masked_mode1 == 1 && pl.nd == 3) || masked_mode1 == 2) && !pl.bulk_st) {
    o << "    } else if (s >= s_lo && s < s_hi) {\n";
    masked_body("s * " + std::to_string(K));
  }
  o << "    } else {\n";
  body(false);
  o << "      prev_fast = false;\n    }\n";
  advance("    ");
  o << "    ++s;\n  }\n";
  {
    bool any_store = false;
    for (const SwDs& D : pl.D) any_store = any_store || D.store;
    if (pl.bulk_st && any_store) o << "  __syncthreads();  // the producer copies out the last step's rows\n";
  }
  if (!pl.tma) o << "  asm volatile(\"cp.async.wait_group 0;\" ::: \"memory\");\n";
  if (pl.trace)
    o << "  if (threadIdx.x == 0) {\n    unsigned long long t_;\n"
         "    asm volatile(\"mov.u64 %0, %%globaltimer;\" : \"=l\"(t_));\n"
         "    p.trace[3 * (static_cast<long long>(blockIdx.y) * gridDim.x + blockIdx.x) + 2] = t_;\n  }\n";
  if (pl.red_op != OOC_RED_NONE) {  // warp tree, then the CTA's warps in order: one partial per CTA
    o << "#pragma unroll\n  for (int w = 16; w > 0; w >>= 1) racc = ooc_red(" << pl.red_op
      << ", racc, __shfl_down_sync(0xffffffffu, racc, w));\n";
    o << "  __shared__ double red_warp[" << NTc / 32 << "];\n";
    o << "  if ((threadIdx.x & 31) == 0) red_warp[threadIdx.x >> 5] = racc;\n  " << cbar << "\n";
    o << "  if (threadIdx.x == 0) {\n    double bsum = red_warp[0];\n";
    o << "    for (int w = 1; w < " << NTc / 32 << "; ++w) bsum = ooc_red(" << pl.red_op << ", bsum, red_warp[w]);\n";
    o << "    p.part[static_cast<long long>(blockIdx.y) * gridDim.x + blockIdx.x] = bsum;\n  }\n";
  }
  o << "}\n";
  return o.str();
}

struct SwKernel {
  void* fn = nullptr;
  int occ = 1;
  bool ok = false;
  std::string err;
};
std::mutex g_sw_mu;

int sweep_K() {
  static int k = [] {
    const char* e = std::getenv("OOC_SWEEP_K");
    const int v = e ? std::atoi(e) : 1;
    return v == 1 || v == 2 || v == 4 || v == 8 ? v : 1;
  }();
  return k;
}
bool sweep_P_forced() { return std::getenv("OOC_SWEEP_P") != nullptr; }
int sweep_P() {
  static int pp = [] {
    const char* e = std::getenv("OOC_SWEEP_P");
    const int v = e ? std::atoi(e) : 3;
    return v >= 1 && v <= 4 ? v : 3;
  }();
  return pp;
}
// bulk-copy (TMA) loads: on unless OOC_SWEEP_TMA=0 (then per-thread cp.async)
bool sweep_tma() {
  static const bool t = !(std::getenv("OOC_SWEEP_TMA") && std::atoi(std::getenv("OOC_SWEEP_TMA")) == 0);
  return t;
}

// ---- structural key of a run: everything analyze() and generate() depend on — loop
// ranges, each argument's dataset identity (first-seen order of view pointers) and view
// box, the tapes without constant values, the dead datasets — hashed to 128 bits, so a
// launch of a known structure does no analysis, code generation or string hashing.
struct Key128 {
  std::uint64_t a = 0, b = 0;
  bool operator==(const Key128& o) const { return a == o.a && b == o.b; }
};
struct Key128Hash {
  std::size_t operator()(const Key128& k) const { return static_cast<std::size_t>(k.a ^ (k.b * 0x9E3779B97F4A7C15ull)); }
};
struct KeyMix {
  std::uint64_t a = 1469598103934665603ull, b = 0x6a09e667f3bcc909ull;
  void put(long long v) {
    const std::uint64_t x = static_cast<std::uint64_t>(v);
    a = (a ^ x) * 1099511628211ull;
    b ^= x + 0x9E3779B97F4A7C15ull + (b << 6) + (b >> 2);
    b *= 0xff51afd7ed558ccdull;
  }
};
// tma_ok: every view 16-byte aligned with an even row stride (bulk-copy requirement)
Key128 run_key(const ooc_loop* Ls, int n, const ooc_redirect* red, int nred, bool with_dead, bool* tma_ok) {
  KeyMix m;
  const double* ids[2 * SW_MAXD];
  int nids = 0;
  bool al = true;
  auto id_of = [&](const double* p) {
    for (int k = 0; k < nids; ++k)
      if (ids[k] == p) return k;
    if (nids < 2 * SW_MAXD) ids[nids++] = p;
    return nids - 1;
  };
  m.put(n);
  m.put(ring_cols());
  for (int i = 0; i < n; ++i) {
    const ooc_loop& L = Ls[i];
    m.put(L.ndim);
    for (int k = 0; k < 3; ++k) {
      m.put(L.lo[k]);
      m.put(L.hi[k]);
    }
    m.put(L.nargs);
    for (int a = 0; a < L.nargs && a < OOC_MAX_ARGS; ++a) {
      const ooc_view& v = L.args[a];
      m.put(id_of(v.data));
      for (int k = 0; k < 3; ++k) {
        m.put(v.lo[k]);
        m.put(v.hi[k]);
        m.put(v.stride[k]);
      }
      al = al && (reinterpret_cast<std::uintptr_t>(v.data) & 15) == 0 && (v.stride[0] & 1) == 0;
    }
    m.put(L.ntape);
    for (int t = 0; t < L.ntape; ++t) {
      const ooc_ins& in = L.tape[t];
      m.put(in.op);
      m.put(in.op == OOC_OP_CONST ? 0 : in.arg);
      m.put(in.offset[0]);
      m.put(in.offset[1]);
      m.put(in.offset[2]);
    }
    m.put(L.nwrites);
    for (int w = 0; w < L.nwrites && w < OOC_MAX_WRITES; ++w) {
      m.put(L.write_arg[w]);
      m.put(L.write_len[w]);
    }
    m.put(L.reduce_op);
    m.put(L.reduce_len);
  }
  if (with_dead)
    for (int r = 0; r < nred; ++r)
      if (!red[r].dst) m.put(1000 + id_of(red[r].src));
  const bool tma = al && sweep_tma();
  m.put(tma ? 1 : 0);
  if (tma_ok) *tma_ok = tma;
  return {m.a, m.b};
}

// One specialisation of a structure: a prefetch depth, its plan, source and kernel.
struct SwVar {
  int P = 0;
  SwPlan pl;
  SwKernel k;
  bool built = false;
};
// Prefetch-depth autotuning per structure: every depth whose rings fit the budget is
// timed on real launches (CUDA events, two rounds, the faster counts) and the fastest
// kept — the same scheme as the tile shapes of jit.cu.
struct SwTune {
  std::vector<int> cands;  // indexes into SwEntry::vars
  std::vector<float> ms;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
  std::vector<char> issued;
  int best = -1;
};
struct SwEntry {
  bool init = false, ok = false;
  std::string why;
  std::vector<std::pair<int, int>> first;  // per plan dataset: (loop, arg) of a view of it
  std::vector<SwVar> vars;
  int def = 0;  // the default / forced depth
  SwTune tune;
  int loops = 0;
  bool tma = false;
  std::size_t gen_hash = 0;  // hash of the kernel source at the default depth (generator version + structure)
};
std::unordered_map<Key128, SwEntry, Key128Hash> g_sw_entries;
// ooc_sweep_check results per structure (no dead-store information involved)
struct SwCheck {
  bool ok = false;
  std::vector<int> flags;
};
std::unordered_map<Key128, SwCheck, Key128Hash> g_sw_checks;

void rebind(SwPlan& pl, const std::vector<std::pair<int, int>>& first, const ooc_loop* Ls) {
  for (std::size_t d = 0; d < pl.D.size(); ++d) pl.D[d].v = &Ls[first[d].first].args[first[d].second];
}

bool init_entry(SwEntry& E, const ooc_loop* loops, int n, const ooc_redirect* red, int nred, bool tma) {
  E.init = true;
  E.loops = n;
  E.tma = tma;
  std::vector<const double*> dead;
  for (int r = 0; r < nred; ++r)
    if (!red[r].dst) dead.push_back(red[r].src);
  SwPlan pl;
  if (!analyze(loops, n, sweep_K(), sweep_P(), pl, &E.why, &dead, tma)) return E.ok = false;
  for (const SwDs& D : pl.D) {
    std::pair<int, int> f{-1, -1};
    for (int i = 0; i < n && f.first < 0; ++i)
      for (int a = 0; a < loops[i].nargs; ++a)
        if (&loops[i].args[a] == D.v) f = {i, a};
    if (f.first < 0) {
      E.why = "dataset view not found";
      return E.ok = false;
    }
    E.first.push_back(f);
  }
  {  // generator identity at a canonical depth (independent of tuning and OOC_SWEEP_P)
    SwPlan canon;
    if (analyze(loops, n, sweep_K(), 3, canon, nullptr, &dead, tma))
      E.gen_hash = std::hash<std::string>{}(generate(loops, canon, nullptr));
    else
      E.gen_hash = std::hash<std::string>{}(generate(loops, pl, nullptr));
  }
  if (sweep_P_forced()) {
    SwVar v;
    v.P = pl.P;
    v.pl = pl;
    E.vars.push_back(v);
    E.def = 0;
    E.tune.best = 0;
    E.tune.cands = {0};
    E.tune.ms = {0.f};
  } else {
    for (int P = 1; P <= 4; ++P) {
      SwVar v;
      v.P = P;
      if (P == pl.P) {
        v.pl = pl;
      } else if (!analyze(loops, n, sweep_K(), P, v.pl, nullptr, &dead, tma)) {
        continue;
      }
      if (P == pl.P) E.def = static_cast<int>(E.vars.size());
      E.vars.push_back(v);
    }
    for (int round = 0; round < 2; ++round)  // two timed launches per depth: the faster counts
      for (std::size_t i = 0; i < E.vars.size(); ++i) E.tune.cands.push_back(static_cast<int>(i));
    E.tune.ms.assign(E.tune.cands.size(), -1.f);
    E.tune.ev.assign(E.tune.cands.size(), {nullptr, nullptr});
    E.tune.issued.assign(E.tune.cands.size(), 0);
    if (E.vars.size() <= 1) E.tune.best = 0;
  }
  return E.ok = true;
}

void resolve_tuning(SwTune& T) {  // timings that finished since the last launch (no blocking)
  if (T.best >= 0) return;
  bool all = !T.cands.empty();
  for (std::size_t i = 0; i < T.cands.size(); ++i) {
    if (T.ms[i] < 0 && T.issued[i] && cudaEventQuery(T.ev[i].second) == cudaSuccess)
      cudaEventElapsedTime(&T.ms[i], T.ev[i].first, T.ev[i].second);
    all = all && T.ms[i] >= 0;
  }
  if (all) {
    T.best = 0;
    for (std::size_t i = 1; i < T.ms.size(); ++i)
      if (T.ms[i] < T.ms[static_cast<std::size_t>(T.best)]) T.best = static_cast<int>(i);
  }
}

}  // namespace

extern "C" int ooc_sweep_3d_enabled(void) { return sweep_3d_enabled() ? 1 : 0; }

extern "C" void ooc_sweep_set_3d(int on) {
  std::lock_guard<std::mutex> lk(g_sw_mu);
  g_sweep3d = on ? 1 : 0;
  g_sw_checks.clear();  // cached verdicts depend on it
}

extern "C" int ooc_sweep_check(const ooc_loop* loops, int n, int* oop_args) {
  OOC_ARG_CHECK(loops && n > 0, "ooc_sweep_check: bad args");
  // same policy as the specialised kernels: off with OOC_JIT=0 (interpreter only), and
  // only for launches of >= the JIT threshold unless specialisation is forced
  long long min_pts = 0;
  const int m = jit_policy(&min_pts);
  if (m == 0) return 0;
  if (m == 1 && static_cast<long long>(loops[0].hi[0] - loops[0].lo[0]) * (loops[0].hi[1] - loops[0].lo[1]) *
                        std::max<long long>(1, loops[0].hi[2] - loops[0].lo[2]) <
                    min_pts)
    return 0;
  bool tma = false;
  const Key128 key = run_key(loops, n, nullptr, 0, false, &tma);
  std::lock_guard<std::mutex> lk(g_sw_mu);
  auto it = g_sw_checks.find(key);
  if (it == g_sw_checks.end()) {
    SwCheck ck;
    SwPlan pl;
    std::string why;
    ck.ok = analyze(loops, n, sweep_K(), sweep_P(), pl, &why, nullptr, tma);
    static const bool dbg = std::getenv("OOC_SWEEP_DEBUG") != nullptr;
    if (dbg && !ck.ok && n > 1) std::fprintf(stderr, "sweep: %d loops rejected: %s\n", n, why.c_str());
    if (ck.ok) {
      ck.flags.assign(static_cast<std::size_t>(n) * OOC_MAX_ARGS, 0);
      for (int i = 0; i < n; ++i)
        for (int a = 0; a < loops[i].nargs && a < OOC_MAX_ARGS; ++a)
          for (const SwDs& D : pl.D)
            if (D.v->data == loops[i].args[a].data)
              ck.flags[static_cast<std::size_t>(i) * OOC_MAX_ARGS + a] = (D.oop ? 1 : 0) | (D.loaded ? 2 : 0) | (D.written ? 4 : 0);
    }
    it = g_sw_checks.emplace(key, std::move(ck)).first;
  }
  if (!it->second.ok) return 0;
  if (oop_args) std::memcpy(oop_args, it->second.flags.data(), it->second.flags.size() * sizeof(int));
  return 1;
}

extern "C" int ooc_sweep_describe(const ooc_loop* loops, int n, const ooc_redirect* red, int nred, char* log,
                                  int len, int compile) {
  OOC_ARG_CHECK(loops && n > 0 && (red || nred == 0), "ooc_sweep_describe: bad args");
  SwPlan pl;
  std::string why;
  bool tma = false;
  run_key(loops, n, nullptr, 0, false, &tma);
  std::vector<const double*> dead;
  for (int r = 0; r < nred; ++r)
    if (!red[r].dst) dead.push_back(red[r].src);
  if (!analyze(loops, n, sweep_K(), sweep_P(), pl, &why, &dead, tma)) {
    if (log && len > 0) std::snprintf(log, static_cast<size_t>(len), "%s", why.c_str());
    return OOC_ERR_UNSUPPORTED;
  }
  std::ostringstream o;
  o << "{\"loops\":" << n << ",\"K\":" << pl.K << ",\"P\":" << pl.P << ",\"tma\":" << (pl.tma ? 1 : 0)
    << ",\"HC\":" << pl.HC << ",\"TC\":" << pl.TC << ",\"warm\":" << pl.warm << ",\"smem\":" << pl.smem << ",\"lags\":[";
  for (int i = 0; i < n; ++i) o << (i ? "," : "") << pl.L[static_cast<std::size_t>(i)].lag;
  o << "],\"halos\":[";
  for (int i = 0; i < n; ++i) o << (i ? "," : "") << pl.L[static_cast<std::size_t>(i)].h;
  o << "],\"barriers\":[";
  for (int i = 0; i < n; ++i) o << (i ? "," : "") << (pl.L[static_cast<std::size_t>(i)].barrier ? 1 : 0);
  o << "],\"datasets\":[";
  for (std::size_t d = 0; d < pl.D.size(); ++d) {
    const SwDs& D = pl.D[d];
    o << (d ? "," : "") << "{\"loaded\":" << D.loaded << ",\"written\":" << D.written << ",\"oop\":" << D.oop
      << ",\"store\":" << D.store << ",\"lagL\":" << D.lagL << ",\"lagS\":" << D.lagS << ",\"W\":" << D.W
      << ",\"rows\":" << D.need << "}";
  }
  // compulsory DRAM bytes of one launch: loaded arrays over the rows the sweep visits,
  // live outputs over what the kernel stores (out of place: the whole launch box)
  long long loaded = 0, stored = 0;
  for (const SwDs& D : pl.D) {
    const ooc_view& v = *D.v;
    // extent of the view across the non-row dimensions (2-D: columns; 3-D: dim 1 x dim 2)
    long long plane = 1;
    for (int k = 1; k < pl.nd; ++k) plane *= v.hi[k] - v.lo[k];
    if (D.loaded) {
      const long long r0 = std::max<long long>(v.lo[0], pl.box[0] - pl.warm), r1 = std::min<long long>(v.hi[0], pl.box[1]);
      loaded += std::max<long long>(0, r1 - r0) * plane * 8;
    }
    if (D.store) {
      long long lo[3] = {pl.box[0], 0, 0}, hi[3] = {pl.box[1], 1, 1};
      if (pl.nd == 2) {
        lo[1] = pl.box[2];
        hi[1] = pl.box[3];
      } else {
        lo[1] = pl.box[4];
        hi[1] = pl.box[5];
        lo[2] = pl.box[2];
        hi[2] = pl.box[3];
      }
      if (!D.oop) {  // in place: the writers' ranges
        for (int k = 0; k < 3; ++k) {
          lo[k] = LLONG_MAX;
          hi[k] = LLONG_MIN;
        }
        for (int j : D.writers)
          for (int k = 0; k < 3; ++k) {
            lo[k] = std::min<long long>(lo[k], loops[j].lo[k]);
            hi[k] = std::max<long long>(hi[k], loops[j].hi[k]);
          }
      }
      long long pts = 1;
      for (int k = 0; k < pl.nd; ++k) pts *= std::max<long long>(0, std::min<long long>(hi[k], v.hi[k]) - std::max<long long>(lo[k], v.lo[k]));
      stored += pts * 8;
    }
  }
  o << "],\"dram_bytes\":{\"loaded\":" << loaded << ",\"stored\":" << stored << "}}";
  std::string out = o.str();
  if (compile) {
    const std::string src = generate(loops, pl, nullptr);
    std::string err;
    if (!jit_build_kernel(src, "ooc_sweep_kernel", pl.NT, pl.smem, nullptr, nullptr, err, /*load=*/false)) {
      if (log && len > 0) std::snprintf(log, static_cast<size_t>(len), "%s", err.c_str());
      return OOC_ERR_UNSUPPORTED;
    }
    if (const char* f = std::getenv("OOC_SWEEP_DUMP")) {  // generated source + ptxas report
      static int ndump = 0;  // "%d" in the name: one file per described run
      char name[512];
      std::snprintf(name, sizeof name, f, ndump++);
      if (FILE* fp = std::fopen(name, "w")) {
        std::fprintf(fp, "%s\n/* %s */\n", src.c_str(), err.c_str());
        std::fclose(fp);
      }
    }
  }
  if (log && len > 0) std::snprintf(log, static_cast<size_t>(len), "%s", out.c_str());
  return OOC_OK;
}

extern "C" int ooc_sweep_report(char* buf, int len) {
  std::lock_guard<std::mutex> lk(g_sw_mu);
  std::ostringstream o;
  o << "[";
  bool first = true;
  for (auto& [key, E] : g_sw_entries) {
    if (!E.ok) continue;
    SwTune& T = E.tune;
    resolve_tuning(T);
    const int best = T.best >= 0 ? T.cands[static_cast<std::size_t>(T.best)] : -1;
    o << (first ? "" : ",") << "{\"loops\":" << E.loops << ",\"key\":\"" << std::hex << key.a << std::dec
      << "\",\"gen_hash\":\"" << std::hex << E.gen_hash << std::dec
      << "\",\"tma\":" << (E.tma ? 1 : 0) << ",\"P\":" << (best >= 0 ? E.vars[static_cast<std::size_t>(best)].P : -1)
      << ",\"smem\":" << (best >= 0 ? E.vars[static_cast<std::size_t>(best)].pl.smem : -1)
      << ",\"occ\":" << (best >= 0 ? E.vars[static_cast<std::size_t>(best)].k.occ : -1) << ",\"ms\":[";
    for (std::size_t i = 0; i < T.cands.size(); ++i)
      o << (i ? "," : "") << "[" << E.vars[static_cast<std::size_t>(T.cands[i])].P << "," << T.ms[i] << "]";
    o << "]}";
    first = false;
  }
  o << "]";
  std::snprintf(buf, static_cast<size_t>(len), "%s", o.str().c_str());
  return OOC_OK;
}

extern "C" int ooc_launch_sweep(ooc_ctx* c, int q, const ooc_loop* loops, int n, const ooc_redirect* red,
                                int nred) {
  OOC_ARG_CHECK(c && loops && n > 0 && q >= 0 && q < OOC_NUM_QUEUES, "ooc_launch_sweep: bad args");
  if (c->red_exact && loops[n - 1].reduce_op != OOC_RED_NONE) {
    set_error("ooc_launch_sweep: exact reductions fold through ooc_launch_group, not in a sweep");
    return OOC_ERR_UNSUPPORTED;
  }
  const auto host0 = std::chrono::steady_clock::now();
  bool tma = false;
  const Key128 key = run_key(loops, n, red, nred, true, &tma);
  std::unique_lock<std::mutex> lk(g_sw_mu);
  SwEntry& E = g_sw_entries[key];
  if (!E.init) init_entry(E, loops, n, red, nred, tma);
  if (!E.ok) {
    set_error("ooc_launch_sweep: group not sweepable: " + E.why);
    return OOC_ERR_UNSUPPORTED;
  }
  // ---- prefetch depth: forced (OOC_SWEEP_P), tuned, or being tuned on this launch
  SwTune& T = E.tune;
  int pick = -1;  // index into T.cands
  bool timing = false;
  resolve_tuning(T);
  if (T.best >= 0) {
    pick = T.best;
  } else {
    c->stats.jit_unsettled++;
    for (std::size_t i = 0; i < T.cands.size() && pick < 0 && !g_frozen; ++i)
      if (!T.issued[i]) pick = static_cast<int>(i);
    timing = pick >= 0;
    if (pick < 0)  // frozen for a graph capture, or all in flight: fastest measured so far
      for (std::size_t i = 0; i < T.cands.size(); ++i)
        if (T.ms[i] >= 0 && (pick < 0 || T.ms[i] < T.ms[static_cast<std::size_t>(pick)])) pick = static_cast<int>(i);
    if (pick < 0) {  // nothing measured yet: the default depth, untimed
      for (std::size_t i = 0; i < T.cands.size() && pick < 0; ++i)
        if (T.cands[i] == E.def) pick = static_cast<int>(i);
    }
  }
  SwVar& V = E.vars[static_cast<std::size_t>(T.cands[static_cast<std::size_t>(pick)])];
  // test hook: every sweep kernel "fails to build", exercising the engine's fallback
  static const bool fail_build = std::getenv("OOC_SWEEP_FAIL_BUILD") != nullptr;
  if (fail_build) {
    set_error("ooc_launch_sweep: build disabled (OOC_SWEEP_FAIL_BUILD)");
    return OOC_ERR_UNSUPPORTED;
  }
  const SwPlan& pl = V.pl;
  long long build_us = 0;
  if (!V.built) {
    V.built = true;
    const auto b0 = std::chrono::steady_clock::now();
    rebind(V.pl, E.first, loops);
    const std::string src = generate(loops, V.pl, nullptr);
    const auto t0 = std::chrono::steady_clock::now();
    V.k.ok = jit_build_kernel(src, "ooc_sweep_kernel", pl.NT, pl.smem, &V.k.fn, &V.k.occ, V.k.err, true);
    c->stats.jit_compiles++;
    c->stats.jit_compile_ms +=
        std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count();
    if (!V.k.ok && V.k.err.empty()) V.k.err = "build failed";
    build_us = std::chrono::duration_cast<std::chrono::microseconds>(std::chrono::steady_clock::now() - b0).count();
  }
  if (!V.k.ok) {
    set_error("ooc_launch_sweep: " + V.k.err);
    return OOC_ERR_UNSUPPORTED;
  }
  SweepParams sp;  // ~6 KB, filled field by field (constants in tape order)
  int ci = 0;
  for (int i = 0; i < n; ++i)
    for (int t = 0; t < loops[i].ntape; ++t)
      if (loops[i].tape[t].op == OOC_OP_CONST) sp.cst[ci++] = loops[i].tape[t].value;
  sp.part = nullptr;
  sp.R0 = pl.box[0];
  sp.R1 = pl.box[1];
  sp.C0 = pl.box[2];
  sp.C1 = pl.box[3];
  sp.B0 = pl.box[4];
  sp.B1 = pl.box[5];
  const int dc = pl.nd - 1;  // column dimension of the loops and views
  for (int i = 0; i < n; ++i) {
    sp.rng[i][0] = loops[i].lo[0];
    sp.rng[i][1] = loops[i].hi[0];
    sp.rng[i][2] = loops[i].lo[dc];
    sp.rng[i][3] = loops[i].hi[dc];
    sp.rng[i][4] = pl.nd == 3 ? loops[i].lo[1] : 0;
    sp.rng[i][5] = pl.nd == 3 ? loops[i].hi[1] : 1;
  }
  for (std::size_t d = 0; d < pl.D.size(); ++d) {
    const SwDs& D = pl.D[d];
    const ooc_view& v = loops[E.first[d].first].args[E.first[d].second];
    sp.src[d] = v.data;
    sp.dst[d] = v.data;
    sp.s0[d] = v.stride[0];
    sp.s1[d] = pl.nd == 3 ? v.stride[1] : 0;
    sp.box[d][0] = v.lo[0];
    sp.box[d][1] = v.hi[0];
    sp.box[d][2] = v.lo[dc];
    sp.box[d][3] = v.hi[dc];
    sp.box[d][4] = pl.nd == 3 ? v.lo[1] : 0;
    sp.box[d][5] = pl.nd == 3 ? v.hi[1] : 1;
    if (D.oop && D.store) {
      double* to = nullptr;
      for (int r = 0; r < nred; ++r)
        if (red[r].src == v.data) to = red[r].dst;
      if (!to) {
        set_error("ooc_launch_sweep: no out-of-place destination for a dataset the group loads and writes");
        return OOC_ERR_ARG;
      }
      sp.dst[d] = to;
    }
  }
  const long long rows = pl.box[1] - pl.box[0];
  // CTA tiles: strips of TC columns (x ntb tiles of TB rows along dim 1 in 3-D)
  const long long ntc = (pl.box[3] - pl.box[2] + pl.TC - 1) / pl.TC;
  const long long strips = ntc * ((pl.box[5] - pl.box[4] + pl.TB - 1) / pl.TB);
  sp.ntc = ntc;
  // Row segments per strip: whole waves of CTAs (the grid is strips x segments; a
  // partial last wave idles SMs), at least ~4 waves, segments >= 8 warm-up depths.
  // A reducing run folds one partial per CTA in CTA order, so its partition must not
  // depend on the tuned depth or the occupancy it allows: it is planned for a fixed
  // 4 CTAs per SM and depth 2 (reductions are reproducible run to run, box to box).
  const bool red_run = pl.red_op != OOC_RED_NONE;
  const long long cap = static_cast<long long>(c->prop.multiProcessorCount) * (red_run ? 4 : V.k.occ);
  const long long depth_rows = (red_run ? 2 : pl.P) * pl.K;
  const long long min_seg = std::max<long long>(64, 8 * (pl.warm + pl.lagS_max + pl.K));
  const long long max_nseg = std::max<long long>(1, rows / min_seg);
  // Time model in swept rows per CTA slot: the work spread over the slots plus a tail of
  // about half a CTA (CTAs finish desynchronised: the edge strips' longer CTAs and the
  // shared DRAM stagger them — measured with OOC_SWEEP_TRACE), each CTA also sweeping its
  // warm-up / lag / prefetch rows without storing them.
  long long nseg = 1;
  double best = 1e300;
  const double overhead = static_cast<double>(pl.warm + pl.lagS_max + depth_rows) + 8.0;  // + pipeline fill
  static const long long force_nseg = [] {
    const char* e = std::getenv("OOC_SWEEP_NSEG");
    return e ? std::atoll(e) : 0LL;
  }();
  for (long long ns = 1; ns <= std::min<long long>(max_nseg, 4096); ++ns) {
    const long long seg = (rows + ns - 1) / ns, real = (rows + seg - 1) / seg, ctas = strips * real;
    if (red_run && ctas > c->red_part_cap) break;  // one partial per CTA
    const double per = static_cast<double>(seg) + overhead;
    const double t = static_cast<double>(ctas) * per / static_cast<double>(cap) + 0.5 * per +
                     (ctas < cap ? static_cast<double>(cap - ctas) * per / static_cast<double>(cap) : 0.0);
    if (t < best - 1e-9) {
      best = t;
      nseg = real;
    }
  }
  if (force_nseg > 0 && !red_run) nseg = std::min<long long>(force_nseg, std::max<long long>(1, rows));
  sp.seg_rows = (rows + nseg - 1) / nseg;
  nseg = (rows + sp.seg_rows - 1) / sp.seg_rows;
  static const bool edge_env = !(std::getenv("OOC_SWEEP_EDGEFIRST") && std::atoi(std::getenv("OOC_SWEEP_EDGEFIRST")) == 0);
  sp.edge_first = edge_env && ntc >= 3 ? 1 : 0;
  if (red_run) {
    if (strips * nseg > c->red_part_cap) {
      set_error("ooc_launch_sweep: too many CTAs for the reduction partials");
      return OOC_ERR_UNSUPPORTED;
    }
    sp.part = c->red_part[q];
  }
  // debug trace (OOC_SWEEP_TRACE): one buffer for the process, reallocated when a launch
  // needs more or runs on another device; each traced launch synchronises before returning
  static const char* trace_file = std::getenv("OOC_SWEEP_TRACE");
  static unsigned long long* trace_buf = nullptr;
  static long long trace_cap = 0;
  static int trace_dev = -1;
  const bool tracing = trace_file && pl.trace;
  if (tracing) {
    const long long need = 3 * strips * nseg;
    if (need > trace_cap || trace_dev != c->device) {
      trace_dev = c->device;
      cudaFree(trace_buf);
      OOC_CUDA_TRY(cudaMalloc(&trace_buf, need * sizeof(unsigned long long)));
      trace_cap = need;
    }
    sp.trace = trace_buf;
  }
  c->stats.sweep_launches++;
  // 3-D: one tiled tensor map per loaded dataset view (box = the RB x RCp plane tile)
  struct alignas(64) HostMaps {
    unsigned long long t[SW_MAXD][16];
  };
  HostMaps maps;
  std::memset(&maps, 0, sizeof maps);
  if (pl.nd == 3) {
    for (std::size_t d = 0; d < pl.D.size(); ++d) {
      if (!pl.D[d].loaded) continue;
      const ooc_view& v = loops[E.first[d].first].args[E.first[d].second];
      const unsigned long long gdim[3] = {static_cast<unsigned long long>(v.hi[2] - v.lo[2]),
                                          static_cast<unsigned long long>(v.hi[1] - v.lo[1]),
                                          static_cast<unsigned long long>(v.hi[0] - v.lo[0])};
      const unsigned long long gstr[2] = {static_cast<unsigned long long>(v.stride[1]) * 8,
                                          static_cast<unsigned long long>(v.stride[0]) * 8};
      const unsigned box[3] = {static_cast<unsigned>(pl.RCp), static_cast<unsigned>(pl.RB), 1u};
      if (!jit_tensor_map(&maps.t[d][0], 3, v.data, gdim, gstr, box)) {
        set_error("ooc_launch_sweep: cuTensorMapEncodeTiled rejected a 3-D view");
        return OOC_ERR_UNSUPPORTED;
      }
    }
  }
  void* args[] = {&sp, &maps};
  std::pair<cudaEvent_t, cudaEvent_t>* tev = nullptr;
  if (timing) {
    tev = &T.ev[static_cast<std::size_t>(pick)];
    if (!tev->first) {
      cudaEventCreate(&tev->first);
      cudaEventCreate(&tev->second);
    }
    cudaEventRecord(tev->first, c->q[q]);
  }
  const int rc = jit_launch_kernel(c, q, V.k.fn, static_cast<unsigned>(strips), static_cast<unsigned>(nseg),
                                   static_cast<unsigned>(pl.NT), static_cast<unsigned>(pl.smem), args);
  if (timing) {
    cudaEventRecord(tev->second, c->q[q]);
    T.issued[static_cast<std::size_t>(pick)] = 1;
  }
  if (tracing && rc == OOC_OK) {  // debug: append "launch cta sm start end" lines
    static int tl = 0;
    const long long nc = strips * nseg;
    std::vector<unsigned long long> h(static_cast<std::size_t>(3 * nc));
    OOC_CUDA_TRY(cudaStreamSynchronize(c->q[q]));
    OOC_CUDA_TRY(cudaMemcpy(h.data(), trace_buf, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    if (FILE* fp = std::fopen(trace_file, "a")) {
      std::fprintf(fp, "# launch %d loops %d grid %lld x %lld seg_rows %lld P %d\n", tl, n, strips, nseg,
                   sp.seg_rows, pl.P);
      for (long long i = 0; i < nc; ++i)
        std::fprintf(fp, "%d %lld %llu %llu %llu\n", tl, i, h[3 * i], h[3 * i + 1], h[3 * i + 2]);
      std::fclose(fp);
    }
    ++tl;
  }
  // host cost of the launch itself (key, lookup, parameters, launch): NVRTC builds excluded
  c->stats.sweep_host_us +=
      std::chrono::duration_cast<std::chrono::microseconds>(std::chrono::steady_clock::now() - host0).count() -
      build_us;
  lk.unlock();
  if (rc != OOC_OK || pl.red_op == OOC_RED_NONE) return rc;
  return launch_fold(c, q, static_cast<int>(strips * nseg), loops[n - 1].reduce_slot, pl.red_op);
}
