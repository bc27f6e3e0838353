// ooc-b200 core types: boxes, stencils, expressions, datasets, loops, chains.
//
// Source-compatible with the reference's OPS-style API (proj/include/ooc/*.hpp):
// the same names, argument meaning and error types, so loop chains written
// against the reference (e.g. proj/src/apps.cpp) compile and run unchanged.
// The storage behind Dataset::host is pinned host memory (PinnedAllocator) so
// the streaming engine's copies are true async DMA; everything else here is
// plain host-side bookkeeping consumed by the planner and the GPU executors.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstdlib>
#include <functional>
#include <limits>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace ooc {

using index_t = std::int64_t;
using Point = std::array<index_t, 3>;

// ---------------------------------------------------------------- errors
// (reference: proj/include/ooc/errors.hpp:9-47)
struct ValidationError : std::runtime_error {
  explicit ValidationError(const std::string& w) : std::runtime_error(w) {}
};
struct StaleDataError : std::runtime_error {
  std::string dataset;
  int discarded_by_chain;
  StaleDataError(std::string name, int chain)
      : std::runtime_error("stale data: dataset '" + name + "' was discarded by chain " +
                           std::to_string(chain) + " (cyclic execution); host values are invalid"),
        dataset(std::move(name)),
        discarded_by_chain(chain) {}
};
struct InfeasibleError : std::runtime_error {
  std::int64_t min_achievable_bytes;
  InfeasibleError(std::int64_t min_bytes, std::int64_t budget)
      : std::runtime_error("infeasible tiling: minimum achievable 3-slot size is " +
                           std::to_string(min_bytes) + " bytes, budget is " +
                           std::to_string(budget) + " bytes"),
        min_achievable_bytes(min_bytes) {}
};
struct CapacityError : std::runtime_error {
  std::int64_t required_bytes;
  CapacityError(std::int64_t required, std::int64_t capacity)
      : std::runtime_error("device capacity exceeded: 3-slot working set needs " +
                           std::to_string(required) + " bytes, capacity is " +
                           std::to_string(capacity) + " bytes"),
        required_bytes(required) {}
};
struct DeadlockError : std::runtime_error {
  explicit DeadlockError(const std::string& w) : std::runtime_error(w) {}
};
/// A CUDA / device-layer failure surfaced through the C ABI (include/ooc_device.h).
struct DeviceError : std::runtime_error {
  int code;
  DeviceError(int c, const std::string& w) : std::runtime_error(w), code(c) {}
};

// ---------------------------------------------------------------- boxes
// Half-open box of rank 1..3; unused trailing dims are [0,1).
// (reference semantics: proj/include/ooc/extent.hpp:14-138)
struct Extent {
  int ndim = 1;
  Point lo{0, 0, 0};
  Point hi{1, 1, 1};

  static Extent make(int nd, Point l, Point h) {
    Extent e;
    e.ndim = nd;
    for (int d = 0; d < 3; ++d) {
      e.lo[d] = d < nd ? l[d] : 0;
      e.hi[d] = d < nd ? h[d] : 1;
    }
    return e;
  }
  static Extent line(index_t l, index_t h) { return make(1, {l, 0, 0}, {h, 1, 1}); }
  static Extent rect(index_t l0, index_t h0, index_t l1, index_t h1) {
    return make(2, {l0, l1, 0}, {h0, h1, 1});
  }
  static Extent box(index_t l0, index_t h0, index_t l1, index_t h1, index_t l2, index_t h2) {
    return make(3, {l0, l1, l2}, {h0, h1, h2});
  }
  static Extent none(int nd) { return make(nd, {0, 0, 0}, {0, 0, 0}); }

  bool empty() const {
    for (int d = 0; d < ndim; ++d)
      if (hi[d] <= lo[d]) return true;
    return false;
  }
  index_t len(int d) const { return hi[d] - lo[d]; }
  index_t size() const {
    return empty() ? 0 : (hi[0] - lo[0]) * (hi[1] - lo[1]) * (hi[2] - lo[2]);
  }
  bool contains(const Point& p) const {
    return p[0] >= lo[0] && p[0] < hi[0] && p[1] >= lo[1] && p[1] < hi[1] && p[2] >= lo[2] &&
           p[2] < hi[2];
  }
  bool contains(const Extent& o) const {
    if (o.empty()) return true;
    for (int d = 0; d < 3; ++d)
      if (o.lo[d] < lo[d] || o.hi[d] > hi[d]) return false;
    return true;
  }
  Extent intersect(const Extent& o) const {
    Extent r = *this;
    for (int d = 0; d < 3; ++d) {
      r.lo[d] = lo[d] > o.lo[d] ? lo[d] : o.lo[d];
      r.hi[d] = hi[d] < o.hi[d] ? hi[d] : o.hi[d];
    }
    return r.empty() ? none(ndim) : r;
  }
  Extent hull(const Extent& o) const {
    if (empty()) return o;
    if (o.empty()) return *this;
    Extent r = *this;
    for (int d = 0; d < 3; ++d) {
      r.lo[d] = lo[d] < o.lo[d] ? lo[d] : o.lo[d];
      r.hi[d] = hi[d] > o.hi[d] ? hi[d] : o.hi[d];
    }
    return r;
  }
  Extent expand(const Point& lo_off, const Point& hi_off) const {
    Extent r = *this;
    for (int d = 0; d < ndim; ++d) {
      r.lo[d] += lo_off[d];
      r.hi[d] += hi_off[d];
    }
    return r;
  }
  Extent with_dim(int d, index_t l, index_t h) const {
    Extent r = *this;
    r.lo[d] = l;
    r.hi[d] = h;
    return r;
  }
  bool operator==(const Extent& o) const { return ndim == o.ndim && lo == o.lo && hi == o.hi; }
  bool operator!=(const Extent& o) const { return !(*this == o); }
  Point strides() const {
    Point s;
    s[2] = 1;
    s[1] = hi[2] - lo[2];
    s[0] = s[1] * (hi[1] - lo[1]);
    return s;
  }
  index_t flatten(const Point& p) const {
    Point s = strides();
    return (p[0] - lo[0]) * s[0] + (p[1] - lo[1]) * s[1] + (p[2] - lo[2]);
  }
  std::string str() const;
};

// ---------------------------------------------------------------- stencils
// (reference semantics: proj/include/ooc/stencil.hpp:13-64)
struct Stencil {
  std::vector<Point> offsets;

  static Stencil point() { return Stencil{{Point{0, 0, 0}}}; }
  static Stencil of(std::vector<Point> offs) { return Stencil{std::move(offs)}; }
  static Stencil line(int dim, index_t radius);
  static Stencil star(int ndim, index_t radius);
  bool is_point() const { return offsets.size() == 1 && offsets[0] == Point{0, 0, 0}; }
  bool has_offset(const Point& off) const {
    return std::find(offsets.begin(), offsets.end(), off) != offsets.end();
  }
};
std::pair<Point, Point> stencil_extents(const Stencil& s);

// ---------------------------------------------------------------- expressions
// (reference semantics: proj/include/ooc/expr.hpp:12-107, proj/src/expr.cpp)
enum class ExprOp : std::uint8_t { constant, read, coord, add, sub, mul, divide, min, max };
inline bool expr_op_is_binary(ExprOp op) {
  return op != ExprOp::constant && op != ExprOp::read && op != ExprOp::coord;
}

struct Expr;
using ExprPtr = std::shared_ptr<const Expr>;
struct Expr {
  ExprOp op = ExprOp::constant;
  double value = 0.0;
  int arg = 0;
  Point offset{0, 0, 0};
  ExprPtr lhs, rhs;
};

namespace ex {
ExprPtr c(double v);
ExprPtr r(int arg, index_t o0 = 0, index_t o1 = 0, index_t o2 = 0);
ExprPtr coord(int dim);
ExprPtr bin(ExprOp op, ExprPtr a, ExprPtr b);
inline ExprPtr add(ExprPtr a, ExprPtr b) { return bin(ExprOp::add, std::move(a), std::move(b)); }
inline ExprPtr sub(ExprPtr a, ExprPtr b) { return bin(ExprOp::sub, std::move(a), std::move(b)); }
inline ExprPtr mul(ExprPtr a, ExprPtr b) { return bin(ExprOp::mul, std::move(a), std::move(b)); }
inline ExprPtr div(ExprPtr a, ExprPtr b) { return bin(ExprOp::divide, std::move(a), std::move(b)); }
inline ExprPtr min(ExprPtr a, ExprPtr b) { return bin(ExprOp::min, std::move(a), std::move(b)); }
inline ExprPtr max(ExprPtr a, ExprPtr b) { return bin(ExprOp::max, std::move(a), std::move(b)); }
}  // namespace ex

/// Postfix program of one expression; `max_stack` is the evaluation depth.
struct ExprTape {
  struct Ins {
    ExprOp op;
    int arg;
    double value;
    Point offset;
  };
  std::vector<Ins> ins;
  int max_stack = 0;
  static ExprTape compile(const ExprPtr& e);
};

template <typename Fn>
void expr_visit(const ExprPtr& e, Fn&& fn) {
  if (!e) return;
  fn(*e);
  expr_visit(e->lhs, fn);
  expr_visit(e->rhs, fn);
}

ExprPtr parse_prefix_expr(const std::string& text, bool allow_coords = false);
std::string expr_to_string(const ExprPtr& e);

// ---------------------------------------------------------------- host storage
/// Page-locked host allocation for dataset storage (falls back to ordinary
/// aligned memory only when no CUDA device exists, e.g. planner-only CPU use).
/// Elements are default-initialised (no zeroing pass): declare_dataset writes
/// every element exactly once, in parallel.
void* pinned_host_alloc(std::size_t bytes);
void pinned_host_free(void* p) noexcept;

template <typename T>
struct PinnedAllocator {
  using value_type = T;
  PinnedAllocator() = default;
  template <typename U>
  PinnedAllocator(const PinnedAllocator<U>&) {}
  T* allocate(std::size_t n) { return static_cast<T*>(pinned_host_alloc(n * sizeof(T))); }
  void deallocate(T* p, std::size_t) noexcept { pinned_host_free(p); }
  template <typename U>
  void construct(U* p) noexcept {
    ::new (static_cast<void*>(p)) U;  // default-init: no zero pass over GBs
  }
  template <typename U, typename... A>
  void construct(U* p, A&&... a) {
    ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
  }
  template <typename U>
  bool operator==(const PinnedAllocator<U>&) const { return true; }
  template <typename U>
  bool operator!=(const PinnedAllocator<U>&) const { return false; }
};
using HostVector = std::vector<double, PinnedAllocator<double>>;

// ---------------------------------------------------------------- datasets
// (reference semantics: proj/include/ooc/dataset.hpp:13-73, proj/src/dataset.cpp:5-38)
using DatasetId = int;

struct Block {
  std::string name;
  int ndim = 0;
};

struct Dataset {
  std::string name;
  int block = 0;
  Extent core;
  Point halo{0, 0, 0};
  index_t elem_bytes = 8;
  HostVector host;

  bool host_stale = false;
  int stale_chain = -1;
  Extent stale_region = {};
  bool ever_written = false;

  Extent alloc() const {
    Extent a = core;
    for (int d = 0; d < a.ndim; ++d) {
      a.lo[d] -= halo[d];
      a.hi[d] += halo[d];
    }
    return a;
  }
  double& at(const Point& p) { return host[static_cast<std::size_t>(alloc().flatten(p))]; }
  double at(const Point& p) const { return host[static_cast<std::size_t>(alloc().flatten(p))]; }
};

struct Mesh {
  std::vector<Block> blocks{{"block", 0}};
  std::vector<Dataset> datasets;

  DatasetId find(const std::string& name) const {
    for (std::size_t i = 0; i < datasets.size(); ++i)
      if (datasets[i].name == name) return static_cast<DatasetId>(i);
    return -1;
  }
  Dataset& operator[](DatasetId id) { return datasets[static_cast<std::size_t>(id)]; }
  const Dataset& operator[](DatasetId id) const { return datasets[static_cast<std::size_t>(id)]; }
};

DatasetId declare_dataset(Mesh& mesh, const std::string& name, const Extent& core, Point halo,
                          index_t elem_bytes, const std::function<double(Point)>& fill);
DatasetId declare_dataset(Mesh& mesh, const std::string& name, const Extent& core, Point halo,
                          index_t elem_bytes, double fill_value);

// ---------------------------------------------------------------- loops
// (reference semantics: proj/include/ooc/loop.hpp:12-115, proj/src/loop.cpp:32-105)
enum class AccessMode { read, write, read_write };
inline bool access_reads(AccessMode m) { return m != AccessMode::write; }
inline bool access_writes(AccessMode m) { return m != AccessMode::read; }
inline const char* access_name(AccessMode m) {
  return m == AccessMode::read ? "READ" : m == AccessMode::write ? "WRITE" : "READ_WRITE";
}

struct LoopArg {
  DatasetId dataset;
  Stencil stencil;
  AccessMode mode;
};

enum class ReduceOp { none, sum, min, max };

struct KernelSpec {
  struct Write {
    int arg;
    ExprPtr expr;
  };
  std::vector<Write> writes;
  ReduceOp reduce = ReduceOp::none;
  ExprPtr reduce_expr;
  std::string reduce_name;
};

struct ParLoop {
  int id = -1;
  Extent range;
  std::vector<LoopArg> args;
  KernelSpec kernel;
  std::vector<ExprTape> write_tapes;
  ExprTape reduce_tape;

  bool has_reduction() const { return kernel.reduce != ReduceOp::none; }
  bool writes_dataset(DatasetId d) const {
    for (const auto& a : args)
      if (a.dataset == d && access_writes(a.mode)) return true;
    return false;
  }
  bool reads_dataset(DatasetId d) const {
    for (const auto& a : args)
      if (a.dataset == d && access_reads(a.mode)) return true;
    return false;
  }
};

void validate_loop(const Mesh& mesh, ParLoop& loop);

inline index_t loop_bytes_per_point(const Mesh& mesh, const ParLoop& loop) {
  index_t n = 0;
  for (const auto& a : loop.args)
    n += mesh[a.dataset].elem_bytes * (a.mode == AccessMode::read_write ? 2 : 1);
  return n;
}

inline double reduce_identity(ReduceOp op) {
  if (op == ReduceOp::min) return std::numeric_limits<double>::infinity();
  if (op == ReduceOp::max) return -std::numeric_limits<double>::infinity();
  return 0.0;
}
/// std::min / std::max semantics exactly: min(a,b) = (b<a)?b:a, max(a,b) = (a<b)?b:a.
inline double reduce_combine(ReduceOp op, double acc, double v) {
  switch (op) {
    case ReduceOp::sum:
      return acc + v;
    case ReduceOp::min:
      return v < acc ? v : acc;
    case ReduceOp::max:
      return acc < v ? v : acc;
    default:
      return acc;
  }
}

// ---------------------------------------------------------------- chains
// (reference semantics: proj/include/ooc/chain.hpp:9-29)
enum class FlushReason { reduction_fetch, data_fetch, explicit_flush, program_end };
inline const char* flush_reason_name(FlushReason r) {
  switch (r) {
    case FlushReason::reduction_fetch:
      return "REDUCTION_FETCH";
    case FlushReason::data_fetch:
      return "DATA_FETCH";
    case FlushReason::explicit_flush:
      return "EXPLICIT_FLUSH";
    default:
      return "PROGRAM_END";
  }
}

struct LoopChain {
  int chain_id = 0;
  std::vector<ParLoop> loops;
  FlushReason reason = FlushReason::program_end;
};

}  // namespace ooc
