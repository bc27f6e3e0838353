// ooc-b200 core: boxes, stencils, expression trees/tapes, datasets, loop validation.
// Semantics follow the reference file:line cited at each function.
#include <cctype>
#include <cstring>
#include <sstream>

#include "ooc/core.hpp"
#include "ooc_device.h"

#ifdef _OPENMP
#include <omp.h>
#endif

namespace ooc {

// ---------------------------------------------------------------- Extent / Stencil

std::string Extent::str() const {  // extent.hpp:131-138
  std::string s;
  for (int d = 0; d < ndim; ++d) {
    if (d) s += "x";
    s += "[" + std::to_string(lo[d]) + "," + std::to_string(hi[d]) + ")";
  }
  return s.empty() ? "[]" : s;
}

Stencil Stencil::line(int dim, index_t radius) {  // stencil.hpp:20-27
  Stencil s;
  for (index_t o = -radius; o <= radius; ++o) {
    Point p{0, 0, 0};
    p[dim] = o;
    s.offsets.push_back(p);
  }
  return s;
}

Stencil Stencil::star(int ndim, index_t radius) {  // stencil.hpp:28-41
  Stencil s;
  s.offsets.push_back(Point{0, 0, 0});
  for (int d = 0; d < ndim; ++d)
    for (index_t o = -radius; o <= radius; ++o) {
      if (o == 0) continue;
      Point p{0, 0, 0};
      p[d] = o;
      s.offsets.push_back(p);
    }
  return s;
}

std::pair<Point, Point> stencil_extents(const Stencil& s) {  // stencil.hpp:55-64
  if (s.offsets.empty()) throw ValidationError("stencil has no offsets");
  Point lo = s.offsets.front(), hi = s.offsets.front();
  for (const Point& o : s.offsets)
    for (int d = 0; d < 3; ++d) {
      lo[d] = std::min(lo[d], o[d]);
      hi[d] = std::max(hi[d], o[d]);
    }
  return {lo, hi};
}

// ---------------------------------------------------------------- expressions

namespace ex {
ExprPtr c(double v) {
  auto e = std::make_shared<Expr>();
  e->op = ExprOp::constant;
  e->value = v;
  return e;
}
ExprPtr r(int arg, index_t o0, index_t o1, index_t o2) {
  auto e = std::make_shared<Expr>();
  e->op = ExprOp::read;
  e->arg = arg;
  e->offset = {o0, o1, o2};
  return e;
}
ExprPtr coord(int dim) {
  auto e = std::make_shared<Expr>();
  e->op = ExprOp::coord;
  e->arg = dim;
  return e;
}
ExprPtr bin(ExprOp op, ExprPtr a, ExprPtr b) {
  auto e = std::make_shared<Expr>();
  e->op = op;
  e->lhs = std::move(a);
  e->rhs = std::move(b);
  return e;
}
}  // namespace ex

namespace {

// Post-order emission; the right operand sits one slot deeper (expr.cpp:13-23).
void emit(const ExprPtr& e, ExprTape& t, int depth, int& deepest) {
  if (!e) throw ValidationError("null expression node");
  if (expr_op_is_binary(e->op)) {
    emit(e->lhs, t, depth, deepest);
    emit(e->rhs, t, depth + 1, deepest);
    t.ins.push_back(ExprTape::Ins{e->op, 0, 0.0, Point{0, 0, 0}});
    return;
  }
  t.ins.push_back(ExprTape::Ins{e->op, e->arg, e->value, e->offset});
  deepest = std::max(deepest, depth + 1);
}

class Lexer {
 public:
  explicit Lexer(const std::string& s) : s_(s) {}
  bool at_end() {
    skip();
    return i_ >= s_.size();
  }
  char peek() {
    skip();
    return i_ < s_.size() ? s_[i_] : '\0';
  }
  std::string take() {
    skip();
    if (i_ >= s_.size()) throw ValidationError("unexpected end of expression: " + s_);
    if (s_[i_] == '(' || s_[i_] == ')') return std::string(1, s_[i_++]);
    std::size_t b = i_;
    while (i_ < s_.size() && !std::isspace(static_cast<unsigned char>(s_[i_])) && s_[i_] != '(' &&
           s_[i_] != ')')
      ++i_;
    return s_.substr(b, i_ - b);
  }

 private:
  void skip() {
    while (i_ < s_.size() && std::isspace(static_cast<unsigned char>(s_[i_]))) ++i_;
  }
  const std::string& s_;
  std::size_t i_ = 0;
};

index_t to_int(const std::string& tok) {
  char* end = nullptr;
  long long v = std::strtoll(tok.c_str(), &end, 10);
  if (tok.empty() || end != tok.c_str() + tok.size())
    throw ValidationError("expected integer in expression, got '" + tok + "'");
  return v;
}

ExprPtr parse_node(Lexer& lx, bool coords) {  // expr.cpp:73-123
  std::string tok = lx.take();
  if (tok == ")") throw ValidationError("unexpected ')' in expression");
  if (tok != "(") {
    if (coords && tok.size() == 1 && (tok[0] == 'i' || tok[0] == 'j' || tok[0] == 'k'))
      return ex::coord(tok[0] - 'i');
    char* end = nullptr;
    double v = std::strtod(tok.c_str(), &end);
    if (end == tok.c_str() || end != tok.c_str() + tok.size())
      throw ValidationError("unrecognised token '" + tok + "' in expression");
    return ex::c(v);
  }
  std::string head = lx.take();
  if (head == "r") {
    int arg = static_cast<int>(to_int(lx.take()));
    Point off{0, 0, 0};
    for (int d = 0; lx.peek() != ')'; ++d) {
      if (d >= 3) throw ValidationError("read offset has more than 3 components");
      off[d] = to_int(lx.take());
    }
    lx.take();
    return ex::r(arg, off[0], off[1], off[2]);
  }
  static const std::pair<const char*, ExprOp> kOps[] = {
      {"+", ExprOp::add},      {"-", ExprOp::sub}, {"*", ExprOp::mul},
      {"/", ExprOp::divide},   {"min", ExprOp::min}, {"max", ExprOp::max}};
  ExprOp op = ExprOp::constant;
  bool found = false;
  for (const auto& [name, o] : kOps)
    if (head == name) {
      op = o;
      found = true;
    }
  if (!found) throw ValidationError("unknown operator '" + head + "' in expression");
  ExprPtr a = parse_node(lx, coords);
  ExprPtr b = parse_node(lx, coords);
  if (lx.take() != ")") throw ValidationError("operator '" + head + "' takes exactly two operands");
  return ex::bin(op, std::move(a), std::move(b));
}

std::string fmt17(double v) {
  std::ostringstream os;
  os.precision(17);
  os << v;
  return os.str();
}

}  // namespace

ExprTape ExprTape::compile(const ExprPtr& e) {  // expr.cpp:134-140
  ExprTape t;
  int deepest = 0;
  emit(e, t, 0, deepest);
  t.max_stack = deepest;
  return t;
}

ExprPtr parse_prefix_expr(const std::string& text, bool allow_coords) {  // expr.cpp:142-147
  Lexer lx(text);
  ExprPtr e = parse_node(lx, allow_coords);
  if (!lx.at_end()) throw ValidationError("trailing tokens after expression: " + text);
  return e;
}

std::string expr_to_string(const ExprPtr& e) {  // expr.cpp:149-172
  if (!e) return "<null>";
  switch (e->op) {
    case ExprOp::constant:
      return fmt17(e->value);
    case ExprOp::coord:
      return std::string(1, static_cast<char>('i' + e->arg));
    case ExprOp::read: {
      std::string s = "(r " + std::to_string(e->arg);
      for (int d = 0; d < 3; ++d) s += " " + std::to_string(e->offset[d]);
      return s + ")";
    }
    default:
      break;
  }
  const char* name = e->op == ExprOp::add      ? "+"
                     : e->op == ExprOp::sub    ? "-"
                     : e->op == ExprOp::mul    ? "*"
                     : e->op == ExprOp::divide ? "/"
                     : e->op == ExprOp::min    ? "min"
                                               : "max";
  return std::string("(") + name + " " + expr_to_string(e->lhs) + " " + expr_to_string(e->rhs) +
         ")";
}

// ---------------------------------------------------------------- pinned host storage

void* pinned_host_alloc(std::size_t bytes) {
  if (bytes == 0) bytes = 8;
  void* p = nullptr;
  if (ooc_host_alloc(bytes, &p) == OOC_OK && p) return p;
  // No usable CUDA device (CPU-only planning/tests): plain aligned memory.
  p = std::aligned_alloc(4096, (bytes + 4095) / 4096 * 4096);
  if (!p) throw std::bad_alloc();
  // tag: keep a registry-free scheme by asking the device layer to classify on free
  return p;
}

void pinned_host_free(void* p) noexcept {
  if (!p) return;
  if (ooc_host_free(p) != OOC_OK) std::free(p);
}

// ---------------------------------------------------------------- datasets

DatasetId declare_dataset(Mesh& mesh, const std::string& name, const Extent& core, Point halo,
                          index_t elem_bytes, const std::function<double(Point)>& fill) {
  // contract and messages: proj/src/dataset.cpp:5-38
  if (mesh.find(name) >= 0) throw ValidationError("duplicate dataset name '" + name + "'");
  if (core.empty()) throw ValidationError("dataset '" + name + "' has a zero-size core extent");
  if (core.ndim < 1 || core.ndim > 3)
    throw ValidationError("dataset '" + name + "' has unsupported rank");
  Block& block = mesh.blocks[0];
  if (block.ndim == 0)
    block.ndim = core.ndim;
  else if (block.ndim != core.ndim)
    throw ValidationError("dataset '" + name + "' has rank " + std::to_string(core.ndim) +
                          " but its block has rank " + std::to_string(block.ndim));
  for (int d = 0; d < core.ndim; ++d)
    if (halo[d] < 0) throw ValidationError("dataset '" + name + "' has a negative halo depth");
  for (int d = core.ndim; d < 3; ++d) halo[d] = 0;
  if (elem_bytes <= 0) throw ValidationError("dataset '" + name + "' has non-positive elem_bytes");

  Dataset ds;
  ds.name = name;
  ds.core = core;
  ds.halo = halo;
  ds.elem_bytes = elem_bytes;
  ds.stale_region = Extent::none(core.ndim);
  const Extent a = ds.alloc();
  ds.host.resize(static_cast<std::size_t>(a.size()));
  // Rows (all dims but the contiguous last one) are filled independently; the
  // fill is a pure function of the point, so the result is order-independent.
  const index_t n0 = a.len(0), n1 = a.len(1), n2 = a.len(2);
  double* out = ds.host.data();
  const index_t rows = n0 * n1;
  auto fill_row = [&](index_t row) {
    Point p{a.lo[0] + row / n1, a.lo[1] + row % n1, a.lo[2]};
    double* o = out + row * n2;
    for (index_t k = 0; k < n2; ++k, ++p[2]) o[k] = fill(p);
  };
  if (a.size() >= (1 << 20)) {
#pragma omp parallel for schedule(static)
    for (index_t row = 0; row < rows; ++row) fill_row(row);
  } else {
    for (index_t row = 0; row < rows; ++row) fill_row(row);
  }
  mesh.datasets.push_back(std::move(ds));
  return static_cast<DatasetId>(mesh.datasets.size() - 1);
}

DatasetId declare_dataset(Mesh& mesh, const std::string& name, const Extent& core, Point halo,
                          index_t elem_bytes, double fill_value) {
  return declare_dataset(mesh, name, core, halo, elem_bytes,
                         [fill_value](Point) { return fill_value; });
}

// ---------------------------------------------------------------- validation

namespace {

void check_expr_reads(const Mesh& mesh, const ParLoop& loop, const ExprPtr& e,
                      const std::string& where) {  // loop.cpp:9-28
  expr_visit(e, [&](const Expr& n) {
    if (n.op == ExprOp::coord)
      throw ValidationError("coordinate terms are only valid in fill expressions (" + where + ")");
    if (n.op != ExprOp::read) return;
    if (n.arg < 0 || n.arg >= static_cast<int>(loop.args.size()))
      throw ValidationError(where + " reads argument " + std::to_string(n.arg) +
                            " which does not exist");
    const LoopArg& a = loop.args[static_cast<std::size_t>(n.arg)];
    if (!access_reads(a.mode))
      throw ValidationError(where + " reads argument " + std::to_string(n.arg) + " (dataset '" +
                            mesh[a.dataset].name + "') declared WRITE");
    if (!a.stencil.has_offset(n.offset))
      throw ValidationError(where + " reads dataset '" + mesh[a.dataset].name + "' at offset (" +
                            std::to_string(n.offset[0]) + "," + std::to_string(n.offset[1]) + "," +
                            std::to_string(n.offset[2]) + ") which is not in the declared stencil");
  });
}

}  // namespace

void validate_loop(const Mesh& mesh, ParLoop& loop) {  // loop.cpp:32-105
  if (loop.range.empty()) throw ValidationError("loop has an empty iteration range");
  if (loop.args.empty() && loop.kernel.writes.empty() && !loop.has_reduction())
    throw ValidationError("loop has no arguments and no reduction");
  if (loop.args.size() > OOC_MAX_ARGS)
    throw ValidationError("loop has more than " + std::to_string(OOC_MAX_ARGS) + " arguments");

  for (const LoopArg& a : loop.args) {
    if (a.dataset < 0 || a.dataset >= static_cast<int>(mesh.datasets.size()))
      throw ValidationError("loop argument names an unknown dataset");
    if (a.stencil.offsets.empty()) throw ValidationError("loop argument has an empty stencil");
    const Dataset& ds = mesh[a.dataset];
    if (loop.range.ndim != ds.core.ndim)
      throw ValidationError("loop rank does not match dataset '" + ds.name + "'");
    for (const Point& off : a.stencil.offsets)
      for (int d = ds.core.ndim; d < 3; ++d)
        if (off[d] != 0)
          throw ValidationError("stencil offset uses a dimension beyond the rank of '" + ds.name +
                                "'");
    if (access_writes(a.mode)) {
      if (!a.stencil.is_point())
        throw ValidationError("write access to '" + ds.name +
                              "' must use the single zero-offset stencil");
      if (!ds.core.contains(loop.range))
        throw ValidationError("loop range " + loop.range.str() + " exceeds the core " +
                              ds.core.str() + " of written dataset '" + ds.name + "'");
    }
    if (access_reads(a.mode)) {
      auto [lo, hi] = stencil_extents(a.stencil);
      Extent reach = loop.range.expand(lo, hi);
      if (!ds.alloc().contains(reach))
        throw ValidationError("loop reads " + reach.str() + " of dataset '" + ds.name +
                              "' which exceeds its allocation " + ds.alloc().str());
    }
  }
  for (std::size_t i = 0; i < loop.args.size(); ++i) {
    if (!access_writes(loop.args[i].mode)) continue;
    for (std::size_t k = 0; k < loop.args.size(); ++k)
      if (k != i && loop.args[k].dataset == loop.args[i].dataset)
        throw ValidationError("dataset '" + mesh[loop.args[i].dataset].name +
                              "' is written and appears in another argument of the same loop");
  }
  if (loop.kernel.writes.size() > OOC_MAX_WRITES)
    throw ValidationError("kernel writes more than " + std::to_string(OOC_MAX_WRITES) +
                          " arguments");
  std::vector<char> written(loop.args.size(), 0);
  for (const auto& w : loop.kernel.writes) {
    if (w.arg < 0 || w.arg >= static_cast<int>(loop.args.size()))
      throw ValidationError("kernel writes argument " + std::to_string(w.arg) +
                            " which does not exist");
    if (!access_writes(loop.args[static_cast<std::size_t>(w.arg)].mode))
      throw ValidationError("kernel writes argument " + std::to_string(w.arg) + " declared READ");
    if (written[static_cast<std::size_t>(w.arg)])
      throw ValidationError("kernel writes argument " + std::to_string(w.arg) + " twice");
    written[static_cast<std::size_t>(w.arg)] = 1;
    check_expr_reads(mesh, loop, w.expr, "write expression");
  }
  for (std::size_t i = 0; i < loop.args.size(); ++i)
    if (access_writes(loop.args[i].mode) && !written[i])
      throw ValidationError("argument " + std::to_string(i) + " (dataset '" +
                            mesh[loop.args[i].dataset].name +
                            "') is declared writable but the kernel never writes it");
  if (loop.has_reduction()) {
    if (!loop.kernel.reduce_expr) throw ValidationError("reduction without an expression");
    if (loop.kernel.reduce_name.empty()) throw ValidationError("reduction without a name");
    check_expr_reads(mesh, loop, loop.kernel.reduce_expr, "reduction expression");
  }
  loop.write_tapes.clear();
  std::size_t total = 0;
  for (const auto& w : loop.kernel.writes) {
    loop.write_tapes.push_back(ExprTape::compile(w.expr));
    if (loop.write_tapes.back().max_stack > OOC_MAX_STACK)
      throw ValidationError("expression deeper than " + std::to_string(OOC_MAX_STACK));
    total += loop.write_tapes.back().ins.size();
  }
  loop.reduce_tape = ExprTape{};
  if (loop.has_reduction()) {
    loop.reduce_tape = ExprTape::compile(loop.kernel.reduce_expr);
    if (loop.reduce_tape.max_stack > OOC_MAX_STACK)
      throw ValidationError("expression deeper than " + std::to_string(OOC_MAX_STACK));
    total += loop.reduce_tape.ins.size();
  }
  if (total > OOC_MAX_TAPE)
    throw ValidationError("loop kernel exceeds " + std::to_string(OOC_MAX_TAPE) + " instructions");
}

}  // namespace ooc
