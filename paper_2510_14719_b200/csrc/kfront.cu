// kfront.cu — `.k` kernel front end: run a kernel written in the reference grammar on the B200
// path ("the compile_kernel analogue").
//
// Reference grammar: ref SPEC.md:120-134, parser ref proj/include/warpspec/parse.hpp:412-686
// (this is an independent implementation of the documented grammar, not a port of that file).
// Semantics of ws_run_kernel mirror the reference's tile-by-tile oracle run
// (`interpret_tiles`, ref proj/tests/support/fixtures.hpp:148-157): buffers are named host
// arrays, parameters without a buffer start zeroed, pids [pid_lo, pid_hi) execute and their
// stores land in the buffers. Instead of interpreting tile ops, the front end
//   1. evaluates only the scalar (index) part of the program per pid and loop iteration,
//   2. recognises the kernel shape and the per-pid tile geometry,
//   3. runs the tile math as tensor-core launches through the C-ABI:
//      gemm.k family (gemm.k / gemm_large.k / gemm_batched.k / gemm_act.k shapes, optional
//      1x1 scale or relu epilogue) -> pids grouped into zero-padded ws_gemm_tn launches;
//      flash .k of SURVEY.md Appendix A -> ws_attn_fwd (acc, l and m written back as the .k's);
//      max-shift attention.k (ref proj/kernels/attention.k) -> GEMM, row-block shift, GEMM.
//   4. applies a RunSpec (ws_runspec, ref driver.hpp:42-57) with compile_kernel's rejections.
// Unsupported shapes fail with WS_UNSUPPORTED_KERNEL, never with a CPU fallback.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <exception>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <unistd.h>

#include "../../include/ws.h"

namespace ws_detail {
ws_status set_error(ws_status s, const std::string& m);  // capi.cu
void count_launch();                                       // capi.cu: ws_launch_count evidence
}  // namespace ws_detail

namespace {

struct KError : std::runtime_error {
  ws_status code;
  KError(ws_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void kfail(ws_status c, const std::string& m) { throw KError(c, m); }

// ------------------------------------------------------------------------------------------------
// lexer
// ------------------------------------------------------------------------------------------------
enum class T { Value, Ident, Int, Real, Shape, Punct, Trans, End };
struct Tok {
  T k;
  std::string s;
  int64_t i = 0, i2 = 0;
  double r = 0;
};

std::vector<Tok> lex_line(const std::string& ln, int line_no) {
  std::vector<Tok> out;
  size_t i = 0, n = ln.size();
  auto err = [&](const std::string& m) { kfail(WS_PARSE, "line " + std::to_string(line_no) + ": " + m); };
  while (i < n) {
    char c = ln[i];
    if (c == '#') break;
    if (isspace(static_cast<unsigned char>(c))) { ++i; continue; }
    if (c == '%') {
      size_t j = i + 1;
      while (j < n && (isalnum(static_cast<unsigned char>(ln[j])) || ln[j] == '_')) ++j;
      if (j == i + 1) {  // modulo operator
        out.push_back({T::Punct, "%"});
        i = j;
        continue;
      }
      out.push_back({T::Value, ln.substr(i + 1, j - i - 1)});
      i = j;
      continue;
    }
    if (c == '.' && i + 1 < n && ln[i + 1] == 'T' && (i + 2 >= n || !isalnum(static_cast<unsigned char>(ln[i + 2])))) {
      out.push_back({T::Trans, ".T"});
      i += 2;
      continue;
    }
    if (c == '.' && i + 1 < n && ln[i + 1] == '.') {
      out.push_back({T::Punct, ".."});
      i += 2;
      continue;
    }
    if (isdigit(static_cast<unsigned char>(c))) {
      size_t j = i;
      while (j < n && isdigit(static_cast<unsigned char>(ln[j]))) ++j;
      if (j < n && ln[j] == 'x' && j + 1 < n && isdigit(static_cast<unsigned char>(ln[j + 1]))) {
        size_t k = j + 1;
        while (k < n && isdigit(static_cast<unsigned char>(ln[k]))) ++k;
        Tok t{T::Shape, ln.substr(i, k - i)};
        t.i = std::stoll(ln.substr(i, j - i));
        t.i2 = std::stoll(ln.substr(j + 1, k - j - 1));
        out.push_back(t);
        i = k;
        continue;
      }
      bool real = false;
      if (j < n && ln[j] == '.' && !(j + 1 < n && ln[j + 1] == '.')) {
        real = true;
        ++j;
        while (j < n && isdigit(static_cast<unsigned char>(ln[j]))) ++j;
      }
      if (j < n && (ln[j] == 'e' || ln[j] == 'E')) {
        real = true;
        ++j;
        if (j < n && (ln[j] == '-' || ln[j] == '+')) ++j;
        while (j < n && isdigit(static_cast<unsigned char>(ln[j]))) ++j;
      }
      Tok t{real ? T::Real : T::Int, ln.substr(i, j - i)};
      if (real)
        t.r = std::stod(t.s);
      else
        t.i = std::stoll(t.s);
      out.push_back(t);
      i = j;
      continue;
    }
    if (isalpha(static_cast<unsigned char>(c)) || c == '_') {
      size_t j = i;
      while (j < n && (isalnum(static_cast<unsigned char>(ln[j])) || ln[j] == '_')) ++j;
      out.push_back({T::Ident, ln.substr(i, j - i)});
      i = j;
      continue;
    }
    if (std::string("(){}[],=<>:+-*/").find(c) != std::string::npos) {
      out.push_back({T::Punct, std::string(1, c)});
      ++i;
      continue;
    }
    err(std::string("unexpected character '") + c + "'");
  }
  out.push_back({T::End, ""});
  return out;
}

// ------------------------------------------------------------------------------------------------
// IR
// ------------------------------------------------------------------------------------------------
enum class K { Pid, Const, Arith, ConstTile, Load, Dot, Ew, Reduce, Store, Yield };
struct Shape {
  int64_t r = 0, c = 0;
  bool real = false;
};
struct Op {
  K k;
  std::string res;                 // result value (empty for store / yield)
  std::vector<std::string> args;   // value operands
  std::string fn;                  // arith / ew / reduce fn name
  std::string buf;                 // tma_load / store buffer
  Shape shape;                     // tile shape
  int64_t ival = 0;                // scalar constant
  bool zeros = false, trans = false;
  int axis = 0;
  std::vector<double> lit;         // tile literal values
};
struct Param {
  std::string name;
  Shape shape;
};
struct Kernel {
  std::string name;
  std::vector<Param> params;
  std::vector<Op> pro, body, epi;
  std::string ind;                                        // induction variable
  int64_t lo = 0, hi = 0;                                 // loop bounds
  std::vector<std::pair<std::string, std::string>> iter;  // (iter arg, init)
};

struct Parser {
  std::vector<Tok> t;
  size_t p = 0;
  int line = 0;
  int gensym = 0;
  std::vector<Op>* out = nullptr;

  [[noreturn]] void err(const std::string& m) { kfail(WS_PARSE, "line " + std::to_string(line) + ": " + m); }
  const Tok& peek(size_t o = 0) { return t[std::min(p + o, t.size() - 1)]; }
  bool punct(const char* s) {
    if (peek().k == T::Punct && peek().s == s) return ++p, true;
    return false;
  }
  void need(const char* s) {
    if (!punct(s)) err(std::string("expected '") + s + "'");
  }
  bool ident(const char* s) {
    if (peek().k == T::Ident && peek().s == s) return ++p, true;
    return false;
  }
  std::string value() {
    if (peek().k != T::Value) err("expected %value");
    return t[p++].s;
  }
  std::string any_ident() {
    if (peek().k != T::Ident) err("expected identifier");
    return t[p++].s;
  }
  int64_t integer() {
    bool neg = punct("-");
    if (peek().k != T::Int) err("expected integer");
    return (neg ? -1 : 1) * t[p++].i;
  }
  Shape shape() {
    if (peek().k != T::Shape) err("expected tile shape RxC");
    Shape s{t[p].i, t[p].i2};
    ++p;
    std::string e = any_ident();
    if (e != "int" && e != "real") err("expected element kind 'int' or 'real'");
    s.real = e == "real";
    return s;
  }
  void end() {
    if (peek().k != T::End) err("unexpected trailing tokens");
  }
  std::string fresh() { return "__t" + std::to_string(gensym++); }
  std::string emit_int(int64_t v) {
    Op o{K::Const};
    o.res = fresh();
    o.ival = v;
    out->push_back(o);
    return o.res;
  }
  std::string emit_arith(const std::string& fn, const std::string& a, const std::string& b) {
    Op o{K::Arith};
    o.res = fresh();
    o.fn = fn;
    o.args = {a, b};
    out->push_back(o);
    return o.res;
  }
  // scalar expression sugar: + - * / % over %ids, integers, pid, parentheses
  std::string term() {
    if (punct("(")) {
      std::string v = expr();
      need(")");
      return v;
    }
    if (punct("-")) {
      if (peek().k == T::Int) return emit_int(-t[p++].i);
      return emit_arith("sub", emit_int(0), term());
    }
    if (peek().k == T::Value) return t[p++].s;
    if (peek().k == T::Int) return emit_int(t[p++].i);
    if (ident("pid")) {
      Op o{K::Pid};
      o.res = fresh();
      out->push_back(o);
      return o.res;
    }
    err("expected scalar operand");
  }
  std::string factor() {
    std::string v = term();
    while (true) {
      if (punct("*"))
        v = emit_arith("mul", v, term());
      else if (punct("/"))
        v = emit_arith("div", v, term());
      else if (punct("%"))
        v = emit_arith("mod", v, term());
      else
        return v;
    }
  }
  std::string expr() {
    std::string v = factor();
    while (true) {
      if (punct("+"))
        v = emit_arith("add", v, factor());
      else if (punct("-"))
        v = emit_arith("sub", v, factor());
      else
        return v;
    }
  }
  std::string operand() {
    if (peek().k == T::Value &&
        !(peek(1).k == T::Punct && std::string("+-*/%").find(peek(1).s) != std::string::npos && peek(1).s.size() == 1))
      return t[p++].s;
    return expr();
  }

  // one statement (not loop structure)
  void stmt(bool in_loop) {
    if (ident("store")) {
      Op o{K::Store};
      o.buf = any_ident();
      need("[");
      std::string r = expr();
      need(",");
      std::string c = expr();
      need("]");
      need("=");
      o.args = {value(), r, c};
      end();
      out->push_back(o);
      return;
    }
    if (ident("yield")) {
      if (!in_loop) err("yield outside loop");
      Op o{K::Yield};
      o.args.push_back(operand());
      while (punct(",")) o.args.push_back(operand());
      end();
      out->push_back(o);
      return;
    }
    std::string res = value();
    need("=");
    Op o{K::Const};
    o.res = res;
    if (ident("pid")) {
      o.k = K::Pid;
    } else if (ident("const")) {
      if (ident("zeros")) {
        need(":");
        o.k = K::ConstTile;
        o.zeros = true;
        o.shape = shape();
      } else if (punct("[")) {
        o.k = K::ConstTile;
        std::vector<double> vals;
        int64_t rows = 0;
        do {
          need("[");
          ++rows;
          do {
            bool neg = punct("-");
            if (peek().k == T::Int)
              vals.push_back((neg ? -1.0 : 1.0) * static_cast<double>(t[p++].i));
            else if (peek().k == T::Real)
              vals.push_back((neg ? -1.0 : 1.0) * t[p++].r);
            else
              err("expected number in tile literal");
          } while (punct(","));
          need("]");
        } while (punct(","));
        need("]");
        need(":");
        o.shape = shape();
        if (rows != o.shape.r || static_cast<int64_t>(vals.size()) != o.shape.r * o.shape.c)
          err("tile literal does not match its shape");
        o.lit = vals;
      } else {
        o.k = K::Const;
        o.ival = integer();
      }
    } else if (peek().k == T::Ident && (peek().s == "add" || peek().s == "sub" || peek().s == "mul" ||
                                        peek().s == "div" || peek().s == "mod")) {
      o.k = K::Arith;
      o.fn = any_ident();
      o.args.push_back(operand());
      need(",");
      o.args.push_back(operand());
    } else if (ident("tma_load")) {
      if (!in_loop) err("tma_load outside the loop");
      o.k = K::Load;
      o.buf = any_ident();
      need("[");
      o.args.push_back(expr());
      need(",");
      o.args.push_back(expr());
      need("]");
      need(":");
      o.shape = shape();
    } else if (ident("dot")) {
      o.k = K::Dot;
      o.args.push_back(value());
      need(",");
      o.args.push_back(value());
      if (peek().k == T::Trans) {
        ++p;
        o.trans = true;
      }
      need(",");
      if (!ident("acc")) err("expected acc=");
      need("=");
      o.args.push_back(value());
    } else if (ident("ew")) {
      o.k = K::Ew;
      o.fn = any_ident();
      o.args.push_back(value());
      if (punct(",")) o.args.push_back(value());
    } else if (ident("reduce")) {
      o.k = K::Reduce;
      o.fn = any_ident();
      o.args.push_back(value());
      if (!ident("axis")) err("expected axis=");
      need("=");
      o.axis = static_cast<int>(integer());
    } else {
      err("unknown operation '" + peek().s + "'");
    }
    end();
    out->push_back(o);
  }
};

Kernel parse(const std::string& text) {
  Kernel g;
  std::vector<std::string> lines;
  {
    size_t s = 0;
    while (s <= text.size()) {
      size_t e = text.find('\n', s);
      if (e == std::string::npos) e = text.size();
      lines.push_back(text.substr(s, e - s));
      s = e + 1;
    }
  }
  Parser ps;
  int state = 0;  // 0 header, 1 prologue, 2 loop body, 3 epilogue, 4 done
  for (size_t li = 0; li < lines.size(); ++li) {
    ps.t = lex_line(lines[li], static_cast<int>(li) + 1);
    ps.p = 0;
    ps.line = static_cast<int>(li) + 1;
    if (ps.peek().k == T::End) continue;
    if (state == 0) {
      if (!ps.ident("kernel")) ps.err("expected 'kernel'");
      g.name = ps.any_ident();
      ps.need("(");
      if (!ps.punct(")")) {
        do {
          Param pr;
          pr.name = ps.any_ident();
          ps.need(":");
          if (!ps.ident("buf")) ps.err("expected buf<...>");
          ps.need("<");
          pr.shape = ps.shape();
          ps.need(">");
          g.params.push_back(pr);
        } while (ps.punct(","));
        ps.need(")");
      }
      ps.need("{");
      ps.end();
      state = 1;
      ps.out = &g.pro;
      continue;
    }
    if (state == 1 && ps.peek().k == T::Ident && ps.peek().s == "loop") {
      ++ps.p;
      g.ind = ps.value();
      if (!ps.ident("in")) ps.err("expected 'in'");
      g.lo = ps.integer();
      ps.need("..");
      g.hi = ps.integer();
      if (ps.ident("iter")) {
        ps.need("(");
        do {
          std::string a = ps.value();
          ps.need("=");
          g.iter.push_back({a, ps.value()});
        } while (ps.punct(","));
        ps.need(")");
      }
      ps.need("{");
      ps.end();
      state = 2;
      ps.out = &g.body;
      continue;
    }
    if (ps.punct("}")) {
      ps.end();
      if (state == 2) {
        state = 3;
        ps.out = &g.epi;
      } else if (state == 1 || state == 3) {
        state = 4;
      } else {
        ps.err("unbalanced '}'");
      }
      continue;
    }
    if (state == 4) ps.err("text after the kernel");
    ps.stmt(state == 2);
  }
  if (state != 4) kfail(WS_PARSE, "kernel body not closed");
  return g;
}

// ------------------------------------------------------------------------------------------------
// scalar evaluation per pid (and per loop iteration)
// ------------------------------------------------------------------------------------------------
int64_t arith(const std::string& f, int64_t a, int64_t b) {
  const uint64_t ua = static_cast<uint64_t>(a), ub = static_cast<uint64_t>(b);
  if (f == "add") return static_cast<int64_t>(ua + ub);  // wrapping, like ref tile.hpp:63-71
  if (f == "sub") return static_cast<int64_t>(ua - ub);
  if (f == "mul") return static_cast<int64_t>(ua * ub);
  if (b == 0) kfail(WS_EVAL, f + " by zero");
  return f == "div" ? a / b : a % b;
}

struct ScalarEnv {
  std::map<std::string, int64_t> v;
  int64_t get(const std::string& n) const {
    auto it = v.find(n);
    if (it == v.end()) kfail(WS_EVAL, "unbound scalar %" + n);
    return it->second;
  }
  void run(const std::vector<Op>& ops, int64_t pid) {
    for (const Op& o : ops) {
      if (o.k == K::Pid) v[o.res] = pid;
      else if (o.k == K::Const) v[o.res] = o.ival;
      else if (o.k == K::Arith) v[o.res] = arith(o.fn, get(o.args[0]), get(o.args[1]));
    }
  }
};


// ------------------------------------------------------------------------------------------------
// RunSpec -> launch choices (ref proj/include/warpspec/driver.hpp:42-57, compile_kernel :116-189)
// ------------------------------------------------------------------------------------------------
struct Plan {
  int d = 0, p = 0;         // aref depth / MMA k-blocks in flight on the GPU; 0 = library default
  int coop = 0;             // 0 = library default, 1 = single-CTA tiles, 2 = CTA-pair tiles
  bool persistent = true;
  std::string mode;         // the pipeline the reference's compile_kernel applies: none|ws|fine|coarse
};

// The rejections of compile_kernel, in its order, evaluated on the parsed graph: D/P range
// (driver.hpp:117-118), the pipelining pass (fine: pipeline.hpp:44-92; coarse: :258-315; auto:
// driver.hpp:129-150), then the cooperative split (grid.hpp:24-46). The reference's register and
// shared-memory gates are cost-model conventions; the kernels apply the real
// sm_100a limits at launch.
Plan resolve_spec(const Kernel& g, const ws_runspec* rs) {
  Plan pl;
  if (!rs) {
    pl.mode = "auto";
    return pl;
  }
  if (rs->d < 0) kfail(WS_PIPELINE_INFEASIBLE, "D must be >= 1");
  if (rs->p < 0) kfail(WS_PIPELINE_INFEASIBLE, "P must be >= 1");
  if (rs->mode < WS_MODE_AUTO || rs->mode > WS_MODE_NONE) kfail(WS_PARSE, "unknown pipeline mode");
  pl.d = rs->d;
  pl.p = rs->p;
  pl.persistent = rs->persistent != 0;
  bool has_t = false, has_c = false, axis0 = false;
  for (const Op& o : g.body) {
    if (o.k == K::Dot) has_t = true;
    if (o.k == K::Ew || o.k == K::Reduce) has_c = true;
    if (o.k == K::Reduce && o.axis == 0) axis0 = true;
  }
  const int64_t trip = g.hi - g.lo;
  if (rs->mode == WS_MODE_NONE) {
    pl.mode = "none";
    pl.d = pl.p = 1;  // the sequential program: one stage, one MMA group in flight
  } else {
    int mode = rs->mode;
    const bool autom = mode == WS_MODE_AUTO;
    if (autom) mode = (has_t && has_c && trip >= 1) ? WS_MODE_COARSE : (has_t && trip >= 1) ? WS_MODE_FINE : -1;
    pl.mode = "ws";
    if (mode == WS_MODE_COARSE) {
      if (trip < 1) kfail(WS_PIPELINE_INFEASIBLE, "coarse-grained schedule needs at least one trip");
      if (!has_t || !has_c)
        kfail(WS_PIPELINE_INFEASIBLE, "coarse-grained schedule needs a tensor-core stage and a transform stage");
      if (pl.d == 1) {
        if (!autom) kfail(WS_PIPELINE_INFEASIBLE, "coarse-grained schedule needs channel depth D >= 2");
        // auto: a staged schedule that does not fit degrades to plain warp specialization
      } else {
        pl.mode = "coarse";
      }
      pl.p = 0;  // no MMA window in a coarse schedule: commits release the stages
    } else if (mode == WS_MODE_FINE) {
      if (has_c) kfail(WS_PIPELINE_INFEASIBLE, "fine-grained pipelining needs a pure dot-chain loop body");
      if (!has_t) kfail(WS_PIPELINE_INFEASIBLE, "fine-grained pipelining needs at least one dot");
      if (pl.d > 0 && pl.p > pl.d)
        kfail(WS_PIPELINE_INFEASIBLE, "P=" + std::to_string(pl.p) + " exceeds channel depth D=" + std::to_string(pl.d) +
                                          " (deadlock: a slot would be reused while borrowed)");
      pl.mode = "fine";
    } else {
      pl.p = 0;
    }
  }
  if (rs->coop_wgs < 0) kfail(WS_INDIVISIBLE_TILE, "cooperative warp group count must be >= 1");
  if (rs->coop_wgs > 1) {
    if (axis0) kfail(WS_INDIVISIBLE_TILE, "row-band split cannot cross an axis-0 reduction");
    for (const Op& o : g.epi)
      if (o.k == K::Store) {
        const Op* src = nullptr;
        for (auto* ops : {&g.epi, &g.body, &g.pro})
          for (const Op& x : *ops)
            if (x.res == o.args[0]) src = &x;
        int64_t rows = src ? src->shape.r : 0;
        if (!src) {  // an iter arg: its init's tile shape
          for (auto& [a, init] : g.iter)
            if (a == o.args[0])
              for (auto* ops : {&g.pro})
                for (const Op& x : *ops)
                  if (x.res == init) rows = x.shape.r;
        }
        if (rows > 0 && rows % rs->coop_wgs != 0)
          kfail(WS_INDIVISIBLE_TILE, "output tile rows " + std::to_string(rows) + " not divisible by " +
                                         std::to_string(rs->coop_wgs) + " warp groups");
      }
  }
  pl.coop = rs->coop_wgs == 0 ? 0 : rs->coop_wgs == 1 ? 1 : 2;
  return pl;
}

// ------------------------------------------------------------------------------------------------
// host buffers, staging
// ------------------------------------------------------------------------------------------------
struct HostBuf {
  std::string name;
  Shape shape;
  void* data = nullptr;     // caller's array (double for real, int64 for int)
  std::vector<double> own;  // zero-initialised storage when the caller passed none
  double get(int64_t r, int64_t c) const {
    const int64_t i = r * shape.c + c;
    return shape.real ? static_cast<const double*>(data)[i] : static_cast<double>(static_cast<const int64_t*>(data)[i]);
  }
  void set(int64_t r, int64_t c, double x) {
    const int64_t i = r * shape.c + c;
    if (shape.real)
      static_cast<double*>(data)[i] = x;
    else
      static_cast<int64_t*>(data)[i] = static_cast<int64_t>(std::llround(x));
  }
  double amax() const {
    double m = 0;
    const int64_t n = shape.r * shape.c;
    for (int64_t i = 0; i < n; ++i) m = std::max(m, std::fabs(get(i / shape.c, i % shape.c)));
    return m;
  }
};

uint16_t to_half_bits(float f, int dt) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if (dt == WS_BF16) {  // round to nearest even
    uint32_t r = u + 0x7FFFu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(r >> 16);
  }
  // fp16 (values of this path are small integers / k/4: normal range, round to nearest even)
  const uint32_t sign = (u >> 16) & 0x8000u;
  int32_t e = static_cast<int32_t>((u >> 23) & 0xFF) - 127 + 15;
  uint32_t m = u & 0x7FFFFFu;
  if ((u & 0x7FFFFFFFu) == 0) return static_cast<uint16_t>(sign);
  if (e <= 0) {  // subnormal
    if (e < -10) return static_cast<uint16_t>(sign);
    m |= 0x800000u;
    const int shift = 14 - e;
    uint32_t half = m >> shift;
    const uint32_t rem = m & ((1u << shift) - 1), mid = 1u << (shift - 1);
    if (rem > mid || (rem == mid && (half & 1))) ++half;
    return static_cast<uint16_t>(sign | half);
  }
  if (e >= 31) return static_cast<uint16_t>(sign | 0x7C00u);
  uint32_t half = (static_cast<uint32_t>(e) << 10) | (m >> 13);
  const uint32_t rem = m & 0x1FFFu;
  if (rem > 0x1000u || (rem == 0x1000u && (half & 1))) ++half;
  return static_cast<uint16_t>(sign | half);
}

float half_to_float(uint16_t h, int dt) {
  uint32_t u;
  if (dt == WS_BF16) {
    u = static_cast<uint32_t>(h) << 16;
  } else {
    const uint32_t s = (h & 0x8000u) << 16, e = (h >> 10) & 0x1F, m = h & 0x3FF;
    if (e == 0) {
      float f = std::ldexp(static_cast<float>(m), -24);
      return s ? -f : f;
    }
    u = s | ((e + 112) << 23) | (m << 13);
  }
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) kfail(WS_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}
void ws_check(ws_status s) {
  if (s != WS_OK) kfail(s, ws_last_error());
}

// Per host thread: device blocks and pinned host blocks reused across calls (a .k run is
// synchronous, so a block is free again when the call returns), grown on demand.
struct Staging {
  struct Blk {
    void* p = nullptr;
    size_t n = 0;
    int dev = -1;
  };
  Blk dev[8], host[8];
  void* device(int i, size_t n) {
    int cur = 0;
    cudaGetDevice(&cur);
    Blk& b = dev[i];
    if (b.n < n || b.dev != cur) {
      if (b.p) cudaFree(b.p);
      b = Blk{};
      cuda_check(cudaMalloc(&b.p, n), "cudaMalloc");
      b.n = n;
      b.dev = cur;
    }
    return b.p;
  }
  void* pinned(int i, size_t n) {
    Blk& b = host[i];
    if (b.n < n) {
      if (b.p) cudaFreeHost(b.p);
      b = Blk{};
      cuda_check(cudaHostAlloc(&b.p, n, cudaHostAllocPortable), "cudaHostAlloc");
      b.n = n;
    }
    return b.p;
  }
  ~Staging() {
    for (Blk& b : dev)
      if (b.p) cudaFree(b.p);
    for (Blk& b : host)
      if (b.p) cudaFreeHost(b.p);
  }
};
thread_local Staging g_stage;

// Host conversion loops over rows [0, n), split over a persistent pool of host threads when large
// (spawning threads per loop cost ~0.3 ms a loop, and the pipelined GEMM path runs a loop per
// row chunk). One loop runs at a time; the calling thread works too. An exception thrown by a row
// (kfail) is rethrown in the caller.
class RowPool {
 public:
  static RowPool& get() {
    // never destroyed: workers may still wait at process exit. A forked child has none of the
    // parent's worker threads, so it builds its own pool.
    static std::mutex mu;
    static RowPool* p = nullptr;
    static pid_t owner = 0;
    std::lock_guard<std::mutex> lk(mu);
    if (!p || owner != getpid()) {
      p = new RowPool();
      owner = getpid();
    }
    return *p;
  }
  int threads() const { return static_cast<int>(th_.size()) + 1; }
  void run(int64_t n, int64_t grain, const std::function<void(int64_t)>& f) {
    std::lock_guard<std::mutex> job(job_mu_);
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &f;
      n_ = n;
      grain_ = std::max<int64_t>(1, grain);
      next_.store(0);
      err_ = nullptr;
      active_ = static_cast<int>(th_.size());
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return active_ == 0; });
    fn_ = nullptr;
    if (err_) std::rethrow_exception(err_);
  }

 private:
  RowPool() {
    const int nt = static_cast<int>(std::min<unsigned>(std::max(1u, std::thread::hardware_concurrency()), 16u));
    for (int t = 1; t < nt; ++t)
      th_.emplace_back([this] {
        uint64_t seen = 0;
        for (;;) {
          {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return gen_ != seen; });
            seen = gen_;
          }
          work();
          std::lock_guard<std::mutex> lk(mu_);
          if (--active_ == 0) done_cv_.notify_all();
        }
      });
    for (auto& t : th_) t.detach();
  }
  void work() {
    for (;;) {
      const int64_t i0 = next_.fetch_add(grain_);
      if (i0 >= n_) return;
      try {
        for (int64_t i = i0; i < std::min(n_, i0 + grain_); ++i) (*fn_)(i);
      } catch (...) {
        std::lock_guard<std::mutex> lk(mu_);
        if (!err_) err_ = std::current_exception();
        next_.store(n_);
      }
    }
  }
  std::vector<std::thread> th_;
  std::mutex job_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int64_t)>* fn_ = nullptr;
  int64_t n_ = 0, grain_ = 1;
  std::atomic<int64_t> next_{0};
  std::exception_ptr err_;
  int active_ = 0;
  uint64_t gen_ = 0;
};

template <class F>
void parallel_rows(int64_t n, int64_t work_per_row, F&& f) {
  const int64_t work = n * std::max<int64_t>(1, work_per_row);
  if (work < (int64_t(1) << 20) || n < 2) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  RowPool& pool = RowPool::get();
  // ~4 grains per thread: balance without per-row atomics
  const int64_t grain = std::max<int64_t>(1, n / (4 * pool.threads()));
  const std::function<void(int64_t)> fn = [&](int64_t i) { f(i); };
  pool.run(n, grain, fn);
}

const Op* def_of(const std::vector<Op>& ops, const std::string& v) {
  for (const Op& o : ops)
    if (o.res == v) return &o;
  return nullptr;
}
const Op* def_any(const Kernel& g, const std::string& v) {
  if (auto* o = def_of(g.body, v)) return o;
  if (auto* o = def_of(g.pro, v)) return o;
  return def_of(g.epi, v);
}
int iter_index(const Kernel& g, const std::string& v) {
  for (size_t i = 0; i < g.iter.size(); ++i)
    if (g.iter[i].first == v) return static_cast<int>(i);
  return -1;
}
const Op* yield_op(const Kernel& g) {
  for (const Op& o : g.body)
    if (o.k == K::Yield) return &o;
  return nullptr;
}
std::vector<const Op*> tile_ops(const std::vector<Op>& ops) {
  std::vector<const Op*> r;
  for (const Op& o : ops)
    if (o.k == K::Load || o.k == K::Dot || o.k == K::Ew || o.k == K::Reduce || o.k == K::ConstTile) r.push_back(&o);
  return r;
}
const Op* const_1x1(const Kernel& g, const std::string& v) {
  const Op* c = def_any(g, v);
  return (c && c->k == K::ConstTile && !c->zeros && c->shape.r == 1 && c->shape.c == 1) ? c : nullptr;
}
bool zeros_tile(const Kernel& g, const std::string& v) {
  const Op* c = def_any(g, v);
  return c && c->k == K::ConstTile && c->zeros;
}

// Per-pid scalar state: the prologue run, iter args initialised; step() runs one iteration's
// body and advances the scalar iter args through the yield.
struct PidEval {
  const Kernel& g;
  ScalarEnv env;
  PidEval(const Kernel& k, int64_t pid) : g(k) {
    env.run(g.pro, pid);
    for (auto& [a, init] : g.iter)
      if (env.v.count(init)) env.v[a] = env.v[init];
    pid_ = pid;
  }
  ScalarEnv step(int64_t j) {
    ScalarEnv e2 = env;
    e2.v[g.ind] = j;
    e2.run(g.body, pid_);
    const Op* y = yield_op(g);
    if (y)
      for (size_t i = 0; i < g.iter.size() && i < y->args.size(); ++i)
        if (e2.v.count(y->args[i])) env.v[g.iter[i].first] = e2.v[y->args[i]];
    return e2;
  }
  int64_t pid_;
};

// int payloads run exactly when every value is exact in the device type and every partial sum
// of the fp32 accumulation stays below 2^24; the requested 16-bit type is kept when it is exact,
// else fp16 (integers up to 2048) when that is
int exact_int_dtype(int dt, double amax_inputs) {
  const double lim = dt == WS_BF16 ? 256.0 : 2048.0;
  if (amax_inputs <= lim) return dt;
  if (amax_inputs <= 2048.0) return WS_F16;
  kfail(WS_UNSUPPORTED_KERNEL, "int payloads with |x| > 2048 are not exact in a 16-bit tensor-core type");
}

// ------------------------------------------------------------------------------------------------
// gemm.k family
// ------------------------------------------------------------------------------------------------
struct PidTile {
  int64_t pid, r0, c0, ra, rb, ka0, kb0;
};

void gemm_launch_knobs(ws_gemm_desc& d, const Plan& pl, int64_t Kp) {
  d.D = pl.d;
  d.P = pl.p;
  d.persistent = pl.persistent ? 1 : 0;
  d.cta_pair = pl.coop == 0 ? (Kp >= 1024 ? 1 : 0) : pl.coop == 2 ? 1 : 0;
}

bool try_gemm(const Kernel& g, std::map<std::string, HostBuf>& bufs, int64_t lo, int64_t hi, int dt, const Plan& pl,
              cudaStream_t st);

// Several independent dot chains in one loop (the reference's `twochain` test kernels,
// ref proj/tests/support/kernel_gen.hpp:55-78: u += a.a^T, v += b.b^T, stored to c and d): each
// chain — its loads, its dot, an optional relu of it, and the store of its accumulator — is cut
// out into a single-chain kernel and run as one gemm. All chains are validated before any runs.
bool try_gemm_chains(const Kernel& g, std::map<std::string, HostBuf>& bufs, int64_t lo, int64_t hi, int dt,
                     const Plan& pl, cudaStream_t st) {
  std::vector<const Op*> dots;
  for (const Op* o : tile_ops(g.body))
    if (o->k == K::Dot) dots.push_back(o);
  if (dots.size() < 2) return false;
  std::vector<Kernel> parts;
  std::set<const Op*> used_body, used_store;
  for (const Op* d : dots) {
    Kernel gk = g;
    std::set<std::string> keep = {d->res, d->args[0], d->args[1]};
    for (const Op& o : g.body)  // a relu of this chain's new accumulator belongs to it
      if (o.k == K::Ew && o.fn == "relu" && o.args.size() == 1 && o.args[0] == d->res) keep.insert(o.res);
    // iter args carrying this chain's values (acc, relu) and the epilogue values derived from them
    std::set<std::string> carried;
    const Op* y = yield_op(g);
    if (!y) return false;
    for (size_t i = 0; i < y->args.size() && i < g.iter.size(); ++i)
      if (keep.count(y->args[i])) carried.insert(g.iter[i].first);
    gk.body.clear();
    for (const Op& o : g.body) {
      const bool tile = o.k == K::Load || o.k == K::Dot || o.k == K::Ew || o.k == K::Reduce;
      if (!tile || keep.count(o.res)) {
        gk.body.push_back(o);
        if (tile) used_body.insert(&o);
      }
    }
    gk.epi.clear();
    for (const Op& o : g.epi) {
      if (o.k == K::Store) {
        std::string v = o.args.empty() ? "" : o.args[0];
        if (const Op* m = def_of(g.epi, v); m && m->k == K::Ew && m->fn == "mul") v = m->args[0];
        if (!carried.count(v)) continue;
        used_store.insert(&o);
      } else if (o.k == K::Ew && o.fn == "mul" && !carried.count(o.args.empty() ? "" : o.args[0])) {
        continue;
      }
      gk.epi.push_back(o);
    }
    // structure check only (an empty pid range runs nothing)
    if (!try_gemm(gk, bufs, lo, lo, dt, pl, st)) return false;
    parts.push_back(std::move(gk));
  }
  for (const Op* o : tile_ops(g.body))
    if (o->k != K::ConstTile && !used_body.count(o)) return false;  // a tile op outside every chain
  for (const Op& o : g.epi)
    if (o.k == K::Store && !used_store.count(&o)) return false;
  for (const Kernel& gk : parts)
    if (!try_gemm(gk, bufs, lo, hi, dt, pl, st)) return false;
  return true;
}

bool try_gemm(const Kernel& g, std::map<std::string, HostBuf>& bufs, int64_t lo, int64_t hi, int dt, const Plan& pl,
              cudaStream_t st) {
  // body: the loads and one dot(a, b.T, acc=<iter arg>) (a and b may be one load: a Gram product),
  // optional relu of the new acc, yield; prologue acc init = zeros; epilogue: store of the acc (or
  // of the relu'd iter arg), or of `ew mul acc, <1x1 const>`
  const Op* dot = nullptr;
  std::vector<const Op*> loads;
  const Op* relu = nullptr;
  for (const Op* o : tile_ops(g.body)) {
    if (o->k == K::Load) loads.push_back(o);
    else if (o->k == K::Dot) {
      if (dot) return try_gemm_chains(g, bufs, lo, hi, dt, pl, st);
      dot = o;
    } else if (o->k == K::Ew && o->fn == "relu" && !relu) relu = o;
    else return false;
  }
  if (!dot || !dot->trans) return false;
  if (loads.size() != 2 && !(loads.size() == 1 && dot->args[0] == dot->args[1])) return false;
  const Op* la = def_of(g.body, dot->args[0]);
  const Op* lb = def_of(g.body, dot->args[1]);
  if (!la || !lb || la->k != K::Load || lb->k != K::Load) return false;
  const Op* y = yield_op(g);
  if (!y) return false;
  const int acc_i = iter_index(g, dot->args[2]);
  if (acc_i < 0 || y->args[acc_i] != dot->res) return false;
  const Op* acc_init = def_of(g.pro, g.iter[acc_i].second);
  if (!acc_init || acc_init->k != K::ConstTile || !acc_init->zeros) return false;
  int relu_i = -1;
  if (relu) {
    if (relu->args[0] != dot->res) return false;
    for (size_t i = 0; i < y->args.size(); ++i)
      if (y->args[i] == relu->res) relu_i = static_cast<int>(i);
    if (relu_i < 0) return false;
  }
  // epilogue
  const Op* store = nullptr;
  const Op* scale_op = nullptr;
  for (const Op* o : tile_ops(g.epi)) {
    if (o->k == K::Ew && o->fn == "mul" && !scale_op) scale_op = o;
    else if (o->k == K::ConstTile) continue;
    else return false;
  }
  for (const Op& o : g.epi)
    if (o.k == K::Store) {
      if (store) return false;
      store = &o;
    }
  if (!store) return false;
  bool act_relu = false;
  double scale = 1.0;
  std::string stored = store->args[0];
  if (scale_op) {
    if (stored != scale_op->res) return false;
    const Op* c = const_1x1(g, scale_op->args[1]);
    if (!c) return false;
    scale = c->lit[0];
    stored = scale_op->args[0];
  }
  const int si = iter_index(g, stored);
  if (si == acc_i) {
    act_relu = false;
  } else if (relu && si == relu_i) {
    act_relu = true;
  } else {
    return false;
  }
  const HostBuf& A = bufs.at(la->buf);
  const HostBuf& B = bufs.at(lb->buf);
  HostBuf& C = bufs.at(store->buf);
  const int64_t BM = la->shape.r, BKa = la->shape.c, BN = lb->shape.r, BKb = lb->shape.c;
  if (BKa != BKb || dot->args.size() != 3) return false;
  const int64_t trip = g.hi - g.lo;
  if (trip < 1) return false;

  // per-pid geometry from the scalar program (and linear K offsets across iterations)
  std::vector<PidTile> tiles;
  for (int64_t pid = lo; pid < hi; ++pid) {
    PidEval pe(g, pid);
    int64_t ra = 0, rb = 0, ka = 0, kb = 0, ka1 = 0, kb1 = 0;
    for (int64_t k = g.lo; k < std::min(g.hi, g.lo + 2); ++k) {
      ScalarEnv e2 = pe.step(k);
      const int64_t r_a = e2.get(la->args[0]), c_a = e2.get(la->args[1]);
      const int64_t r_b = e2.get(lb->args[0]), c_b = e2.get(lb->args[1]);
      if (k == g.lo) {
        ra = r_a, rb = r_b, ka = c_a, kb = c_b;
      } else {
        if (r_a != ra || r_b != rb) kfail(WS_UNSUPPORTED_KERNEL, "tile rows change across iterations");
        ka1 = c_a, kb1 = c_b;
      }
    }
    if (trip > 1 && (ka1 - ka != BKa || kb1 - kb != BKb))
      kfail(WS_UNSUPPORTED_KERNEL, "K offsets do not advance by the tile depth");
    ScalarEnv ee = pe.env;
    ee.run(g.epi, pid);
    tiles.push_back({pid, ee.get(store->args[1]), ee.get(store->args[2]), ra, rb, ka, kb});
  }
  if (tiles.empty()) return true;
  const int64_t Kd = trip * BKa;

  // group pids that form one GEMM: same A/B row offsets relative to the C tile and same K range
  std::map<std::vector<int64_t>, std::vector<PidTile>> groups;
  for (auto& t : tiles) groups[{t.ra - t.r0, t.rb - t.c0, t.ka0, t.kb0}].push_back(t);

  // exactness of the device arithmetic for int payloads: exact operands, fp32-exact partial sums
  if (!A.shape.real || !B.shape.real) {
    const double ma = A.amax(), mb = B.amax();
    dt = exact_int_dtype(dt, std::max(ma, mb));
    if (ma * mb * static_cast<double>(Kd) >= 16777216.0)
      kfail(WS_UNSUPPORTED_KERNEL, "int payloads could overflow fp32-exact accumulation (>= 2^24)");
  }

  for (auto& kv : groups) {
    const std::vector<int64_t>& key = kv.first;
    const std::vector<PidTile>& ts = kv.second;
    const int64_t dA = key[0], dB = key[1], ka0 = key[2], kb0 = key[3];
    int64_t rmin = INT64_MAX, rmax = INT64_MIN, cmin = INT64_MAX, cmax = INT64_MIN;
    for (auto& t : ts) {
      rmin = std::min(rmin, t.r0), rmax = std::max(rmax, t.r0 + BM);
      cmin = std::min(cmin, t.c0), cmax = std::max(cmax, t.c0 + BN);
    }
    // bounds, like slice_tile / store_tile (ref tile.hpp:249-278)
    if (rmin < 0 || cmin < 0 || rmax > C.shape.r || cmax > C.shape.c || rmin + dA < 0 || rmax + dA > A.shape.r ||
        cmin + dB < 0 || cmax + dB > B.shape.r || ka0 < 0 || ka0 + Kd > A.shape.c || kb0 < 0 || kb0 + Kd > B.shape.c)
      kfail(WS_EVAL, "tile access out of bounds");
    const int64_t M = rmax - rmin, N = cmax - cmin;
    const int64_t Mp = (M + 255) / 256 * 256, Np = (N + 255) / 256 * 256, Kp = (Kd + 63) / 64 * 64;
    auto* ha = static_cast<uint16_t*>(g_stage.pinned(0, static_cast<size_t>(Mp * Kp) * 2));
    auto* hb = static_cast<uint16_t*>(g_stage.pinned(1, static_cast<size_t>(Np * Kp) * 2));
    void* da = g_stage.device(0, static_cast<size_t>(Mp * Kp) * 2);
    void* db = g_stage.device(1, static_cast<size_t>(Np * Kp) * 2);
    void* dc = g_stage.device(2, static_cast<size_t>(Mp * Np) * 4);
    // operands: converted to 16 bits and copied in row chunks, so the host->device copy of one
    // chunk runs while the host threads convert the next
    auto stage_in = [&](const HostBuf& X, int64_t rows, int64_t rows_p, int64_t r_src, int64_t k_src, uint16_t* h,
                        void* d) {
      const int64_t nch = rows_p >= 2048 ? 8 : 1;
      const double* xr = X.shape.real ? static_cast<const double*>(X.data) : nullptr;
      for (int64_t ch = 0; ch < nch; ++ch) {
        const int64_t r0 = rows_p * ch / nch, r1 = rows_p * (ch + 1) / nch;
        parallel_rows(r1 - r0, Kp, [&](int64_t i) {
          const int64_t r = r0 + i;
          uint16_t* row = h + r * Kp;
          if (r >= rows) {
            std::memset(row, 0, Kp * 2);
            return;
          }
          if (xr) {
            const double* src = xr + (r_src + r) * X.shape.c + k_src;
            for (int64_t k = 0; k < Kd; ++k) row[k] = to_half_bits(static_cast<float>(src[k]), dt);
          } else {
            for (int64_t k = 0; k < Kd; ++k) row[k] = to_half_bits(static_cast<float>(X.get(r_src + r, k_src + k)), dt);
          }
          for (int64_t k = Kd; k < Kp; ++k) row[k] = 0;
        });
        cuda_check(cudaMemcpyAsync(static_cast<uint16_t*>(d) + r0 * Kp, h + r0 * Kp, static_cast<size_t>((r1 - r0) * Kp) * 2,
                                   cudaMemcpyHostToDevice, st),
                   "H2D");
      }
    };
    stage_in(A, M, Mp, rmin + dA, ka0, ha, da);
    stage_in(B, N, Np, cmin + dB, kb0, hb, db);
    ws_gemm_desc d{};
    d.in_dtype = dt;
    d.out_dtype = WS_F32;
    d.M = Mp, d.N = Np, d.K = Kp;
    d.A = da, d.lda = Kp, d.B = db, d.ldb = Kp, d.C = dc, d.ldc = Np;
    d.scale_a = static_cast<float>(scale), d.scale_b = 1.f;
    gemm_launch_knobs(d, pl, Kp);
    d.act = act_relu ? 1 : 0;
    ws_check(ws_gemm_tn(&d, st));
    // result: copied out in row chunks; the host threads write chunk i into the caller's buffer
    // while chunk i+1 is in flight. Only the pids' own tiles are written (ref store_tile).
    auto* hc = static_cast<float*>(g_stage.pinned(2, static_cast<size_t>(Mp * Np) * 4));
    const int64_t nch = M >= 2048 ? 8 : 1;
    struct Events {  // destroyed on every exit, kfail included
      std::vector<cudaEvent_t> v;
      ~Events() {
        for (cudaEvent_t e : v) cudaEventDestroy(e);
      }
    } ev;
    ev.v.assign(static_cast<size_t>(nch), nullptr);
    std::vector<cudaEvent_t>& evs = ev.v;
    for (auto& e : evs) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    auto chunk_rows = [&](int64_t ch, int64_t& r0, int64_t& r1) {
      r0 = M * ch / nch;
      r1 = M * (ch + 1) / nch;
    };
    for (int64_t ch = 0; ch < nch; ++ch) {
      int64_t r0, r1;
      chunk_rows(ch, r0, r1);
      cuda_check(cudaMemcpyAsync(hc + r0 * Np, static_cast<float*>(dc) + r0 * Np, static_cast<size_t>((r1 - r0) * Np) * 4,
                                 cudaMemcpyDeviceToHost, st),
                 "D2H");
      cuda_check(cudaEventRecord(evs[static_cast<size_t>(ch)], st), "event");
    }
    double* cr = C.shape.real ? static_cast<double*>(C.data) : nullptr;
    for (int64_t ch = 0; ch < nch; ++ch) {
      int64_t r0, r1;  // rows relative to rmin
      chunk_rows(ch, r0, r1);
      cuda_check(cudaEventSynchronize(evs[static_cast<size_t>(ch)]), "sync");
      parallel_rows(static_cast<int64_t>(ts.size()), BM * BN / nch, [&](int64_t i) {
        const PidTile& t = ts[static_cast<size_t>(i)];
        const int64_t lo_r = std::max(t.r0 - rmin, r0), hi_r = std::min(t.r0 - rmin + BM, r1);
        for (int64_t rr = lo_r; rr < hi_r; ++rr) {
          const float* src = hc + rr * Np + (t.c0 - cmin);
          const int64_t r = rmin + rr;
          if (cr) {
            double* dst = cr + r * C.shape.c + t.c0;
            for (int64_t c = 0; c < BN; ++c) dst[c] = src[c];
          } else {
            for (int64_t c = 0; c < BN; ++c) C.set(r, t.c0 + c, src[c]);
          }
        }
      });
    }
  }
  return true;
}

// ------------------------------------------------------------------------------------------------
// flash .k
// ------------------------------------------------------------------------------------------------
// The whole dataflow of the .k is matched, op by op (operand order of commutative ops free):
//   s  = dot q_tile, k_tile.T, acc = zeros | mask-bank tile      ss = ew mul s, <1x1 scale>
//   rm = reduce max ss axis=1     mn = ew max m, rm              d  = ew sub ss, mn
//   pp = ew exp d                 dm = ew sub m, mn              al = ew exp dm
//   rs = reduce add pp axis=1     la = ew mul l, al              l1 = ew add la, rs
//   as = ew mul acc, al           acc1 = dot pp, v_tile, acc = as
//   yield acc1 -> acc, mn -> m, l1 -> l;  stores of acc, l and m in the epilogue
// with acc, l starting at zeros and m at a constant <= -1e4. Any other tile op — a bias, a
// padding mask, a different rescale — makes the kernel unsupported rather than misread.
bool try_flash(const Kernel& g, std::map<std::string, HostBuf>& bufs, int64_t lo, int64_t hi, int dt, const Plan& pl,
               cudaStream_t st) {
  std::vector<const Op*> dots;
  for (const Op* o : tile_ops(g.body))
    if (o->k == K::Dot) dots.push_back(o);
  if (dots.size() != 2) return false;
  const Op* qk = dots[0]->trans ? dots[0] : dots[1];
  const Op* pv = dots[0]->trans ? dots[1] : dots[0];
  if (!qk->trans || pv->trans) return false;
  const Op* y = yield_op(g);
  if (!y || y->args.size() != g.iter.size()) return false;
  auto body = [&](const std::string& v) { return def_of(g.body, v); };
  // score scaling and row max
  const Op *ss = nullptr, *rm = nullptr, *mn = nullptr, *dd = nullptr, *pp = nullptr, *dm = nullptr, *al = nullptr,
           *rs = nullptr, *la = nullptr, *l1 = nullptr, *as = nullptr;
  const Op* sc = nullptr;
  for (const Op& o : g.body)
    if (o.k == K::Ew && o.fn == "mul" && o.args.size() == 2 && (o.args[0] == qk->res || o.args[1] == qk->res)) {
      sc = const_1x1(g, o.args[0] == qk->res ? o.args[1] : o.args[0]);
      if (sc) ss = &o;
    }
  if (!ss || sc->lit[0] <= 0) return false;
  // acc1 = dot pp, tv, acc = as
  pp = body(pv->args[0]);
  as = body(pv->args[2]);
  const Op* lv = body(pv->args[1]);
  if (!pp || !as || !lv || lv->k != K::Load) return false;
  if (pp->k != K::Ew || pp->fn != "exp" || pp->args.size() != 1) return false;
  dd = body(pp->args[0]);
  if (!dd || dd->k != K::Ew || dd->fn != "sub" || dd->args.size() != 2 || dd->args[0] != ss->res) return false;
  mn = body(dd->args[1]);
  if (!mn || mn->k != K::Ew || mn->fn != "max" || mn->args.size() != 2) return false;
  // mn = max(m, rm), rm = reduce max ss axis 1
  const std::string m_it = iter_index(g, mn->args[0]) >= 0 ? mn->args[0] : mn->args[1];
  rm = body(m_it == mn->args[0] ? mn->args[1] : mn->args[0]);
  if (iter_index(g, m_it) < 0 || !rm || rm->k != K::Reduce || rm->fn != "max" || rm->axis != 1 ||
      rm->args[0] != ss->res)
    return false;
  // as = acc * al, al = exp(m - mn)
  const std::string acc_it = iter_index(g, as->args[0]) >= 0 ? as->args[0] : as->args.size() > 1 ? as->args[1] : "";
  if (as->k != K::Ew || as->fn != "mul" || as->args.size() != 2 || iter_index(g, acc_it) < 0) return false;
  al = body(acc_it == as->args[0] ? as->args[1] : as->args[0]);
  if (!al || al->k != K::Ew || al->fn != "exp" || al->args.size() != 1) return false;
  dm = body(al->args[0]);
  if (!dm || dm->k != K::Ew || dm->fn != "sub" || dm->args.size() != 2 || dm->args[0] != m_it || dm->args[1] != mn->res)
    return false;
  // l1 = l * al + rowsum(pp)
  for (const Op& o : g.body) {
    if (o.k == K::Reduce && o.fn == "add" && o.axis == 1 && o.args[0] == pp->res) rs = &o;
  }
  if (!rs) return false;
  for (const Op& o : g.body)
    if (o.k == K::Ew && o.fn == "add" && o.args.size() == 2 && (o.args[0] == rs->res || o.args[1] == rs->res)) {
      const Op* cand = body(o.args[0] == rs->res ? o.args[1] : o.args[0]);
      if (cand && cand->k == K::Ew && cand->fn == "mul" && cand->args.size() == 2 &&
          (cand->args[0] == al->res || cand->args[1] == al->res)) {
        la = cand;
        l1 = &o;
      }
    }
  if (!la || !l1) return false;
  const std::string l_it = la->args[0] == al->res ? la->args[1] : la->args[0];
  const int ia = iter_index(g, acc_it), im = iter_index(g, m_it), il = iter_index(g, l_it);
  if (ia < 0 || im < 0 || il < 0 || ia == im || ia == il || im == il) return false;
  if (y->args[ia] != pv->res || y->args[im] != mn->res || y->args[il] != l1->res) return false;
  // loads and the QK accumulator
  const Op* lq = body(qk->args[0]);
  const Op* lk = body(qk->args[1]);
  if (!lq || !lk || lq->k != K::Load || lk->k != K::Load) return false;
  const Op* s_init = def_any(g, qk->args[2]);
  if (!s_init) return false;
  const bool causal = s_init->k == K::Load;
  if (!causal && !zeros_tile(g, qk->args[2])) return false;
  // nothing else in the body: every tile op is one of the matched ones
  std::set<const Op*> known = {qk, pv, ss, rm, mn, dd, pp, dm, al, rs, la, l1, as, lq, lk, lv};
  if (causal) known.insert(s_init);
  for (const Op* o : tile_ops(g.body))
    if (!known.count(o) && !(o->k == K::ConstTile)) kfail(WS_UNSUPPORTED_KERNEL, "flash kernel has an extra tile op '" + o->res + "'");
  // initial values: acc and l zeros, m a large negative constant (the .k's -1e6)
  if (!zeros_tile(g, g.iter[ia].second) || !zeros_tile(g, g.iter[il].second)) return false;
  {
    const Op* m0 = def_of(g.pro, g.iter[im].second);
    double v0 = 1;
    if (m0 && m0->k == K::ConstTile && !m0->zeros) {
      v0 = *std::max_element(m0->lit.begin(), m0->lit.end());
    } else if (m0 && m0->k == K::Ew && m0->fn == "add" && m0->args.size() == 2) {
      const Op* c = const_1x1(g, m0->args[0]) ? const_1x1(g, m0->args[0]) : const_1x1(g, m0->args[1]);
      const std::string z = c == const_1x1(g, m0->args[0]) ? m0->args[1] : m0->args[0];
      if (c && zeros_tile(g, z)) v0 = c->lit[0];
    }
    if (v0 > -1e4) return false;
  }
  // outputs: stores of the three iter args acc (pv chain), l (row sums), m (running max); nothing
  // else in the epilogue
  std::string o_buf, l_buf, m_buf;
  for (const Op& s : g.epi) {
    if (s.k == K::Store) {
      const int i = iter_index(g, s.args[0]);
      if (i == ia) o_buf = s.buf;
      else if (i == il) l_buf = s.buf;
      else if (i == im) m_buf = s.buf;
      else return false;
    } else if (s.k != K::Arith && s.k != K::Const && s.k != K::Pid) {
      return false;
    }
  }
  if (o_buf.empty() || l_buf.empty() || m_buf.empty()) return false;
  const double scale = sc->lit[0];
  const HostBuf& Q = bufs.at(lq->buf);
  const HostBuf& Kb = bufs.at(lk->buf);
  const HostBuf& V = bufs.at(lv->buf);
  const int64_t BR = lq->shape.r, D = lq->shape.c, BC = lk->shape.r;
  const int64_t trip = g.hi - g.lo, S = trip * BC;
  if (S <= 0 || Q.shape.r % S != 0 || Kb.shape.r != Q.shape.r || V.shape.r != Q.shape.r || Q.shape.c != D ||
      lk->shape.c != D || lv->shape.r != BC || lv->shape.c != D || Kb.shape.c != D || V.shape.c != D)
    return false;
  const int64_t BH = Q.shape.r / S;
  const int64_t nqb = S / BR;
  if (S % BR) return false;
  // causal: the mask bank tile is BR x BC from a BR x 3BC bank [0 | lower-triangular | masked],
  // block 0 below the diagonal, 1 on it, 2 above (BR == BC so diagonal blocks are square)
  const HostBuf* MB = causal ? &bufs.at(s_init->buf) : nullptr;
  if (causal) {
    if (BR != BC || s_init->shape.r != BR || s_init->shape.c != BC || MB->shape.r != BR || MB->shape.c < 3 * BC)
      kfail(WS_UNSUPPORTED_KERNEL, "flash mask bank is not the [0 | causal | masked] layout");
    for (int64_t r = 0; r < BR; ++r)
      for (int64_t c = 0; c < 3 * BC; ++c) {
        const int blk = static_cast<int>(c / BC);
        const int64_t cc = c % BC;
        const bool masked = blk == 2 || (blk == 1 && cc > r);
        const double v = MB->get(r, c);
        if (masked ? !(v <= -1e5) : v != 0.0)
          kfail(WS_UNSUPPORTED_KERNEL, "flash mask bank is not causal (mb[" + std::to_string(r) + "," +
                                           std::to_string(c) + "] = " + std::to_string(v) + ")");
      }
  }
  // the pid geometry, on every pid that runs and every iteration: q rows = pid*BR (col 0); k/v
  // rows (b,h)*S + j*BC (col 0); causal mask block = 0 / 1 / 2 below / on / above the diagonal
  for (int64_t pid = lo; pid < hi; ++pid) {
    PidEval pe(g, pid);
    const int64_t bh = pid / nqb, qb = pid % nqb;
    for (int64_t j = g.lo; j < g.hi; ++j) {
      ScalarEnv e2 = pe.step(j);
      const int64_t jj = j - g.lo;
      if (e2.get(lq->args[0]) != pid * BR || e2.get(lq->args[1]) != 0 || e2.get(lk->args[0]) != bh * S + jj * BC ||
          e2.get(lk->args[1]) != 0 || e2.get(lv->args[0]) != bh * S + jj * BC || e2.get(lv->args[1]) != 0)
        kfail(WS_UNSUPPORTED_KERNEL, "flash kernel pid geometry differs from the batched (b,h)-major layout");
      if (causal) {
        const int64_t want = jj < qb ? 0 : jj == qb ? BC : 2 * BC;
        if (e2.get(s_init->args[0]) != 0 || e2.get(s_init->args[1]) != want)
          kfail(WS_UNSUPPORTED_KERNEL, "flash mask selection is not the causal block selector");
      }
      if (j - g.lo >= 1 && !causal) break;  // non-causal: the affine k/v walk is checked on two steps
    }
  }
  if ((D != 64 && D != 128) || S % 128 != 0)
    kfail(WS_UNSUPPORTED_KERNEL, "flash on B200 needs head dim 64/128 and S % 128 == 0 (S=" + std::to_string(S) +
                                     ", D=" + std::to_string(D) + ")");
  // the stored tiles (all rows of pids [lo, hi)) must be the q rows, at column 0
  const int64_t bh0 = lo / nqb, bh1 = (hi - 1) / nqb + 1;
  const size_t n = static_cast<size_t>(BH * S * D);
  const size_t nr = static_cast<size_t>((bh1 - bh0) * S * D), off = static_cast<size_t>(bh0 * S * D);
  auto* hq = static_cast<uint16_t*>(g_stage.pinned(0, nr * 2));
  auto* hk = static_cast<uint16_t*>(g_stage.pinned(1, nr * 2));
  auto* hv = static_cast<uint16_t*>(g_stage.pinned(2, nr * 2));
  parallel_rows((bh1 - bh0) * S, D, [&](int64_t r) {
    for (int64_t c = 0; c < D; ++c) {
      const size_t i = static_cast<size_t>(r * D + c);
      hq[i] = to_half_bits(static_cast<float>(Q.get(bh0 * S + r, c)), dt);
      hk[i] = to_half_bits(static_cast<float>(Kb.get(bh0 * S + r, c)), dt);
      hv[i] = to_half_bits(static_cast<float>(V.get(bh0 * S + r, c)), dt);
    }
  });
  auto* dq = static_cast<uint16_t*>(g_stage.device(0, n * 2));
  auto* dk = static_cast<uint16_t*>(g_stage.device(1, n * 2));
  auto* dv = static_cast<uint16_t*>(g_stage.device(2, n * 2));
  auto* dout = static_cast<uint16_t*>(g_stage.device(3, n * 2));
  auto* dlse = static_cast<float*>(g_stage.device(4, static_cast<size_t>(BH * S) * 4));
  auto* dmx = static_cast<float*>(g_stage.device(5, static_cast<size_t>(BH * S) * 4));
  cuda_check(cudaMemcpyAsync(dq + off, hq, nr * 2, cudaMemcpyHostToDevice, st), "H2D");
  cuda_check(cudaMemcpyAsync(dk + off, hk, nr * 2, cudaMemcpyHostToDevice, st), "H2D");
  cuda_check(cudaMemcpyAsync(dv + off, hv, nr * 2, cudaMemcpyHostToDevice, st), "H2D");
  ws_attn_desc a{};
  a.dtype = dt;
  a.B = 1, a.H = static_cast<int32_t>(BH), a.S = static_cast<int32_t>(S), a.Dh = static_cast<int32_t>(D);
  a.causal = causal;
  a.softmax_scale = static_cast<float>(scale);
  a.Q = dq, a.K = dk, a.V = dv, a.O = dout, a.LSE = dlse, a.MX = dmx;
  a.bh_begin = static_cast<int32_t>(bh0), a.bh_end = static_cast<int32_t>(bh1);
  a.D = pl.d == 0 ? 0 : std::max(pl.d, 2);  // none / plain ws programs: the smallest ring
  a.grid_per_item = pl.persistent ? 2 : 1;
  ws_check(ws_attn_fwd(&a, st));
  auto* ho = static_cast<uint16_t*>(g_stage.pinned(3, nr * 2));
  auto* hl = static_cast<float*>(g_stage.pinned(4, static_cast<size_t>((bh1 - bh0) * S) * 4));
  auto* hm = static_cast<float*>(g_stage.pinned(5, static_cast<size_t>((bh1 - bh0) * S) * 4));
  cuda_check(cudaMemcpyAsync(ho, dout + off, nr * 2, cudaMemcpyDeviceToHost, st), "D2H");
  cuda_check(cudaMemcpyAsync(hl, dlse + bh0 * S, static_cast<size_t>((bh1 - bh0) * S) * 4, cudaMemcpyDeviceToHost, st),
             "D2H");
  cuda_check(cudaMemcpyAsync(hm, dmx + bh0 * S, static_cast<size_t>((bh1 - bh0) * S) * 4, cudaMemcpyDeviceToHost, st),
             "D2H");
  cuda_check(cudaStreamSynchronize(st), "sync");
  // The .k's outputs: m = the exact running max, l = sum exp(ss - m) = exp(lse - m), and the
  // un-normalised accumulator acc = O * l.
  HostBuf& O = bufs.at(o_buf);
  HostBuf& L = bufs.at(l_buf);
  HostBuf& Mx = bufs.at(m_buf);
  parallel_rows(hi - lo, BR * D, [&](int64_t i) {
    const int64_t pid = lo + i;
    for (int64_t r = pid * BR; r < pid * BR + BR; ++r) {
      const int64_t rr = r - bh0 * S;
      const double m = hm[rr], l = std::exp(static_cast<double>(hl[rr]) - m);
      for (int64_t c = 0; c < D; ++c) O.set(r, c, static_cast<double>(half_to_float(ho[rr * D + c], dt)) * l);
      L.set(r, 0, l);
      Mx.set(r, 0, m);
    }
  });
  return true;
}

// ------------------------------------------------------------------------------------------------
// max-shift attention (ref proj/kernels/attention.k:1-21)
// ------------------------------------------------------------------------------------------------
// s = q_tile . k_tile^T (acc zeros); m = rowmax s; acc += (s - m) . v_tile, per iteration. On the
// GPU: one GEMM for every score block of every pid (S = Q . Kstack^T, fp32), a row-block shift
// kernel (P = S - blockwise row max, 16-bit), one GEMM for the accumulation (acc = P . Vstack).
// Exact for int payloads while |s - m| and the inputs are exact in the 16-bit type and the
// accumulator stays below 2^24.
__global__ void ws_rowblock_shift_kernel(const float* __restrict__ s, int64_t lds, uint16_t* __restrict__ p,
                                         int64_t ldp, int rows, int valid_cols, int bc, int nblk_pad, int f16) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t r = idx / nblk_pad, b = idx % nblk_pad;
  if (r >= rows) return;
  const float* sr = s + r * lds + b * bc;
  uint16_t* pr = p + r * ldp + b * bc;
  if (b * bc >= valid_cols) {
    for (int c = 0; c < bc; ++c) pr[c] = 0;
    return;
  }
  float m = sr[0];
  for (int c = 1; c < bc; ++c) m = fmaxf(m, sr[c]);
  for (int c = 0; c < bc; ++c) {
    const float x = sr[c] - m;
    pr[c] = f16 ? __half_as_ushort(__float2half_rn(x)) : __bfloat16_as_ushort(__float2bfloat16_rn(x));
  }
}

bool try_maxshift(const Kernel& g, std::map<std::string, HostBuf>& bufs, int64_t lo, int64_t hi, int dt,
                  const Plan& pl, cudaStream_t st) {
  std::vector<const Op*> dots;
  for (const Op* o : tile_ops(g.body))
    if (o->k == K::Dot) dots.push_back(o);
  if (dots.size() != 2) return false;
  const Op* qk = dots[0]->trans ? dots[0] : dots[1];
  const Op* pv = dots[0]->trans ? dots[1] : dots[0];
  if (!qk->trans || pv->trans) return false;
  auto body = [&](const std::string& v) { return def_of(g.body, v); };
  const Op* sub = body(pv->args[0]);
  if (!sub || sub->k != K::Ew || sub->fn != "sub" || sub->args.size() != 2 || sub->args[0] != qk->res) return false;
  const Op* rm = body(sub->args[1]);
  if (!rm || rm->k != K::Reduce || rm->fn != "max" || rm->axis != 1 || rm->args[0] != qk->res) return false;
  if (!zeros_tile(g, qk->args[2])) return false;
  const Op* lq = body(qk->args[0]);
  const Op* lk = body(qk->args[1]);
  const Op* lv = body(pv->args[1]);
  if (!lq || !lk || !lv || lq->k != K::Load || lk->k != K::Load || lv->k != K::Load) return false;
  const Op* y = yield_op(g);
  const int ia = iter_index(g, pv->args[2]);
  if (!y || ia < 0 || y->args[ia] != pv->res || !zeros_tile(g, g.iter[ia].second)) return false;
  std::set<const Op*> known = {qk, pv, sub, rm, lq, lk, lv};
  for (const Op* o : tile_ops(g.body))
    if (!known.count(o) && o->k != K::ConstTile) return false;
  const Op* store = nullptr;
  for (const Op& o : g.epi) {
    if (o.k == K::Store) {
      if (store || iter_index(g, o.args[0]) != ia) return false;
      store = &o;
    } else if (o.k != K::Arith && o.k != K::Const && o.k != K::Pid) {
      return false;
    }
  }
  if (!store) return false;
  const int64_t BR = lq->shape.r, D = lq->shape.c, BC = lk->shape.r, DV = lv->shape.c;
  if (lk->shape.c != D || lv->shape.r != BC) return false;
  const HostBuf& Q = bufs.at(lq->buf);
  const HostBuf& Kt = bufs.at(lk->buf);
  const HostBuf& V = bufs.at(lv->buf);
  HostBuf& O = bufs.at(store->buf);
  const int64_t trip = g.hi - g.lo;
  if (trip < 1) return false;
  // geometry: q tile per pid (fixed across iterations); k / v tiles per iteration, the same for
  // every pid (one shared key/value sequence)
  std::vector<std::pair<int64_t, int64_t>> kc, vc;
  struct PidRows {
    int64_t qr, qc, orow, ocol;
  };
  std::vector<PidRows> pr;
  for (int64_t pid = lo; pid < hi; ++pid) {
    PidEval pe(g, pid);
    PidRows x{};
    for (int64_t j = g.lo; j < g.hi; ++j) {
      ScalarEnv e2 = pe.step(j);
      const int64_t jj = j - g.lo;
      const std::pair<int64_t, int64_t> kk{e2.get(lk->args[0]), e2.get(lk->args[1])},
          vv{e2.get(lv->args[0]), e2.get(lv->args[1])};
      if (pid == lo) {
        kc.push_back(kk);
        vc.push_back(vv);
      } else if (kc[jj] != kk || vc[jj] != vv) {
        kfail(WS_UNSUPPORTED_KERNEL, "max-shift attention: key/value tiles differ between pids");
      }
      const int64_t r = e2.get(lq->args[0]), c = e2.get(lq->args[1]);
      if (jj == 0) x.qr = r, x.qc = c;
      else if (r != x.qr || c != x.qc) kfail(WS_UNSUPPORTED_KERNEL, "max-shift attention: the query tile moves");
    }
    ScalarEnv ee = pe.env;
    ee.run(g.epi, pid);
    x.orow = ee.get(store->args[1]);
    x.ocol = ee.get(store->args[2]);
    pr.push_back(x);
  }
  if (pr.empty()) return true;
  auto oob = [](const HostBuf& b, int64_t r, int64_t c, int64_t R, int64_t C) {
    return r < 0 || c < 0 || r + R > b.shape.r || c + C > b.shape.c;
  };
  for (auto& x : pr)
    if (oob(Q, x.qr, x.qc, BR, D) || oob(O, x.orow, x.ocol, BR, DV)) kfail(WS_EVAL, "tile access out of bounds");
  for (int64_t j = 0; j < trip; ++j)
    if (oob(Kt, kc[j].first, kc[j].second, BC, D) || oob(V, vc[j].first, vc[j].second, BC, DV))
      kfail(WS_EVAL, "tile access out of bounds");
  // exactness: inputs exact in the 16-bit type, |s - m| <= 2 max|q| max|k| D exact, and the
  // accumulator below 2^24
  const bool ints = !Q.shape.real || !Kt.shape.real || !V.shape.real;
  if (ints) {
    const double mq = Q.amax(), mk = Kt.amax(), mv = V.amax();
    const double shift = 2.0 * mq * mk * static_cast<double>(D);
    dt = exact_int_dtype(dt, std::max({mq, mk, mv, shift}));
    if (mq * mk * static_cast<double>(D) >= 16777216.0 || shift * mv * static_cast<double>(trip * BC) >= 16777216.0)
      kfail(WS_UNSUPPORTED_KERNEL, "int payloads could overflow fp32-exact accumulation (>= 2^24)");
  }
  const int64_t npid = static_cast<int64_t>(pr.size());
  const int64_t M = npid * BR, Mp = (M + 255) / 256 * 256;
  const int64_t N1 = trip * BC, Np = (N1 + 255) / 256 * 256;
  const int64_t Kp = (D + 63) / 64 * 64;
  const int64_t DVp = (DV + 255) / 256 * 256;
  auto* hq = static_cast<uint16_t*>(g_stage.pinned(0, static_cast<size_t>(Mp * Kp) * 2));
  auto* hk = static_cast<uint16_t*>(g_stage.pinned(1, static_cast<size_t>(Np * Kp) * 2));
  auto* hv = static_cast<uint16_t*>(g_stage.pinned(2, static_cast<size_t>(DVp * Np) * 2));
  std::memset(hq, 0, static_cast<size_t>(Mp * Kp) * 2);
  std::memset(hk, 0, static_cast<size_t>(Np * Kp) * 2);
  std::memset(hv, 0, static_cast<size_t>(DVp * Np) * 2);
  for (int64_t i = 0; i < npid; ++i)
    for (int64_t r = 0; r < BR; ++r)
      for (int64_t c = 0; c < D; ++c)
        hq[(i * BR + r) * Kp + c] = to_half_bits(static_cast<float>(Q.get(pr[i].qr + r, pr[i].qc + c)), dt);
  for (int64_t j = 0; j < trip; ++j)
    for (int64_t r = 0; r < BC; ++r) {
      for (int64_t c = 0; c < D; ++c)
        hk[(j * BC + r) * Kp + c] = to_half_bits(static_cast<float>(Kt.get(kc[j].first + r, kc[j].second + c)), dt);
      for (int64_t c = 0; c < DV; ++c)  // V^T: [value column][key]
        hv[c * Np + j * BC + r] = to_half_bits(static_cast<float>(V.get(vc[j].first + r, vc[j].second + c)), dt);
    }
  void* dq = g_stage.device(0, static_cast<size_t>(Mp * Kp) * 2);
  void* dk = g_stage.device(1, static_cast<size_t>(Np * Kp) * 2);
  void* dv = g_stage.device(2, static_cast<size_t>(DVp * Np) * 2);
  auto* ds = static_cast<float*>(g_stage.device(3, static_cast<size_t>(Mp * Np) * 4));
  auto* dp = static_cast<uint16_t*>(g_stage.device(4, static_cast<size_t>(Mp * Np) * 2));
  auto* dacc = static_cast<float*>(g_stage.device(5, static_cast<size_t>(Mp * DVp) * 4));
  cuda_check(cudaMemcpyAsync(dq, hq, static_cast<size_t>(Mp * Kp) * 2, cudaMemcpyHostToDevice, st), "H2D");
  cuda_check(cudaMemcpyAsync(dk, hk, static_cast<size_t>(Np * Kp) * 2, cudaMemcpyHostToDevice, st), "H2D");
  cuda_check(cudaMemcpyAsync(dv, hv, static_cast<size_t>(DVp * Np) * 2, cudaMemcpyHostToDevice, st), "H2D");
  ws_gemm_desc d1{};
  d1.in_dtype = dt, d1.out_dtype = WS_F32;
  d1.M = Mp, d1.N = Np, d1.K = Kp;
  d1.A = dq, d1.lda = Kp, d1.B = dk, d1.ldb = Kp, d1.C = ds, d1.ldc = Np;
  d1.scale_a = d1.scale_b = 1.f;
  gemm_launch_knobs(d1, pl, Kp);
  ws_check(ws_gemm_tn(&d1, st));
  const int nblk_pad = static_cast<int>(Np / BC) + (Np % BC ? 1 : 0);
  if (Np % BC) kfail(WS_UNSUPPORTED_KERNEL, "max-shift attention: the key block must divide 256");
  const int64_t threads = Mp * nblk_pad;
  ws_rowblock_shift_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, st>>>(
      ds, Np, dp, Np, static_cast<int>(Mp), static_cast<int>(N1), static_cast<int>(BC), nblk_pad, dt == WS_F16);
  cuda_check(cudaGetLastError(), "row-block shift launch");
  ws_detail::count_launch();
  ws_gemm_desc d2{};
  d2.in_dtype = dt, d2.out_dtype = WS_F32;
  d2.M = Mp, d2.N = DVp, d2.K = Np;
  d2.A = dp, d2.lda = Np, d2.B = dv, d2.ldb = Np, d2.C = dacc, d2.ldc = DVp;
  d2.scale_a = d2.scale_b = 1.f;
  gemm_launch_knobs(d2, pl, Np);
  ws_check(ws_gemm_tn(&d2, st));
  auto* hacc = static_cast<float*>(g_stage.pinned(3, static_cast<size_t>(Mp * DVp) * 4));
  cuda_check(cudaMemcpyAsync(hacc, dacc, static_cast<size_t>(Mp * DVp) * 4, cudaMemcpyDeviceToHost, st), "D2H");
  cuda_check(cudaStreamSynchronize(st), "sync");
  for (int64_t i = 0; i < npid; ++i)
    for (int64_t r = 0; r < BR; ++r)
      for (int64_t c = 0; c < DV; ++c) O.set(pr[i].orow + r, pr[i].ocol + c, hacc[(i * BR + r) * DVp + c]);
  return true;
}

}  // namespace

extern "C" ws_status ws_run_kernel_spec(const char* ktext, ws_kbuffer* buffers, int32_t nbuffers, int64_t pid_lo,
                                        int64_t pid_hi, int32_t dtype, const ws_runspec* spec, void* cuda_stream) {
  try {
    if (!ktext) kfail(WS_TYPE, "null kernel text");
    if (dtype != WS_BF16 && dtype != WS_F16) kfail(WS_TYPE, "device dtype must be BF16 or F16");
    if (pid_hi < pid_lo) kfail(WS_TYPE, "pid_hi < pid_lo");
    Kernel g = parse(ktext);
    const Plan pl = resolve_spec(g, spec);
    std::map<std::string, HostBuf> bufs;
    for (const Param& p : g.params) {
      HostBuf b;
      b.name = p.name;
      b.shape = p.shape;
      for (int32_t i = 0; i < nbuffers; ++i)
        if (buffers[i].name && p.name == buffers[i].name) {
          if (buffers[i].rows != p.shape.r || buffers[i].cols != p.shape.c || (buffers[i].is_real != 0) != p.shape.real)
            kfail(WS_EVAL, "buffer '" + p.name + "' does not match the parameter's shape/element kind");
          b.data = buffers[i].data;
        }
      bufs.emplace(p.name, std::move(b));
    }
    for (auto& [n, b] : bufs)
      if (!b.data) {  // parameters without a caller buffer start zeroed (ref interp.hpp:140-154)
        b.own.assign(static_cast<size_t>(b.shape.r * b.shape.c), 0.0);
        b.shape.real = true;
        b.data = b.own.data();
      }
    if (pid_hi == pid_lo) return WS_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
    if (try_gemm(g, bufs, pid_lo, pid_hi, dtype, pl, st)) return WS_OK;
    if (try_flash(g, bufs, pid_lo, pid_hi, dtype, pl, st)) return WS_OK;
    if (try_maxshift(g, bufs, pid_lo, pid_hi, dtype, pl, st)) return WS_OK;
    kfail(WS_UNSUPPORTED_KERNEL,
          "kernel '" + g.name + "' is none of the gemm.k family, the flash kernel or the max-shift attention kernel");
  } catch (const KError& e) {
    return ws_detail::set_error(e.code, e.what());
  } catch (const std::exception& e) {
    return ws_detail::set_error(WS_EVAL, e.what());
  }
}

extern "C" ws_status ws_run_kernel(const char* ktext, ws_kbuffer* buffers, int32_t nbuffers, int64_t pid_lo,
                                   int64_t pid_hi, int32_t dtype, void* cuda_stream) {
  return ws_run_kernel_spec(ktext, buffers, nbuffers, pid_lo, pid_hi, dtype, nullptr, cuda_stream);
}
