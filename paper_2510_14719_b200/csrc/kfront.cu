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
//      flash .k of SURVEY.md Appendix A -> ws_attn_fwd.
// Unsupported shapes fail with WS_UNSUPPORTED_KERNEL, never with a CPU fallback.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ws.h"

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
// host buffers
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

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};
void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) kfail(WS_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}
void ws_check(ws_status s) {
  if (s != WS_OK) kfail(s, ws_last_error());
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

// ------------------------------------------------------------------------------------------------
// gemm.k family
// ------------------------------------------------------------------------------------------------
struct PidTile {
  int64_t pid, r0, c0, ra, rb, ka0, kb0;
};

bool try_gemm(const Kernel& g, std::map<std::string, HostBuf>& bufs, int64_t lo, int64_t hi, int dt, cudaStream_t st) {
  // body: exactly two loads and one dot(a, b.T, acc=<iter arg>), optional relu of the new acc,
  // yield; prologue acc init = zeros; epilogue: store of the acc (or of the relu'd iter arg), or
  // of `ew mul acc, <1x1 const>`
  const Op* dot = nullptr;
  std::vector<const Op*> loads;
  const Op* relu = nullptr;
  for (const Op* o : tile_ops(g.body)) {
    if (o->k == K::Load) loads.push_back(o);
    else if (o->k == K::Dot) {
      if (dot) return false;
      dot = o;
    } else if (o->k == K::Ew && o->fn == "relu" && !relu) relu = o;
    else return false;
  }
  if (!dot || loads.size() != 2 || !dot->trans) return false;
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
    relu_i = -1;
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
    const Op* c = def_any(g, scale_op->args[1]);
    if (!c || c->k != K::ConstTile || c->zeros || c->shape.r != 1 || c->shape.c != 1) return false;
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
    ScalarEnv env;
    env.run(g.pro, pid);
    std::map<std::string, int64_t> iter_s;
    for (auto& [a, init] : g.iter)
      if (env.v.count(init)) env.v[a] = env.v[init];
    int64_t ra = 0, rb = 0, ka = 0, kb = 0, ka1 = 0, kb1 = 0;
    for (int64_t k = g.lo; k < std::min(g.hi, g.lo + 2); ++k) {
      ScalarEnv e2 = env;
      e2.v[g.ind] = k;
      e2.run(g.body, pid);
      const int64_t r_a = e2.get(la->args[0]), c_a = e2.get(la->args[1]);
      const int64_t r_b = e2.get(lb->args[0]), c_b = e2.get(lb->args[1]);
      if (k == g.lo) {
        ra = r_a, rb = r_b, ka = c_a, kb = c_b;
      } else {
        if (r_a != ra || r_b != rb) kfail(WS_UNSUPPORTED_KERNEL, "tile rows change across iterations");
        ka1 = c_a, kb1 = c_b;
      }
      // advance scalar iter args with the yield
      for (size_t i = 0; i < g.iter.size(); ++i)
        if (e2.v.count(y->args[i])) env.v[g.iter[i].first] = e2.v[y->args[i]];
    }
    if (trip > 1 && (ka1 - ka != BKa || kb1 - kb != BKb))
      kfail(WS_UNSUPPORTED_KERNEL, "K offsets do not advance by the tile depth");
    ScalarEnv ee = env;
    ee.run(g.epi, pid);
    tiles.push_back({pid, ee.get(store->args[1]), ee.get(store->args[2]), ra, rb, ka, kb});
  }
  if (tiles.empty()) return true;
  const int64_t Kd = trip * BKa;

  // group pids that form one GEMM: same A/B row offsets relative to the C tile and same K range
  std::map<std::vector<int64_t>, std::vector<PidTile>> groups;
  for (auto& t : tiles) groups[{t.ra - t.r0, t.rb - t.c0, t.ka0, t.kb0}].push_back(t);

  // exactness of the device arithmetic for the reference's payloads
  auto amax = [](const HostBuf& b) {
    double m = 0;
    const int64_t n = b.shape.r * b.shape.c;
    for (int64_t i = 0; i < n; ++i) m = std::max(m, std::fabs(b.get(i / b.shape.c, i % b.shape.c)));
    return m;
  };
  if (!A.shape.real || !B.shape.real) {
    if (amax(A) * amax(B) * static_cast<double>(Kd) >= 16777216.0)
      kfail(WS_UNSUPPORTED_KERNEL, "int payloads could overflow fp32-exact accumulation (>= 2^24)");
  }

  for (auto& [key, ts] : groups) {
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
    std::vector<uint16_t> ha(static_cast<size_t>(Mp * Kp), 0), hb(static_cast<size_t>(Np * Kp), 0);
    for (int64_t r = 0; r < M; ++r)
      for (int64_t k = 0; k < Kd; ++k) ha[r * Kp + k] = to_half_bits(static_cast<float>(A.get(rmin + dA + r, ka0 + k)), dt);
    for (int64_t n = 0; n < N; ++n)
      for (int64_t k = 0; k < Kd; ++k) hb[n * Kp + k] = to_half_bits(static_cast<float>(B.get(cmin + dB + n, kb0 + k)), dt);
    DevBuf da, db, dc;
    cuda_check(cudaMalloc(&da.p, ha.size() * 2), "cudaMalloc");
    cuda_check(cudaMalloc(&db.p, hb.size() * 2), "cudaMalloc");
    cuda_check(cudaMalloc(&dc.p, static_cast<size_t>(Mp * Np) * 4), "cudaMalloc");
    cuda_check(cudaMemcpyAsync(da.p, ha.data(), ha.size() * 2, cudaMemcpyHostToDevice, st), "H2D");
    cuda_check(cudaMemcpyAsync(db.p, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice, st), "H2D");
    ws_gemm_desc d{};
    d.in_dtype = dt;
    d.out_dtype = WS_F32;
    d.M = Mp, d.N = Np, d.K = Kp;
    d.A = da.p, d.lda = Kp, d.B = db.p, d.ldb = Kp, d.C = dc.p, d.ldc = Np;
    d.scale_a = static_cast<float>(scale), d.scale_b = 1.f;
    d.persistent = 1;
    d.cta_pair = Kp >= 1024 ? 1 : 0;
    d.act = act_relu ? 1 : 0;
    ws_check(ws_gemm_tn(&d, st));
    std::vector<float> hc(static_cast<size_t>(Mp * Np));
    cuda_check(cudaMemcpyAsync(hc.data(), dc.p, hc.size() * 4, cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaStreamSynchronize(st), "sync");
    for (auto& t : ts)
      for (int64_t r = 0; r < BM; ++r)
        for (int64_t c = 0; c < BN; ++c) C.set(t.r0 + r, t.c0 + c, hc[(t.r0 - rmin + r) * Np + (t.c0 - cmin + c)]);
  }
  return true;
}

// ------------------------------------------------------------------------------------------------
// flash .k
// ------------------------------------------------------------------------------------------------
bool try_flash(const Kernel& g, std::map<std::string, HostBuf>& bufs, int64_t lo, int64_t hi, int dt, cudaStream_t st) {
  std::vector<const Op*> dots, loads;
  int n_exp = 0, n_rmax = 0, n_radd = 0;
  for (const Op* o : tile_ops(g.body)) {
    if (o->k == K::Dot) dots.push_back(o);
    else if (o->k == K::Load) loads.push_back(o);
    else if (o->k == K::Ew && o->fn == "exp") ++n_exp;
    else if (o->k == K::Reduce && o->fn == "max" && o->axis == 1) ++n_rmax;
    else if (o->k == K::Reduce && o->fn == "add" && o->axis == 1) ++n_radd;
  }
  if (dots.size() != 2 || n_exp < 1 || n_rmax != 1 || n_radd != 1) return false;
  const Op* qk = dots[0]->trans ? dots[0] : dots[1];
  const Op* pv = dots[0]->trans ? dots[1] : dots[0];
  if (!qk->trans || pv->trans) return false;
  const Op* lq = def_of(g.body, qk->args[0]);
  const Op* lk = def_of(g.body, qk->args[1]);
  const Op* lv = def_of(g.body, pv->args[1]);
  if (!lq || !lk || !lv || lq->k != K::Load || lk->k != K::Load || lv->k != K::Load) return false;
  const Op* s_init = def_any(g, qk->args[2]);
  const bool causal = s_init && s_init->k == K::Load;  // mask bank
  // softmax scale: the 1x1 constant multiplying the scores
  double scale = -1;
  for (const Op& o : g.body)
    if (o.k == K::Ew && o.fn == "mul" && o.args[0] == qk->res) {
      const Op* c = def_any(g, o.args[1]);
      if (c && c->k == K::ConstTile && !c->zeros && c->shape.r == 1 && c->shape.c == 1) scale = c->lit[0];
    }
  if (scale <= 0) return false;
  // outputs: stores of the three iter args acc (pv chain), l (row sums), m (running max)
  const Op* y = yield_op(g);
  if (!y) return false;
  std::string o_buf, l_buf, m_buf;
  for (const Op& s : g.epi) {
    if (s.k != K::Store) continue;
    const int i = iter_index(g, s.args[0]);
    if (i < 0) return false;
    const Op* src = def_of(g.body, y->args[i]);
    if (!src) return false;
    if (src == pv) o_buf = s.buf;
    else if (src->k == K::Ew && src->fn == "max") m_buf = s.buf;
    else if (src->k == K::Ew && src->fn == "add") l_buf = s.buf;
    else return false;
  }
  if (o_buf.empty() || l_buf.empty() || m_buf.empty()) return false;
  const HostBuf& Q = bufs.at(lq->buf);
  const HostBuf& Kb = bufs.at(lk->buf);
  const HostBuf& V = bufs.at(lv->buf);
  const int64_t BR = lq->shape.r, D = lq->shape.c, BC = lk->shape.r;
  const int64_t trip = g.hi - g.lo, S = trip * BC;
  if (S <= 0 || Q.shape.r % S != 0 || Kb.shape.r != Q.shape.r || V.shape.r != Q.shape.r || Q.shape.c != D)
    return false;
  const int64_t BH = Q.shape.r / S;
  // verify the batched pid geometry on the pids that run: q rows = pid*BR; k/v rows start at
  // (pid / (S/BR)) * S and advance by BC
  const int64_t nqb = S / BR;
  for (int64_t pid : {lo, hi - 1}) {
    ScalarEnv env;
    env.run(g.pro, pid);
    for (auto& [a, init] : g.iter)
      if (env.v.count(init)) env.v[a] = env.v[init];
    ScalarEnv e2 = env;
    e2.v[g.ind] = g.lo;
    e2.run(g.body, pid);
    if (e2.get(lq->args[0]) != pid * BR || e2.get(lk->args[0]) != (pid / nqb) * S || e2.get(lv->args[0]) != (pid / nqb) * S)
      kfail(WS_UNSUPPORTED_KERNEL, "flash kernel pid geometry differs from the batched (b,h)-major layout");
  }
  if ((D != 64 && D != 128) || S % 128 != 0)
    kfail(WS_UNSUPPORTED_KERNEL, "flash on B200 needs head dim 64/128 and S % 128 == 0 (S=" + std::to_string(S) +
                                     ", D=" + std::to_string(D) + ")");
  const int64_t bh0 = lo / nqb, bh1 = (hi - 1) / nqb + 1;
  const size_t n = static_cast<size_t>(BH * S * D);
  std::vector<uint16_t> hq(n), hk(n), hv(n);
  for (int64_t r = bh0 * S; r < bh1 * S; ++r)
    for (int64_t c = 0; c < D; ++c) {
      hq[r * D + c] = to_half_bits(static_cast<float>(Q.get(r, c)), dt);
      hk[r * D + c] = to_half_bits(static_cast<float>(Kb.get(r, c)), dt);
      hv[r * D + c] = to_half_bits(static_cast<float>(V.get(r, c)), dt);
    }
  DevBuf dq, dk, dv, dout, dlse;
  for (DevBuf* b : {&dq, &dk, &dv, &dout}) cuda_check(cudaMalloc(&b->p, n * 2), "cudaMalloc");
  cuda_check(cudaMalloc(&dlse.p, static_cast<size_t>(BH * S) * 4), "cudaMalloc");
  cuda_check(cudaMemcpyAsync(dq.p, hq.data(), n * 2, cudaMemcpyHostToDevice, st), "H2D");
  cuda_check(cudaMemcpyAsync(dk.p, hk.data(), n * 2, cudaMemcpyHostToDevice, st), "H2D");
  cuda_check(cudaMemcpyAsync(dv.p, hv.data(), n * 2, cudaMemcpyHostToDevice, st), "H2D");
  ws_attn_desc a{};
  a.dtype = dt;
  a.B = 1, a.H = static_cast<int32_t>(BH), a.S = static_cast<int32_t>(S), a.Dh = static_cast<int32_t>(D);
  a.causal = causal;
  a.softmax_scale = static_cast<float>(scale);
  a.Q = dq.p, a.K = dk.p, a.V = dv.p, a.O = dout.p, a.LSE = static_cast<float*>(dlse.p);
  a.bh_begin = static_cast<int32_t>(bh0), a.bh_end = static_cast<int32_t>(bh1);
  ws_check(ws_attn_fwd(&a, st));
  std::vector<uint16_t> ho(n);
  std::vector<float> hl(static_cast<size_t>(BH * S));
  cuda_check(cudaMemcpyAsync(ho.data(), dout.p, n * 2, cudaMemcpyDeviceToHost, st), "D2H");
  cuda_check(cudaMemcpyAsync(hl.data(), dlse.p, hl.size() * 4, cudaMemcpyDeviceToHost, st), "D2H");
  cuda_check(cudaStreamSynchronize(st), "sync");
  // Write back in the .k's (acc, l, m) form with m = lse, l = 1, acc = O: the harness step
  // o = acc / l and lse = m + log(l) is invariant to the choice of m.
  HostBuf& O = bufs.at(o_buf);
  HostBuf& L = bufs.at(l_buf);
  HostBuf& Mx = bufs.at(m_buf);
  auto half_to_float = [dt](uint16_t h) {
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
  };
  for (int64_t pid = lo; pid < hi; ++pid)
    for (int64_t r = pid * BR; r < pid * BR + BR; ++r) {
      for (int64_t c = 0; c < D; ++c) O.set(r, c, half_to_float(ho[r * D + c]));
      L.set(r, 0, 1.0);
      Mx.set(r, 0, hl[r]);
    }
  return true;
}

}  // namespace

extern "C" ws_status ws_run_kernel(const char* ktext, ws_kbuffer* buffers, int32_t nbuffers, int64_t pid_lo,
                                   int64_t pid_hi, int32_t dtype, void* cuda_stream);

namespace ws_detail {
ws_status set_error(ws_status s, const std::string& m);
}

ws_status ws_run_kernel(const char* ktext, ws_kbuffer* buffers, int32_t nbuffers, int64_t pid_lo, int64_t pid_hi,
                        int32_t dtype, void* cuda_stream) {
  try {
    if (!ktext) kfail(WS_TYPE, "null kernel text");
    if (dtype != WS_BF16 && dtype != WS_F16) kfail(WS_TYPE, "device dtype must be BF16 or F16");
    if (pid_hi < pid_lo) kfail(WS_TYPE, "pid_hi < pid_lo");
    Kernel g = parse(ktext);
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
    if (try_gemm(g, bufs, pid_lo, pid_hi, dtype, st)) return WS_OK;
    if (try_flash(g, bufs, pid_lo, pid_hi, dtype, st)) return WS_OK;
    kfail(WS_UNSUPPORTED_KERNEL, "kernel '" + g.name + "' is neither a gemm.k-family nor a flash kernel");
  } catch (const KError& e) {
    return ws_detail::set_error(e.code, e.what());
  } catch (const std::exception& e) {
    return ws_detail::set_error(WS_EVAL, e.what());
  }
}
