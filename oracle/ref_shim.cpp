// ref_shim.cpp — a C entry layer over the UNMODIFIED reference headers, compiled from
// /root/reference/proj/include by oracle/Makefile into oracle/_ref/libwsref.so.
//
// TEST INFRASTRUCTURE ONLY (the checker, and the `--impl reference` CPU arm of bench.py). It
// contains no arithmetic of its own: every value it returns is produced by
//   warpspec::parse_kernel          ref proj/include/warpspec/validate.hpp:349
//   warpspec::generate_inputs       ref proj/include/warpspec/driver.hpp:79-89
//   warpspec::interpret_sequential  ref proj/include/warpspec/interp.hpp:157-185
// run tile by tile exactly like the reference's own fixture interpret_tiles
// (ref proj/tests/support/fixtures.hpp:148-157).
#include <cstdint>
#include <cstring>
#include <string>

#include "warpspec/driver.hpp"
#include "warpspec/interp.hpp"
#include "warpspec/validate.hpp"

namespace {
thread_local std::string g_err;

int set_err(const std::exception& e, char* err, int errlen) {
  g_err = e.what();
  if (err && errlen > 0) {
    std::strncpy(err, g_err.c_str(), errlen - 1);
    err[errlen - 1] = 0;
  }
  if (auto* ce = dynamic_cast<const warpspec::CompileError*>(&e)) return 1 + static_cast<int>(ce->code());
  return 100;
}
}  // namespace

extern "C" {

// Number of params of a kernel; -1 on parse error.
int wsref_num_params(const char* ktext) {
  try {
    return static_cast<int>(warpspec::parse_kernel(ktext).params.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Param i: name (copied into name_out), rows, cols, is_real.
int wsref_param(const char* ktext, int i, char* name_out, int name_len, int64_t* rows, int64_t* cols, int* is_real) {
  try {
    auto g = warpspec::parse_kernel(ktext);
    const auto& p = g.params.at(static_cast<size_t>(i));
    std::strncpy(name_out, p.name.c_str(), name_len - 1);
    name_out[name_len - 1] = 0;
    *rows = p.type.rows;
    *cols = p.type.cols;
    *is_real = p.type.elem == warpspec::Elem::Real;
    return 0;
  } catch (const std::exception& e) {
    return set_err(e, nullptr, 0);
  }
}

// The reference's deterministic inputs for param `name` of the kernel (double or int64 array).
int wsref_generate(const char* ktext, uint64_t seed, const char* name, void* out) {
  try {
    auto g = warpspec::parse_kernel(ktext);
    auto bufs = warpspec::generate_inputs(g.params, seed);
    const auto& t = bufs.at(name);
    if (t.type.elem == warpspec::Elem::Real)
      std::memcpy(out, t.rv.data(), t.rv.size() * sizeof(double));
    else
      std::memcpy(out, t.iv.data(), t.iv.size() * sizeof(int64_t));
    return 0;
  } catch (const std::exception& e) {
    return set_err(e, nullptr, 0);
  }
}

// Run pids [pid_lo, pid_hi) of the kernel over the given buffers (in/out, every param in
// declaration order; double for real params, int64 for int params), like interpret_tiles.
int wsref_run(const char* ktext, void** data, int64_t pid_lo, int64_t pid_hi, char* err, int errlen) {
  try {
    auto g = warpspec::parse_kernel(ktext);
    warpspec::Buffers in;
    for (size_t i = 0; i < g.params.size(); ++i) {
      const auto& p = g.params[i];
      warpspec::Tile t(p.type);
      if (p.type.elem == warpspec::Elem::Real)
        std::memcpy(t.rv.data(), data[i], t.rv.size() * sizeof(double));
      else
        std::memcpy(t.iv.data(), data[i], t.iv.size() * sizeof(int64_t));
      in.emplace(p.name, std::move(t));
    }
    warpspec::Buffers bufs = warpspec::prepare_buffers(g.params, in);
    for (int64_t pid = pid_lo; pid < pid_hi; ++pid) {
      warpspec::ExecContext ctx;
      ctx.pid = pid;
      bufs = warpspec::interpret_sequential(g, bufs, ctx);
    }
    for (size_t i = 0; i < g.params.size(); ++i) {
      const auto& t = bufs.at(g.params[i].name);
      if (t.type.elem == warpspec::Elem::Real)
        std::memcpy(data[i], t.rv.data(), t.rv.size() * sizeof(double));
      else
        std::memcpy(data[i], t.iv.data(), t.iv.size() * sizeof(int64_t));
    }
    return 0;
  } catch (const std::exception& e) {
    return set_err(e, err, errlen);
  }
}

const char* wsref_last_error(void) { return g_err.c_str(); }

}  // extern "C"
