/*
 * ws.hpp — reference-side C++ binding of the B200 path: the reference's own types in and out.
 *
 * Header-only; include it next to the reference's headers (it uses warpspec::Buffers / Tile /
 * KernelGraph / CompileError from proj/include/warpspec). It is the `ws::run` shim of SURVEY.md §7
 * step 2: a `.k` kernel text plus the reference's by-value Buffers (ref
 * proj/include/warpspec/interp.hpp:31) go to the GPU through the C-ABI in ws.h and come back as
 * Buffers, so the reference's check pattern applies unchanged — run_compiled compares the
 * simulator's buffers with interpret_sequential's (ref proj/include/warpspec/driver.hpp:242-266);
 * here `ws::run(text, inputs, launch) == interpret_tiles(...)`, or `ws::run(graph, inputs, launch)`.
 *
 * Errors: a non-OK ws_status is rethrown as warpspec::CompileError with the mirrored ErrorCode
 * (ws_status 1..12 = ErrorCode order + 1, ref proj/include/warpspec/errors.hpp:10-23); CUDA
 * failures as std::runtime_error — the reference CLI's exit-code split (tools/warpspec.cpp:95-101).
 */
#ifndef WS_HPP_
#define WS_HPP_

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "warpspec/errors.hpp"
#include "warpspec/interp.hpp"
#include "warpspec/print.hpp"
#include "warpspec/validate.hpp"
#include "ws.h"

namespace ws {

struct Launch {
  int64_t pid_lo = 0;      // the .k pid range to run, like interpret_tiles' tile loop
  int64_t pid_hi = 1;
  int32_t dtype = WS_BF16; // device storage type of the real payloads (exact for the reference's)
  void* stream = nullptr;  // cudaStream_t; the call is synchronous w.r.t. the host buffers
  // the reference's RunSpec knobs (ref proj/include/warpspec/driver.hpp:42-57), validated with
  // compile_kernel's rejections; unset = the library's measured defaults
  bool use_spec = false;
  ws_runspec spec{0, 0, WS_MODE_AUTO, 0, 1};
  // from a reference RunSpec: d, p, mode, coop_wgs, persistent (tiles / paths stay the caller's)
  template <class RunSpecT>
  void set_spec(const RunSpecT& rs) {
    use_spec = true;
    spec.d = rs.d;
    spec.p = rs.p;
    spec.mode = static_cast<int32_t>(rs.mode);  // PipelineMode order: Auto, Fine, Coarse, None
    spec.coop_wgs = rs.coop_wgs;
    spec.persistent = rs.persistent ? 1 : 0;
  }
};

inline void check(ws_status s) {
  if (s == WS_OK) return;
  const std::string msg = ws_last_error();
  if (s >= WS_PARSE && s <= WS_EVAL)
    throw warpspec::CompileError(static_cast<warpspec::ErrorCode>(static_cast<int>(s) - 1), msg);
  throw std::runtime_error("ws: " + msg);
}

namespace detail {
// Marshal `inputs` against the graph's declared parameters and run `ktext` (the graph's text).
inline warpspec::Buffers run_graph(const warpspec::KernelGraph& g, const std::string& ktext,
                                   const warpspec::Buffers& inputs, const Launch& launch) {
  warpspec::Buffers out;
  std::vector<ws_kbuffer> bufs;
  bufs.reserve(g.params.size());
  for (const auto& p : g.params) {
    auto it = inputs.find(p.name);
    warpspec::Tile t = it != inputs.end() ? it->second : warpspec::Tile(p.type);
    if (t.type != p.type)
      throw warpspec::CompileError(warpspec::ErrorCode::Type, "buffer " + p.name + " is " + t.type.str() +
                                                                  ", the kernel declares " + p.type.str());
    out[p.name] = std::move(t);
  }
  for (const auto& p : g.params) {
    warpspec::Tile& t = out[p.name];
    ws_kbuffer b{};
    b.name = p.name.c_str();
    b.rows = t.type.rows;
    b.cols = t.type.cols;
    b.is_real = t.type.elem == warpspec::Elem::Real;
    b.data = b.is_real ? static_cast<void*>(t.rv.data()) : static_cast<void*>(t.iv.data());
    bufs.push_back(b);
  }
  check(ws_run_kernel_spec(ktext.c_str(), bufs.data(), static_cast<int32_t>(bufs.size()), launch.pid_lo,
                           launch.pid_hi, launch.dtype, launch.use_spec ? &launch.spec : nullptr, launch.stream));
  return out;
}
}  // namespace detail

// Run pids [launch.pid_lo, launch.pid_hi) of `ktext` on the GPU. Parameters missing from `inputs`
// start zeroed (ref interp.hpp:140-154 prepare_buffers); every parameter is returned.
inline warpspec::Buffers run(const std::string& ktext, const warpspec::Buffers& inputs, const Launch& launch = {}) {
  return detail::run_graph(warpspec::parse_kernel(ktext), ktext, inputs, launch);  // the reference's front end
}

// SURVEY.md §8b's shim signature: a parsed KernelGraph in, Buffers out. The graph is printed back
// to `.k` text by the reference's own printer (ref proj/include/warpspec/print.hpp:160), the form
// the C-ABI takes. Not re-parsed by parse_kernel: the reference's parser rejects its printer's
// exponent form for constants such as -1e6 ("[[-1e+06]]"); the C-ABI's front end accepts it.
inline warpspec::Buffers run(const warpspec::KernelGraph& g, const warpspec::Buffers& inputs,
                             const Launch& launch = {}) {
  return detail::run_graph(g, warpspec::print_kernel(g), inputs, launch);
}

}  // namespace ws

#endif  // WS_HPP_
