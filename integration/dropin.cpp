// dropin.cpp — the reference's own flow with the B200 path as the backend (the maintainer-side
// binding of INTEGRATION.md, compiled and run).
//
// For each `.k` file given: parse it with the reference's front end, generate its inputs with the
// reference's generator (warpspec::generate_inputs, ref proj/include/warpspec/driver.hpp:79-89),
// run every pid through the reference interpreter tile by tile (the reference fixture
// interpret_tiles, ref proj/tests/support/fixtures.hpp:148-157) and through ws::run (include/ws.hpp
// -> ws_run_kernel -> sm_100a kernels), and compare the two Buffers maps: exactly for the gemm.k
// family and the integer attention.k, buffer by buffer to the north star's tolerances for a flash
// kernel (each of its three stored buffers: the accumulator o within 1e-2 of its largest entry, the
// row sums lsum within 1e-3 relative, the running max mx to fp32 rounding). With --spec the
// reference's own RunSpec (d, p, mode, coop_wgs, persistent; warpspec::RunSpec) goes through
// ws::Launch::set_spec, and a rejection is reported with the reference's ErrorCode name.
// Exit status 0 iff every kernel matches. Built by integration/Makefile against the unmodified
// reference headers (build container only); the binary travels to the GPU box with the snapshot.
//
//   dropin <kernel.k>... [--pids N] [--flash] [--spec D,P,MODE,COOP,PERSISTENT]
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "warpspec/driver.hpp"
#include "warpspec/interp.hpp"
#include "warpspec/validate.hpp"
#include "ws.hpp"

namespace {

warpspec::Buffers interpret_tiles(const warpspec::KernelGraph& g, const warpspec::Buffers& inputs, int64_t tiles) {
  warpspec::Buffers bufs = warpspec::prepare_buffers(g.params, inputs);
  for (int64_t t = 0; t < tiles; ++t) {
    warpspec::ExecContext ctx;
    ctx.pid = t;
    bufs = warpspec::interpret_sequential(g, bufs, ctx);
  }
  return bufs;
}

bool exact(const warpspec::Buffers& a, const warpspec::Buffers& b, std::string& why) {
  for (const auto& [name, t] : a) {
    auto it = b.find(name);
    if (it == b.end()) { why = name + " missing"; return false; }
    if (!(t == it->second)) { why = name + " differs"; return false; }
  }
  return true;
}

}  // namespace

int main(int argc, char** argv) {
  std::vector<std::string> files;
  int64_t pids = -1;
  bool flash = false, use_spec = false;
  warpspec::RunSpec spec;
  for (int i = 1; i < argc; ++i) {
    if (!std::strcmp(argv[i], "--pids") && i + 1 < argc) pids = std::atoll(argv[++i]);
    else if (!std::strcmp(argv[i], "--flash")) flash = true;
    else if (!std::strcmp(argv[i], "--spec") && i + 1 < argc) {
      char mode[32] = {0};
      int pers = 0;
      if (std::sscanf(argv[++i], "%d,%d,%31[a-z],%d,%d", &spec.d, &spec.p, mode, &spec.coop_wgs, &pers) != 5) {
        std::printf("bad --spec\n");
        return 2;
      }
      spec.mode = warpspec::parse_pipeline_mode(mode);
      spec.persistent = pers != 0;
      use_spec = true;
    } else files.push_back(argv[i]);
  }
  int failures = 0;
  for (const auto& f : files) {
    std::ifstream in(f);
    std::stringstream ss;
    ss << in.rdbuf();
    const std::string text = ss.str();
    try {
      const warpspec::KernelGraph g = warpspec::parse_kernel(text);
      warpspec::Buffers inputs = warpspec::generate_inputs(g.params, 2026);
      if (flash) {
        // outputs start zeroed; the causal mask bank [0 | lower-tri 0 / upper -1e7 | -1e7] is set
        // by the harness, not the generator
        for (auto& [name, t] : inputs) {
          if (name == "o" || name == "lsum" || name == "mx") t = warpspec::Tile(t.type);
          if (name == "mb") {
            t = warpspec::Tile(t.type);
            const int64_t br = t.type.rows, bc = t.type.cols / 3;
            for (int64_t r = 0; r < br; ++r)
              for (int64_t c = 0; c < bc; ++c) {
                if (c > r) t.at_r(r, bc + c) = -1e7;
                t.at_r(r, 2 * bc + c) = -1e7;
              }
          }
        }
      }
      const int64_t n = pids > 0 ? pids : 1;
      const warpspec::Buffers want = interpret_tiles(g, inputs, n);
      ws::Launch l;
      l.pid_lo = 0;
      l.pid_hi = n;
      if (use_spec) l.set_spec(spec);
      const warpspec::Buffers got = ws::run(text, inputs, l);
      // the KernelGraph overload (printed back to text by the reference's printer) must give the
      // same buffers bit for bit
      const warpspec::Buffers got_g = ws::run(g, inputs, l);
      std::string why;
      bool ok;
      if (!exact(got, got_g, why)) {
        std::printf("FAIL %s: ws::run(KernelGraph) differs from ws::run(text): %s\n", f.c_str(), why.c_str());
        ++failures;
        continue;
      }
      if (!flash) {
        ok = exact(want, got, why);
      } else {
        // the .k's three stored buffers, each within its tolerance: acc (un-normalised), l, m
        const auto& wo = want.at("o").rv; const auto& wl = want.at("lsum").rv; const auto& wm = want.at("mx").rv;
        const auto& go = got.at("o").rv; const auto& gl = got.at("lsum").rv; const auto& gm = got.at("mx").rv;
        const int64_t D = want.at("o").type.cols;
        double maxacc = 0, dacc = 0, dl = 0, dm = 0;
        for (size_t r = 0; r < wl.size(); ++r) {
          if (wl[r] == 0) continue;  // rows outside the pids run
          for (int64_t c = 0; c < D; ++c) {
            maxacc = std::fmax(maxacc, std::fabs(wo[r * D + c]));
            dacc = std::fmax(dacc, std::fabs(go[r * D + c] - wo[r * D + c]));
          }
          dl = std::fmax(dl, std::fabs(gl[r] - wl[r]) / wl[r]);
          dm = std::fmax(dm, std::fabs(gm[r] - wm[r]) / std::fmax(1.0, std::fabs(wm[r])));
        }
        ok = dacc <= 1e-2 * maxacc && dl <= 1e-3 && dm <= 1e-5;
        if (!ok)
          why = "o (acc) rel err " + std::to_string(dacc / maxacc) + ", lsum rel err " + std::to_string(dl) +
                ", mx err " + std::to_string(dm);
      }
      std::printf("%s %s (%lld pids)%s%s\n", ok ? "PASS" : "FAIL", f.c_str(), static_cast<long long>(n),
                  ok ? "" : ": ", ok ? "" : why.c_str());
      failures += !ok;
    } catch (const warpspec::CompileError& e) {
      std::printf("REJECTED %s: %s: %s\n", f.c_str(), warpspec::error_code_name(e.code()), e.what());
      ++failures;
    } catch (const std::exception& e) {
      std::printf("FAIL %s: %s\n", f.c_str(), e.what());
      ++failures;
    }
  }
  return failures == 0 ? 0 : 1;
}
