// sp_rng.cu — the reference's per-start RNG draws for the run engine, generated on the host in C.
//
// A noisy scenario draws, every time an execution starts, from the run's numpy Generator
// (backend.py:52-57, 186, in this order):
//     latency *= math.exp(rng.normal(0.0, noise_sigma))      if noise_sigma > 0
//     straggled = rng.random() < straggle_rate               if straggle_rate > 0
//     will_fail = rng.random() < failure_rate                if failure_rate > 0
// The stream is independent of the simulation (every start consumes the same pattern), so the
// k-th start's draws can be produced ahead of the run.  numpy's default_rng is PCG64
// (XSL-RR 128/64; next_uint64 steps the LCG then outputs the new state); Generator.random is
// (next_uint64 >> 11) * 2^-53; Generator.normal(0, s) is 0.0 + s * z with numpy's ziggurat
// standard normal (tables in sp_ziggurat.h, the rare paths through the C library's log1p /
// exp); CPython's math.exp is the C library's exp.  Compiled for the host with
// -ffp-contract=off, like numpy's baseline build, so every draw has numpy's bits
// (tests/test_rng.py).  Replicas are independent and are spread over host threads.
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <thread>
#include <vector>

#include "sp_internal.cuh"
#include "sp_ziggurat.h"

namespace {

struct Pcg64 {
  unsigned __int128 state, inc;
  uint64_t next64() {
    const unsigned __int128 mult =
        ((unsigned __int128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
    state = state * mult + inc;
    const uint64_t v = (uint64_t)(state >> 64) ^ (uint64_t)state;
    const unsigned rot = (unsigned)(state >> 122);
    return (v >> rot) | (v << ((64u - rot) & 63u));
  }
  double next_double() { return (double)(next64() >> 11) * (1.0 / 9007199254740992.0); }
  double standard_normal() {  // numpy random_standard_normal (distributions.c)
    using namespace sp_zig;
    for (;;) {
      uint64_t r = next64();
      const int idx = (int)(r & 0xff);
      r >>= 8;
      const int sign = (int)(r & 0x1);
      const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
      double x = (double)rabs * wi_double[idx];
      if (sign & 0x1) x = -x;
      if (rabs < ki_double[idx]) return x;
      if (idx == 0) {
        for (;;) {
          const double xx = -ziggurat_nor_inv_r * log1p(-next_double());
          const double yy = -log1p(-next_double());
          if (yy + yy > xx * xx) return ((rabs >> 8) & 0x1) ? -(ziggurat_nor_r + xx) : ziggurat_nor_r + xx;
        }
      } else {
        if (((fi_double[idx - 1] - fi_double[idx]) * next_double() + fi_double[idx]) < exp(-0.5 * x * x))
          return x;
      }
    }
  }
};

}  // namespace

extern "C" int sp_des_draws(int32_t R, const uint64_t* pcg_state, int32_t cap, double noise_sigma,
                            double straggle_rate, double failure_rate, double* factor,
                            uint8_t* bits) {
  if (R < 0 || cap < 0 || (R > 0 && !pcg_state) || (noise_sigma > 0.0 && !factor) ||
      ((straggle_rate > 0.0 || failure_rate > 0.0) && !bits))
    return sp::fail(SP_E_INVALID, "des_draws: bad argument");
  auto one = [&](int r) {
    Pcg64 g;
    const uint64_t* s = pcg_state + 4 * (size_t)r;  // state hi, lo, inc hi, lo
    g.state = ((unsigned __int128)s[0] << 64) | s[1];
    g.inc = ((unsigned __int128)s[2] << 64) | s[3];
    double* f = factor ? factor + (size_t)r * cap : nullptr;
    uint8_t* b = bits ? bits + (size_t)r * cap : nullptr;
    for (int k = 0; k < cap; ++k) {
      if (f) f[k] = noise_sigma > 0.0 ? exp(0.0 + noise_sigma * g.standard_normal()) : 1.0;
      uint8_t v = 0;
      if (straggle_rate > 0.0 && g.next_double() < straggle_rate) v |= 1;
      if (failure_rate > 0.0 && g.next_double() < failure_rate) v |= 2;
      if (b) b[k] = v;
    }
  };
  const int nt = std::max(1, std::min<int>((int)std::thread::hardware_concurrency(), R));
  if (nt <= 1 || R < 4) {
    for (int r = 0; r < R; ++r) one(r);
    return SP_OK;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&, t]() {
      for (int r = t; r < R; r += nt) one(r);
    });
  for (auto& x : th) x.join();
  return SP_OK;
}
