// des_host.cpp — TEST HARNESS ONLY: the run engine's source (csrc/sp_des.cuh, sp_des_host.h)
// compiled for the host, so the CPU test suite can check the engine's logic against
// oracle/engine.py and the reference engine in a container without a GPU.  Same entry semantics
// as sp_des_run(SP_MEM_HOST); replicas run one after another.  The product path is the device
// kernel k_des_run; nothing under paper_2102_01887_b200/ loads this library.
#include <cstdlib>
#include <string>
#include <vector>

#include "sp_des_host.h"

using namespace spdes;

static std::string g_err;

extern "C" const char* des_host_error() { return g_err.c_str(); }

extern "C" int des_host_run(const sp_des_spec* spec, double cap_scale, int32_t R, int32_t T,
                            const int32_t* frame_off, const int32_t* attrs, const int32_t* trace_of,
                            const double* target_s,
                            int32_t draw_cap, const double* draw_factor, const uint8_t* draw_bits,
                            int32_t log_cap, sp_des_log* log, double* lat_out, sp_des_out* out,
                            int32_t ev_cap, sp_des_event* events) {
  HostImage h;
  h.cap_scale = cap_scale;
  if (!build_image(*spec, h, g_err)) return -1;
  if (!plan_run(h, T, frame_off, attrs, draw_cap, log_cap, g_err, ev_cap)) return -1;
  const Image& im = h.im;
  std::vector<char> arena((size_t)im.arena_bytes + 16);
  char* base = (char*)(((uintptr_t)arena.data() + 15) & ~(uintptr_t)15);
  const Entries E = entries_view(h.dcols.data(), h.icols.data(), im.n_entries);
  for (int r = 0; r < R; ++r) {
    const int tr = trace_of ? trace_of[r] : r;
    const int f0 = frame_off[tr];
    Run run(im, E, base, (double*)(base + im.o_lat), 1, attrs + (int64_t)f0 * im.n_attrs, frame_off[tr + 1] - f0, target_s[r],
            draw_factor ? draw_factor + (size_t)r * draw_cap : nullptr,
            draw_bits ? draw_bits + (size_t)r * draw_cap : nullptr,
            log ? reinterpret_cast<LogRec*>(log) + (size_t)r * log_cap : nullptr);
    if (events) run.evlog = reinterpret_cast<EvRec*>(events) + (size_t)r * ev_cap;
    run.run();
    run.write_out(*reinterpret_cast<Out*>(out + r));
    if (lat_out)
      for (int i = 0; i < im.n_entries; ++i) lat_out[(size_t)r * im.n_entries + i] = run.lat(i);
  }
  return 0;
}
