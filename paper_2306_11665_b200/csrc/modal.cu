// K4: curvilinear modal Euler volume term (config 5).  Placeholder until the
// fused kernel lands; reports ENOTSUP so callers fail loudly.
#include "common.cuh"

extern "C" int sfb_euler_volume_curvilinear_modal(int64_t, int64_t, const double*, const double*,
                                                  const double*, double, double, const double*,
                                                  const double*, double*, double*, sfb_stream_t) {
  return sfb::fail(SFB_ENOTSUP, "euler_volume_curvilinear_modal: not built yet");
}
