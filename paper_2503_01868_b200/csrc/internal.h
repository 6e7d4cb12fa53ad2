// Internal (C++-linkage) entry points shared between translation units.
#pragma once

namespace hy {
int mr_mixer_fwd(const void* proj, void* y, const float* feat_taps, const void* feat_pack, const void* hist,
                 int lhf, const float* taps_hat, const float* decay, int lh, int gs, int B, int C, int L,
                 void* stream);
}  // namespace hy
