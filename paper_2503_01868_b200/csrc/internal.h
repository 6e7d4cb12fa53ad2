// Internal (C++-linkage) entry points shared between translation units.
#pragma once

namespace hy {
int mr_mixer_fwd(const void* proj, void* y, const float* feat_taps, const void* feat_pack, const void* hist,
                 int lhf, const float* taps_hat, const float* decay, int lh, int gs, int B, int C, int L,
                 void* stream);
// register-blocked four-step FFT conv (fft_fast.cu) for 2^14 <= N <= 2^18
bool fft_fast_supported(int N);
int fft_fast_run(const void* q, const void* k, const void* v, void* y, const float* taps, int B, int C, int L,
                 int lh, int gs, int dtype, int N, int row_block, void* tw, void* hf, void* x, void* stream);
int fft_fast_spectrum(const float* taps, int G, int lh, int N, void* spec, void* tw, void* stream);
int fft_fast_conv_spec(const void* q, const void* k, const void* v, void* y, const void* spec, int B, int C, int L,
                       int gs, int dtype, int N, int row_block, void* tw, void* x, void* stream);
// kernel F as a TMA-fed chunk stream (mixer.cu) for lh <= 8 on 16-byte aligned rows
bool fir_stream_eligible(const void* q, const void* k, const void* v, const void* y, int lh, int L, int dtype);
int fir_stream_fwd(const void* q, const void* k, const void* v, void* y, const float* taps, int B, int C, int L,
                   int lh, int gs, int dtype, void* stream);
// implicit-filter long conv on the staged-row tcgen05 kernel (block_conv_sm100.cu): 64-chunk
// tiles; seg_len = 0 (plain rows) or a multiple of 8192
int li_conv_tc_fwd(const void* q, const void* k, const void* v, void* y, const float* residues, const float* poles,
                   int npoles, int gs, int B, int C, int L, int seg_len, long long seg_stride, void* stream);
// fused mixers (featurizers + gates + implicit / K-block conv) on the staged-row tcgen05 kernel
int mixer_tc_fwd(const void* proj, void* y, const float* feat_taps, int lhf, const float* taps_hat,
                 const float* decay, int lh, const float* residues, const float* poles, int npoles, int gs, int B,
                 int C, int L, void* stream);
}  // namespace hy
