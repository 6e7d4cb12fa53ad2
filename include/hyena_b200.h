/*
 * hyena_b200.h — C-ABI of the B200-native StripedHyena 2 convolution hot path.
 *
 * Every entry point takes caller-owned DEVICE pointers (plain pointers and
 * sizes, no torch types), enqueues work on the caller's cudaStream_t (passed
 * as void*), never synchronises, never allocates, and returns an int status
 * (HY_OK = 0). hy_last_error() returns a thread-local message for the last
 * failure. Layout of every activation is (B, C, L) contiguous, time innermost:
 * element (b, c, t) lives at ((b * C) + c) * L + t. This is the reference's
 * (channels, length) SeqTensor layout (core.py:25-45) with a batch dimension.
 *
 * Filter taps are per GROUP: taps[g * lh + j] multiplies the input j steps in
 * the past for every channel c with c / group_size == g (core.py:161-204).
 * Taps are fp32 for HY_F32 / HY_BF16 activations and fp64 for HY_F64.
 *
 * Reference interfaces replaced (paths relative to
 * /root/reference/pkg/src/convhybrid/):
 *   hy_causal_conv_fwd      core.py:212-226      direct_causal_conv (any filter length)
 *                           hyena.py:122-126     the featurizer conv inside _featurize
 *                           blockconv.py:103-121 block_conv (same numbers, K spill factors)
 *   hy_gated_conv_fwd       blockconv.py:182-220 two_stage_forward(v, groups, lb, q, k) for
 *                                                fp32/fp64 (CUDA-core FIR, any filter length)
 *   hy_two_stage_fwd        blockconv.py:160-220 two_stage_forward / _two_stage_core on tcgen05
 *                           blockconv.py:267-293 chunk_parallel_forward (shared taps, gs = C)
 *                           core.py:144-146      RegularizedFilter decay, fused in-kernel
 *   hy_hyena_mixer_fwd      hyena.py:162-186     _featurize(q,k,v) conv + inner conv + gates,
 *                                                fused (the projections stay cuBLAS GEMMs)
 *   hy_fft_conv_fwd         fft.py:128-145       fft_conv, fused with the k*v / q gates as used
 *                           hyena.py:183-186     by the LI operator (backend="fft")
 *   hy_halo_correction_fwd  cpsim.py:498-510     p2p_conv_overlapped's correction conv
 *   hy_causal_conv_bwd      core.py:245-268      causal_conv_input_grad + causal_conv_taps_grad
 *                           blockconv.py:223-264 two_stage_backward (transposed factors, two-pass dtaps)
 *                           cpsim.py:440-446     a2a_conv_backward's slab step (_slab_backward)
 *   hy_featurize_fwd        hyena.py:122-126,184 _featurize(q, k, v) + gated = k * v (CP LI layer;
 *                           cpsim.py:498-510     the featurizer halo as an explicit history)
 *   hy_mixer_bwd_prep       hyena.py:262-270     gate products of hyena_backward (u, dc) fused with
 *                                                the recomputed featurizers
 *   hy_featurizer_bwd       hyena.py:234-247     _feat_backward for q, k, v fused with the gate
 *                           hyena.py:262-270     products of hyena_backward (one HBM pass)
 *   hy_two_stage_taps_grad  blockconv.py:246-262 two_stage_backward's two-pass filter gradient (tcgen05)
 *   hy_block_conv_fwd       blockconv.py:103-121 block_conv (K spill factors) on tcgen05, bf16, lh <= 513
 *   hy_qkv_feat_gemm        hyena.py:122-126,184 W_qkv projections with _featurize and k * v in the GEMM
 *                                                epilogue (tcgen05)
 *   hy_li_scan_fwd          fft.py:128-145       fft_conv on an ImplicitFilter bank (core.py:147-151), gated as
 *                           hyena.py:183-186     hyena_forward's LI inner conv, by exact per-mode scans
 *   hy_li_scan_mixer_fwd    hyena.py:162-186     the LI mixer (featurizers + gates + modal scan), fused
 *   hy_fft_c2c              fft.py:116-125       fft / ifft; cpsim.py:596-615 the distributed FFT's local transform
 *   hy_gate_mul             hyena.py:186         q * conv_out (the CP LI layer's gate after the return all-to-all)
 *   hy_split3_cat           hyena.py:124,188     the fp32 projections' operand split (split-bf16 GEMM)
 *   hy_li_param_grad        hyena.py:193-211     filter_param_grads(ImplicitFilter, dtaps) fused with
 *                           core.py:255-268      the tap correlation it consumes
 */
#ifndef HYENA_B200_H
#define HYENA_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define HY_API __attribute__((visibility("default")))
#else
#define HY_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum hy_status {
  HY_OK = 0,
  HY_ERR_INVALID = 1,     /* bad shape / argument: the Python layer raises ValueError */
  HY_ERR_INELIGIBLE = 2,  /* filter needs > 1 spill factor: TwoStageIneligibleError */
  HY_ERR_UNSUPPORTED = 3, /* dtype / size not handled by this kernel */
  HY_ERR_CUDA = 4         /* launch / runtime failure */
};

enum hy_dtype { HY_F32 = 0, HY_BF16 = 1, HY_F64 = 2 };

/* ABI version (major * 100 + minor) and last-error text (thread-local). */
HY_API int hy_version(void);
HY_API const char* hy_last_error(void);

/* Causal FIR, any filter length:
 *   y[b,c,t] = sum_{j < lh, j <= t} taps[c/gs, j] * x[b,c,t-j]
 * CUDA cores, fp32 accumulation (fp64 for HY_F64). lh <= 8 on 16-byte aligned rows
 * (L % 8 == 0, fp32 / bf16): a TMA-fed chunk stream with warp-shuffle history (every byte
 * read once); otherwise tiled windows with 128-bit coalesced loads. */
HY_API int hy_causal_conv_fwd(const void* x, void* y, const void* taps,
                       int B, int C, int L, int lh, int group_size, int dtype, void* stream);

/* Gated FIR: y = q * conv(k * v); q and/or k may be NULL (gate omitted). */
HY_API int hy_gated_conv_fwd(const void* q, const void* k, const void* v, void* y, const void* taps,
                      int B, int C, int L, int lh, int group_size, int dtype, void* stream);

/* Two-stage blocked conv on tcgen05 (bf16 operands, fp32 TMEM accumulation):
 *   u = k * v;  Y_n = T0 U_n + T1 U_{n-1} (128-step chunks);  y = q * Y
 * taps_hat: fp32 (n_groups, lh); decay: fp32 (n_groups) holding rate*log2(base),
 * or NULL for explicit taps, giving h[t] = taps_hat[t] * exp2(-decay * t).
 * Requires dtype == HY_BF16, lh <= 129, L % 8 == 0, 16-byte aligned pointers. */
HY_API int hy_two_stage_fwd(const void* q, const void* k, const void* v, void* y,
                     const float* taps_hat, const float* decay,
                     int B, int C, int L, int lh, int group_size, int dtype, void* stream);

/* Featurizer taps packed once per parameter set for the tcgen05 mixer: per channel the
 * q / k / v banded matrices F[n][k] = h[8*KS + n - k] (KS = 1 for lhf <= 9, else 2) in the
 * core-matrix order the featurizer MMAs read. out: hy_feat_pack_size() bytes of device memory. */
HY_API size_t hy_feat_pack_size(int C, int lhf);
HY_API int hy_feat_pack(const float* feat_taps, int C, int lhf, void* out, void* stream);

/* Fused Hyena mixer (everything between the projections):
 *   proj: (B, 3C, L) = [W_q^T x ; W_k^T x ; W_v^T x] per batch element
 *   q,k,v = featurizer FIRs (feat_taps: (3, C, lhf) per CHANNEL, zero padded)
 *   y = q * inner(k * v)     (inner taps per group, optional decay as above)
 * MR / SE in bf16 with lh <= 129 and feat_pack given: tcgen05 kernel (featurizers and the
 * two-stage conv as MMAs). SE (lh <= 16) otherwise: CUDA-core kernel, fp32 or bf16.
 * HY_F64 and longer filters return HY_ERR_UNSUPPORTED (the host composes kernels). */
#define HY_MIXER_HISTORY 144
/* hist (nullable, tcgen05 path only): (B, 3C, HY_MIXER_HISTORY) bf16, the projections of the
 * HY_MIXER_HISTORY steps before t = 0 (context parallel: the predecessor rank's last steps);
 * NULL means zeros (sequence start), as in the reference. */
HY_API int hy_hyena_mixer_fwd(const void* proj, void* y, const void* feat_taps, const void* feat_pack,
                       const void* hist, int lhf, const void* inner_taps, const float* inner_decay,
                       int lh, int group_size, int B, int C, int L, int dtype, void* stream);

/* Hyena-LI on tcgen05 (bf16) for an implicit filter h_t = sum_n R_n lam_n^t (core.py:147-151,
 * |lam| <= 1, npoles <= 8; residues / poles: fp32 (n_groups, npoles)): the causal conv over
 * the whole sequence as intra-chunk Toeplitz MMAs (h[0..127]) plus the exact per-mode
 * recurrence carried chunk to chunk (tf32 MMA). Same numbers as fft_conv on the materialised
 * taps (fft.py:128-145); HBM-bound instead of FFT-bound.
 *   hy_li_mixer_fwd: from the (B, 3C, L) projections, featurizers and gates fused (LI operator)
 *   hy_li_conv_fwd:  y = q * (h conv (k * v)), q / k nullable */
HY_API int hy_li_mixer_fwd(const void* proj, void* y, const float* feat_taps, const void* feat_pack, int lhf,
                           const float* residues, const float* poles, int npoles, int group_size,
                           int B, int C, int L, int dtype, void* stream);
HY_API int hy_li_conv_fwd(const void* q, const void* k, const void* v, void* y, const float* residues,
                          const float* poles, int npoles, int group_size, int B, int C, int L, int dtype,
                          void* stream);
/* Ungated implicit long conv of C rows stored in time segments, element (c, t) of v and y at
 * c * seg_len + (t / seg_len) * seg_stride + t % seg_len (seg_len a multiple of 4096 dividing
 * L, seg_stride >= C * seg_len): the rank-major buffer of the context-parallel all-to-all
 * (cpsim.py:336-375), convolved in place of the reference's slab conv without a transpose. */
HY_API int hy_li_conv_segmented_fwd(const void* v, void* y, const float* residues, const float* poles,
                                    int npoles, int group_size, int C, int L, int seg_len,
                                    long long seg_stride, int dtype, void* stream);

/* SE mixer only (CUDA cores, fp32 / bf16, lh and lhf <= 16), same arguments. */
HY_API int hy_se_mixer_fwd(const void* proj, void* y, const void* feat_taps, int lhf,
                           const void* inner_taps, const float* inner_decay, int lh, int group_size,
                           int B, int C, int L, int dtype, void* stream);

/* FFT causal conv fused with gates: y = q * (h conv (k * v)) truncated to L,
 * h given as per-group taps (n_groups, lh) with lh <= L; q/k may be NULL.
 * fp32 complex FFT of size next_pow2(L + lh - 1). ws: device workspace of
 * hy_fft_conv_workspace_size() bytes. */
HY_API size_t hy_fft_conv_workspace_size(int B, int C, int L, int lh, int group_size, int dtype);
HY_API int hy_fft_conv_fwd(const void* q, const void* k, const void* v, void* y, const void* taps,
                    int B, int C, int L, int lh, int group_size, int dtype,
                    void* ws, size_t ws_bytes, void* stream);

/* Cached filter spectra for the register four-step path (2^14 <= N <= 2^18, N =
 * next_pow2(L + lh - 1)): hy_fft_spectrum() writes the spectrum of every group's zero-padded
 * taps (G, lh) fp32 into spec (hy_fft_spectrum_size() bytes; 0 = size not covered) once per
 * filter bank — the FFT(pad(h)) half of fft.py:128-145 as a parameter transform; ws:
 * hy_fft_conv_workspace_size(1, G, L, lh, 1, HY_F32) bytes. hy_fft_conv_spec_fwd() is
 * hy_fft_conv_fwd() reading those spectra instead of transforming the taps. */
HY_API size_t hy_fft_spectrum_size(int n_groups, int L, int lh);
HY_API int hy_fft_spectrum(const void* taps, int n_groups, int L, int lh, void* spec, void* ws,
                           size_t ws_bytes, void* stream);
HY_API int hy_fft_conv_spec_fwd(const void* q, const void* k, const void* v, void* y, const void* spec,
                                int B, int C, int L, int lh, int group_size, int dtype,
                                void* ws, size_t ws_bytes, void* stream);

/* Overlapped-p2p correction: y[:, t] += sum_{j > t} taps[j] * halo[:, H + t - j]
 * for t < H = lh - 1, where halo (B, C, H) holds the predecessor's last H steps. */
HY_API int hy_halo_correction_fwd(const void* halo, void* y, const void* taps,
                           int B, int C, int L, int lh, int group_size, int dtype, void* stream);

/* ---------------------------------------------------------------- backward
 * Adjoints of the causal FIR (core.py:245-268), CUDA cores, fp32 / bf16 / fp64:
 *   dx[b,c,t]    = sum_j taps[c/gs, j] * dy[b,c,t+j]                (causal_conv_input_grad)
 *   dtaps[g, j]  = sum_{c in g} sum_{b,t} dy[b,c,t] * x[b,c,t-j]    (causal_conv_taps_grad)
 * dx or dtaps may be NULL (not computed). dtaps is fp32 for HY_F32 / HY_BF16, fp64 for HY_F64,
 * summed deterministically (per-CTA partials in ws, then a fixed-order fp64 reduce: the
 * two-pass filter gradient of blockconv.py:246-262). lh <= 2048. Used for the SE / MR inner
 * conv and the featurizers in two_stage_backward (blockconv.py:223-264) / hyena_backward
 * (hyena.py:250-284), and for the slab step of a2a_conv_backward (cpsim.py:440-446). */
HY_API size_t hy_causal_conv_bwd_workspace_size(int B, int C, int L, int lh, int dtype);
HY_API int hy_causal_conv_bwd(const void* dy, const void* x, void* dx, void* dtaps, const void* taps,
                              int B, int C, int L, int lh, int group_size, int dtype,
                              void* ws, size_t ws_bytes, void* stream);
/* Featurizers + k * v gate in one stream (forward; the context-parallel LI layer):
 *   u = (Fk conv pk) * (Fv conv pv),  fq = Fq conv pq               (B, C, L) each
 * rhist (nullable): (B, 3C, 8) raw projections of the 8 steps before t = 0 ([q; k; v] rows, the
 * predecessor rank's), the featurizers' history instead of zeros. lhf <= 8, fp32 / bf16. */
HY_API int hy_featurize_fwd(const void* proj, const void* rhist, const float* feat_taps, int lhf, int B, int C,
                            int L, int dtype, void* u, void* fq, void* stream);
/* Backward prologue of the mixer (hyena.py:262-270), one stream over the projections:
 *   u = (Fk conv pk) * (Fv conv pv),   dc = dmixed * (Fq conv pq)      (B, C, L) each
 * (the featurizers recomputed with the TMA-fed stream of hy_se_mixer_fwd). lhf <= 8, fp32 / bf16,
 * L % 8 == 0, 16-byte aligned. dc_rev (nullable) also receives dc time-reversed per row, so the
 * anti-causal inner conv runs as the causal tcgen05 kernel without a flip pass. */
HY_API int hy_mixer_bwd_prep(const void* proj, const void* dmixed, const float* feat_taps, int lhf, int B, int C,
                             int L, int dtype, void* u, void* dc, void* dc_rev, void* stream);
/* Fused featurizer backward of the mixer (hyena.py:234-247 for q, k, v with the gate products
 * of hyena.py:262-270), one pass: from the projections proj (B, 3C, L) = [q; k; v] rows, the
 * gradient at the mixer output dmixed (B, C, L), the inner conv output conv_out (B, C, L) and
 * du (B, C, L) (gradient at u = k * v):
 *   dfq = dmixed * conv_out, dfk = du * (Fv conv pv), dfv = du * (Fk conv pk)
 *   dproj[x][t] = sum_j Fx[j] dfx[t + j],   dfeat[x][c][j] = sum_{b,t} dfx[t] px[t - j]
 * feat_taps / dfeat: fp32 (3, C, lhf), lhf <= 8; fp32 / bf16 activations, L % 8 == 0,
 * 16-byte aligned; ws: hy_featurizer_bwd_workspace_size bytes (fp64 accumulators).
 * du_reversed != 0: du rows are stored time-reversed (the output of the causal conv run on the
 * reversed dc), read back mirrored in shared memory. */
HY_API size_t hy_featurizer_bwd_workspace_size(int C, int lhf);
HY_API int hy_featurizer_bwd(const void* proj, const void* dmixed, const void* conv_out, const void* du,
                             const float* feat_taps, int lhf, int B, int C, int L, int dtype, void* dproj,
                             float* dfeat, void* ws, size_t ws_bytes, int du_reversed, void* stream);
/* Two-stage filter gradient on tcgen05 (bf16, lh <= 129): both passes of blockconv.py:246-262
 * in one kernel — per channel the chunk outer products P0 = sum_n dC_n U_n^T and
 * P1 = sum_n dC_n U_{n-1}^T accumulate in TMEM (M = N = 128, K = chunks, summed over the
 * batch), then their block diagonals are scattered onto the taps in the epilogue:
 *   dtaps[g, j] = sum_{c in g} sum_{b,t} dc[b,c,t] * u[b,c,t-j]   (fp32 (G, lh))
 * dc, u: (B, C, L) bf16, L % 8 == 0. ws: hy_two_stage_taps_grad_workspace_size bytes. */
HY_API size_t hy_two_stage_taps_grad_workspace_size(int C, int lh);
HY_API int hy_two_stage_taps_grad(const void* dc, const void* u, float* dtaps, int B, int C, int L, int lh,
                                  int group_size, int dtype, void* ws, size_t ws_bytes, void* stream);
/* Two-stage filter gradient, pass 2 (blockconv.py:253-262): from the chunk-summed outer
 * products P0 = sum_n dC_n U_n^T, P1 = sum_n dC_n U_{n-1}^T (fp32, (C, lb, lb) each; pass 1 is
 * a tensor-core batched GEMM over the chunked rows) scatter the block diagonals onto the taps:
 * dtaps[g, j] = sum_{c in g} (sum_{i-i'=j} P0[c,i,i'] + sum_{lb+i-i'=j} P1[c,i,i']), j < lh <= 2 lb.
 * ws: C * lh fp32. */
HY_API int hy_toeplitz_taps_reduce(const float* P0, const float* P1, float* dtaps, float* ws, size_t ws_bytes,
                                   int C, int lb, int lh, int group_size, void* stream);
/* Hyena-LI filter-parameter gradients for h_t = sum_n R_n lam_n^t (npoles <= 8) straight from
 * dc (gradient at the conv output) and u (conv input), without the length-L tap gradient:
 *   d_res[g,n]  = sum_{b, c in g} sum_s dc[s] S_n[s],     S_n[s] = lam_n S_n[s-1] + u[s]
 *   d_pole[g,n] = R_n sum_{b, c in g} sum_s dc[s] P_n[s], P_n[s] = lam_n P_n[s-1] + S_n[s-1]
 * = filter_param_grads(ImplicitFilter, causal_conv_taps_grad(dc, u)) (hyena.py:193-211).
 * fp32 / bf16 activations; d_res, d_pole fp32 (n_groups, npoles). */
HY_API size_t hy_li_param_grad_workspace_size(int B, int C);
HY_API int hy_li_param_grad(const void* dc, const void* u, const float* residues, const float* poles, int npoles,
                            int group_size, int B, int C, int L, int dtype, float* d_res, float* d_pole,
                            void* ws, size_t ws_bytes, void* stream);

/* The q/k/v projection GEMM with the featurizers in its epilogue (hyena.py:122-126, the gate
 * product of hyena.py:184): out (B, 2D, L) = [fq; u],
 * fq = h_q * (W_q^T x), u = (h_k * (W_k^T x)) (h_v * (W_v^T x)), causal FIRs of lhf <= 8 taps on
 * the fp32 accumulators. tcgen05 / TMA, bf16 x (B, D, L) and w_perm (3D, D) — [W_q; W_k; W_v]^T
 * with rows regrouped as D/128 tiles of q rows then D/64 tiles of [64 k rows; the same channels'
 * 64 v rows] (ops.qkv_weight_permute); feat_taps fp32 (3, D, lhf). D % 128 == 0, L % 256 == 0.
 * segments: time segments per 128-row tile (0 = chosen for the grid). */
HY_API int hy_qkv_feat_gemm(const void* w_perm, const void* x, const float* feat_taps, int lhf, void* fq, void* u,
                            int B, int D, int L, int segments, int dtype, void* stream);

/* K-block causal conv on tcgen05 (blockconv.py:103-121 block_conv; the K + 1 spill factors
 * T_k[m][j] = h[128 k + m - j] as accumulating MMAs over row-shifted views of one U buffer),
 * optionally gated y = q * conv(k * v) and with the MR decay (taps_hat * 2^(-decay * t)):
 * bf16, 1 <= lh <= 513, L % 8 == 0. q / k / decay nullable. */
HY_API int hy_block_conv_fwd(const void* q, const void* k, const void* v, void* y, const float* taps_hat,
                             const float* decay, int B, int C, int L, int lh, int group_size, int dtype,
                             void* stream);
/* Hyena-LI long conv as an exact modal state scan on CUDA cores (the reference-precision path):
 *   y = q * (h conv (k * v)),  h_t = sum_n R_n lam_n^t  (core.py:147-151, fft.py:128-145)
 * computed as y[t] = q[t] sum_n R_n s_n[t], s_n[t] = lam_n s_n[t-1] + k[t] v[t]. Any dtype
 * (fp32 / bf16 with fp32 states, fp64 with fp64 states; fp64 tile carries), 1..64 poles per
 * group, any L; q / k nullable. residues, poles: fp64 (n_groups, npoles). */
HY_API int hy_li_scan_fwd(const void* q, const void* k, const void* v, void* y, const double* residues,
                          const double* poles, int npoles, int group_size, int B, int C, int L, int dtype,
                          void* stream);
/* The same modal scan fused with the featurizers (lhf <= 8) and gates: the LI mixer from the
 * projections proj (B, 3C, L) = [q; k; v] rows, y = Fq(pq) * (h conv (Fk(pk) * Fv(pv)))
 * (hyena.py:162-186), one pass. feat_taps (3, C, lhf): fp32 for fp32 / bf16 rows, fp64 for fp64;
 * residues, poles fp64. */
HY_API int hy_li_scan_mixer_fwd(const void* proj, void* y, const void* feat_taps, int lhf, const double* residues,
                                const double* poles, int npoles, int group_size, int B, int C, int L, int dtype,
                                void* stream);
/* Batched complex FFT of rows of power-of-two length n, natural order in and out (radix-2 Stockham;
 * one CTA per row in shared memory up to 8192 (complex128) / 16384 (complex64) points, one stage
 * per launch through the workspace above): x, y (batch, n) complex64 (dtype HY_F32) or complex128
 * (HY_F64), out of place; inverse != 0 flips the twiddle sign and does NOT scale (fft.py:116-125's
 * ifft carries the 1/n). ws: hy_fft_c2c_workspace_size bytes (0 for short rows). */
HY_API size_t hy_fft_c2c_workspace_size(long long batch, long long n, int dtype);
HY_API int hy_fft_c2c(const void* x, void* y, long long batch, long long n, int inverse, int dtype, void* ws,
                      size_t ws_bytes, void* stream);
/* out = a * b elementwise over n contiguous elements (bf16 / fp32 / fp64, fp32 arithmetic for
 * bf16): the LI context-parallel layer's q gate on the returned slab (hyena.py:186). */
HY_API int hy_gate_mul(const void* a, const void* b, void* out, long long n, int dtype, void* stream);
/* fp32 activation -> the K-concatenated bf16 operand of the split-bf16 fp32 GEMM (blas.py; the
 * fp32 projections of hyena.py:124,188 on tensor cores): x (batch, K, N) fp32, out
 * (batch, 5K, N) bf16 = [X1; X2; X0; X1; X0] with X0 = bf16(x), X1 = bf16(x - X0),
 * X2 = bf16(x - X0 - X1) (x == X0 + X1 + X2 exactly). One pass, 4 bytes in / 10 out. */
HY_API int hy_split3_cat(const float* x, void* out, long long batch, long long K, long long N, void* stream);

/* Debug / tuning: CTA-0 per-tile timeline (clock64) of the last two-stage launch made
 * with HY_TS_TRACE=1 in the environment; n <= 4096 values, 8 events per tile. */
HY_API int hy_debug_two_stage_trace(unsigned long long* host_out, int n);

#ifdef __cplusplus
}
#endif

#endif /* HYENA_B200_H */
