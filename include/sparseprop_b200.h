/*
 * sparseprop_b200.h -- C-ABI of the B200 (sm_100a) e-prop training-step kernels.
 *
 * The reference (`sparseprop` 0.1.0, arXiv 2501.11407 artifact) is pure Python and has
 * no FFI of its own; its hot path is one Python function,
 *   eprop_sparse_gradient(net, x_seq, label, smooth=False) -> GradResult
 *   (/root/reference/pkg/src/sparseprop/gradients.py:132-185),
 * whose per-step loop (gradients.py:157-176) is what these entry points replace, one
 * kernel per stage of SURVEY.md section 8(b).  The Python host package
 * `paper_2501_11407_b200` binds them with ctypes (INTEGRATION.md shows the binding).
 *
 * Conventions
 *   - every pointer is a DEVICE pointer unless stated; every call is asynchronous on
 *     `stream` (a cudaStream_t; 0 = legacy default stream) and never allocates;
 *   - return 0 on success, 2 on a bad argument (ShapeMismatch / ValueError in Python),
 *     3 on a launch failure; spb_last_error() returns the message (thread-local);
 *   - sizes: B batch, n hidden neurons, k inputs, m classes, Tc time-chunk length
 *     (multiple of 8), len <= Tc valid steps in this chunk, t0 global step of its first
 *     row, T sequence length; n_pad = round_up(n,128), k_pad = round_up(k,64).
 *   - spike inputs are uint8 event counts x[b][t][j] (binary for Poisson data,
 *     small integers after channel pooling, datasets.py:138-159).
 */
#ifndef SPARSEPROP_B200_H
#define SPARSEPROP_B200_H

#include <stdint.h>
#include <cuda_runtime.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Library identification / error text. */
const char* spb_last_error(void);
int spb_version(void);
int spb_device_sm(void); /* compute capability of the current device, e.g. 100 */

/* K2  Exact input projection on INT8 tensor cores (proj.cu).  The weights are sliced
 *     once per update into P signed digits per entry (P=6 radix-256 digits for fp32
 *     weights, P=8 radix-128 digits for fp64; csrc/digits.cuh) with a per-neuron
 *     power-of-two scale; spikes are uint8 counts; tcgen05
 *     kind::i8 accumulates exactly in int32 and the digits are recombined in int64, so
 *     I = W x_t is exact up to one final fp64 rounding.  Replaces `net.neuron.w @ x_t`
 *     (gradients.py:125).
 *   spb_slice_weights: w [n][k] fp32 (w_is_f64=0) / fp64 -> wq [P][n_pad32][Kpad] int8,
 *                      sexp [n] int32 (n_pad32 = round_up(n,32), Kpad = round_up(k,128)).
 *   spb_pack_spikes:   x row (b, s < len) at x + b*stride_b + s*kb -> xq [B*Tc][Kpad] uint8,
 *                      zero padded; bits = 0: kb = k bytes (counts), bits = 1: kb = ceil(k/8)
 *                      bytes, channel j = bit (j & 7) of byte j >> 3 (packbits, little);
 *                      output row b*Tc + s, or s*B + b with time_major != 0.
 *   spb_input_proj:    cur[row][i] = sum_j xq[row][j] W[i][j] for row < M (= B*Tc), fp64;
 *                      persistent grid of min(tiles, sm_count) CTAs.  k = the real input
 *                      count (columns k..Kpad-1 of xq/wq are zero): when the last partial
 *                      128-byte K block holds <= 64 inputs it runs as a 64-byte block.  binary != 0 promises
 *                      0/1 spikes (and k <= 16384): the 7 digit sums then recombine in one
 *                      int64 (same bits, half the fp64 work). */
int spb_slice_weights(const void* w, int w_is_f64, int n, int k, int Kpad, int n_pad32, int P,
                      int8_t* wq, int* sexp, cudaStream_t stream);
int spb_pack_spikes(const uint8_t* x, long long stride_b, int B, int k, int bits, int len, int Tc,
                    int Kpad, int time_major, uint8_t* xq, cudaStream_t stream);
/* spb_pack_spikes (sample-major) that also writes the one-chunk raw-spike GEMM operand of
 * K5: xh bf16 [B*KR][Kpad], row b*KR + s + 1 = the spikes of step s (row 0 untouched,
 * zero) -- K4 folded into the pack. */
int spb_pack_spikes_xh(const uint8_t* x, long long stride_b, int B, int k, int bits, int len,
                       int Tc, int Kpad, int KR, uint8_t* xq, void* xh, cudaStream_t stream);
int spb_input_proj(const uint8_t* xq, const int8_t* wq, const int* sexp, int M, int n, int n_pad32,
                   int k, int Kpad, int P, double* cur, int sm_count, int binary,
                   cudaStream_t stream);
/* spb_input_proj over rin live rows per sample: xq holds B*rin rows (row b*rin + s), the
 * current of row b*rin + s lands in cur row b*rout + s (rout = the current buffer's KR >=
 * rin); rin == rout is spb_input_proj with M = B*rin.  The one-chunk update packs only
 * the chunk's live steps (len of KR = Tc + 1 rows: C3 250 of 256, K2 0.217 -> 0.208 ms). */
int spb_input_proj_rows(const uint8_t* xq, const int8_t* wq, const int* sexp, int B, int rin,
                        int rout, int n, int n_pad32, int k, int Kpad, int P, double* cur,
                        int sm_count, int binary, cudaStream_t stream);
/* Profiling variant of spb_input_proj (W-resident kernel): probe bit 0 skips the epilogue,
 * bit 1 the spike-operand loads; probe = 0 is the production kernel. */
int spb_input_proj_probe(const uint8_t* xq, const int8_t* wq, const int* sexp, int M, int n,
                         int n_pad32, int k, int Kpad, int P, double* cur, int sm_count,
                         int binary, int probe, cudaStream_t stream);

/* K1  Neuron dynamics over one time chunk from the exact current cur [B*KR][n] (row
 *     b*KR+s, sample-aligned): ALIF/LIF state update, spike and surrogate derivative.
 *     Replaces _step_state (gradients.py:118-129) + heaviside/surrogate_grad
 *     (graph.py:40-52) + the readout spike filter (gradients.py:173-174).
 *     smooth != 0: spikes are 0.5 + d/(1+slope|d|) (surrogate_smooth, graph.py:45-47; the
 *             reference's smooth=True finite-difference mode), raster bit = z > 0.5.
 *     u, a    [B][n] fp64 state, carried across chunks (t0 == 0: fresh zero state, not read)
 *     pass 0 (A): zbar, zsum [B][n] fp64 carried; raster [B][T][ceil(n/32)] bit-packed
 *                 spikes (optional, may be NULL); psi_scratch optional: when given, the
 *                 surrogate rows are parked exactly as pass B does (one-chunk sequences
 *                 then run pass 2 instead of pass 1).
 *     pass 2 (B scan only): the pass-B outputs below from a psi_scratch already filled
 *                 by pass A of the same chunk (no dynamics kernel; cur/u/a unused).
 *     pass 1 (B): wsig [B][n] = W_out^T g; ctab[T] fp32 readout gains c_t.  A backward scan
 *                 over the chunk (second kernel) emits, MN-major (neurons contiguous,
 *                 row stride ldc >= n, ldc % 8 == 0) over (sample b, row rho < KR):
 *                   c_hi/c_lo [B*KR][ldc]  gradient coefficient C_rho (bf16 hi/lo split)
 *                   w_hi/w_lo [B*KR][ldc]  ALIF trace-carry coefficient W_rho (pass NULL
 *                                          when no later chunk needs the trace)
 *                   mdt [B][n] float2      ALIF (M, Dt) of the chunk (always, ALIF)
 *                 psi_scratch [B][KR+1][n] fp32 working buffer of the scan.
 *                 (forward.cu header has the algebra).  KR >= Tc+1, KR % 8 == 0.
 *     reset != 0 (pass B): the soft reset makes G_u per-synapse (neurons.py:266-271); the
 *                 scan (K1r) then emits C for the RAW input operand (K4 with alpha = 0),
 *                 w = W_u, ALIF also wa_hi/wa_lo = W_a, and in mdt: LIF float2
 *                 (M_u, Dt_uu), ALIF float[8] (M_u, M_a, Dt_uu, Dt_ua, Dt_au, Dt_aa, 0, 0)
 *                 per (sample, neuron) -- consumed by K6 (LIF) / K6r (ALIF). */
int spb_forward_chunk(int pass, const double* cur, int B, int n, int Tc, int KR, int len, int t0,
                      int T, double alpha, double theta, double slope, double beta, double rho,
                      double kappa, int reset, int alif, int smooth, double* u, double* a,
                      double* zbar, double* zsum, uint32_t* raster, const float* wsig,
                      const float* ctab, void* c_hi, void* c_lo, void* w_hi, void* w_lo,
                      void* wa_hi, void* wa_lo, int ldc, float* mdt, float* psi_scratch,
                      cudaStream_t stream);


/* K1rec Recurrent hidden layer (forward_rec.cu, parity unpinned):
 *     u <- alpha u + (cur[row][i] + sum_{j: z_{t-1}[j]} W_rec[i][j]), otherwise as K1.
 *     wrecT [n][n] = W_rec transposed (fp32, or fp64 with w_is_f64), n <= 2048; one CTA
 *     per sample, the recurrent sum over active j ascending in fp64.  pass 0 (A): zbar,
 *     zsum, raster (full words, optional); psi_scratch and zchunk [B][KR][ceil(n/32)]
 *     (row r = spikes z_{t0+r-1}, bit-packed) are written when given (pass B needs both).
 * spb_pack_rec: x~ operand rows (b, s) = [xq row (k bytes, at b*xq_sb + s*xq_st) |
 *     z_{t0+s-1} as n bytes] -> out [B*Tc][Kx], Kx >= k + n; K4 then filters kx = k + n
 *     columns and K5 / K6 produce the gradient of [W | W_rec]. */
int spb_forward_rec_chunk(int pass, const double* cur, const void* wrecT, int w_is_f64, int B,
                          int n, int Tc, int KR, int len, int t0, int T, double alpha,
                          double theta, double slope, double beta, double rho, double kappa,
                          int reset, int alif, int smooth, double* u, double* a, double* zbar,
                          double* zsum, uint32_t* raster, float* psi_scratch, uint32_t* zchunk,
                          cudaStream_t stream);
int spb_pack_rec(const uint8_t* xq, long long xq_sb, long long xq_st, const uint32_t* zchunk,
                 int B, int k, int n, int Tc, int KR, int len, int Kx, uint8_t* out,
                 cudaStream_t stream);

/* K4  Presynaptic filter xbar_t = alpha*xbar_{t-1} + x_t (the factorised LIF trace G_u,
 *     gradients.py:89-94 with H_I = alpha, F rows = x_t; test_gradients.py:81-91).
 *     x byte counts of (b, s) at x[b*stride_b + s*stride_t + j] (the K2 operand xq works);
 *     xbar_state [B][k] fp64 carry (fresh != 0: start from zero); xh/xl [B*KR][kp] bf16
 *     hi/lo split, MN-major (channels
 *     contiguous, kp >= k, kp % 8 == 0): row b*KR + rho, rho = 0 holds xbar_{t0-1},
 *     rho = s+1 holds xbar_{t0+s}; zero elsewhere. */
int spb_xbar_chunk(const uint8_t* x, long long stride_b, long long stride_t, int B, int k, int kp,
                   int KR, int len, int fresh, double alpha, double* xbar_state, void* xh,
                   void* xl, cudaStream_t stream);
/* Same contract as spb_xbar_chunk, computed on 64-row time segments (KR/64 x the threads;
 * values equal up to fp64 rounding): for a K4 on the critical path (multi-chunk pass B). */
int spb_xbar_chunk_seg(const uint8_t* x, long long stride_b, long long stride_t, int B, int k, int kp,
                       int KR, int len, int fresh, double alpha, double* xbar_state, void* xh,
                       void* xl, cudaStream_t stream);
/* Multi-chunk raw-spike operand: xh rows rho >= 1 = the raw spikes of the chunk (exact in
 * bf16, no lo part), row 0 = 0; the fp64 filter state xbar_state is advanced with alpha
 * (as spb_xbar_chunk) and the entry state xbar_{t0-1} is written to xs_hi/xs_lo [B][kp]
 * (bf16 hi/lo) for the row-0 terms of K5 (a K = B GEMM) and K6 (epilogue). */
int spb_xbar_chunk_raw(const uint8_t* x, long long stride_b, long long stride_t, int B, int k,
                       int kp, int KR, int len, int fresh, double alpha, double* xbar_state,
                       void* xh, void* xs_hi, void* xs_lo, cudaStream_t stream);

/* K3  Readout + loss: s_b = W_out zsum_b, loss_b = CE(s_b, y_b), g_b = softmax - onehot,
 *     wsig_b = W_out^T g_b.  Replaces gradients.py:163-164,177-178 and
 *     softmax_cross_entropy (gradients.py:66-75).  wout [m][n] fp64; labels int64 [B]
 *     (checked in range by the host: LabelOutOfRange); correct[b] = argmax(s_b)==y_b. */
int spb_readout_loss(const double* wout, const double* zsum, const long long* labels, int B, int n,
                     int m, double* s_out, double* loss, double* g, float* wsig, int* correct,
                     cudaStream_t stream);

/* K7  gwo[c][i] = sum_b g[b][c] zsum[b][i]   (gradients.py:181, summed over the batch). */
int spb_readout_grad(const double* g, const double* zsum, int B, int n, int m, double* gwo,
                     cudaStream_t stream);

/* K5  Chunk gradient GEMM on tcgen05 tensor cores (TMA-fed, bf16 hi/lo split, fp32
 *     TMEM accumulation) on CTA pairs (cta_group::2, 256x256 per pair; each split runs on
 *     2*ceil(ldp/256)*ceil(M/256) CTAs), split-K over `splits`:
 *       partial[z][i][j] = sum_{K in split z} (Ah+Al)[K][i] (Bh+Bl)[K][j]  (i<M, j<ldp)
 *     at partial + z*slice_stride (row stride ldp); every slice is written for rows <
 *     round_up(M,128).  Requires ldp % 8 == 0, slice_stride >= round_up(M,128)*ldp.
 *     bl = NULL: B exact in bf16 (raw spikes), 2 MMAs per step.
 *     With A = C (K1) and B = xbar (K4) this is every intra-chunk gradient term: the
 *     factorisable LIF part G_u = 1 (x) xbar and the intra-chunk ALIF part.  Replaces the
 *     xbar/xsum n x k accumulation of gradients.py:165-172,180.  A* [K][lda] MN-major
 *     (lda >= M, lda % 8 == 0), B* [K][ldb] MN-major (ldb >= N_rows, ldb % 8 == 0);
 *     16-byte aligned, K % 8 == 0. */
int spb_grad_gemm_partials(const void* ah, const void* al, int lda, const void* bh, const void* bl,
                           int ldb, int M, int N_rows, int K, int splits, float* partial, int ldp,
                           long long slice_stride, cudaStream_t stream);

/* K5s CUDA-core version of K5 on the same operands (test cross-check only). */
int spb_grad_gemm_simt(const void* ah, const void* al, int lda, const void* bh, const void* bl,
                       int ldb, int M, int N, int K, double* grad, int ldg, cudaStream_t stream);

/* K6  ALIF adaptation trace carried across chunks on tcgen05 tensor cores (elig.cu), on
 *     CTA pairs (tcgen05.mma.cta_group::2: 256 neurons x 256 inputs per pair, eps streamed
 *     in 128 x 32 TMA boxes through an 8-slot ring); each of the `splits` sample ranges
 *     runs on 2 * ceil(kp/256) * ceil(n_pad/256) CTAs:
 *       E_end[b,i,:] = Dt[b,i] E0[b,i,:] + sum_rho W_rho[b,i] xbar_rho[b,:]   (if do_mma)
 *       partial[z][i][j] = sum_{b in split z} M[b,i] E0[b,i,j]
 *     eps [B][n_pad][ke] fp32 (E0 read if load_eps, E_end written if store_eps), w* the K1s
 *     operand [B*KR][ldw] and x* the K4 operand [B*KR][kp] (both MN-major), mdt from K1s;
 *     partial [splits][n_pad][kp].
 *     n_pad % 128 == 0, kp % 128 == 0, ke % 4 == 0, KR % 32 == 0.  Replaces the ALIF G_a
 *     block of eprop_trace_update (gradients.py:89-94) and x_step (gradients.py:165-167).
 *     xl = NULL: the raw-spike operand (rows rho >= 1 raw spikes, row 0 zero; W from scan
 *     pass 3/4 with the input filter folded in), 2 MMAs per step; then xs_hi/xs_lo [B][kp]
 *     (spb_xbar_chunk_raw's entry state, NULL for a fresh state) add the row-0 term
 *     W_0[b,i] xbar_{t0-1}[b,j] to E_end in the epilogue. */
int spb_alif_carry_chunk(const void* wh, const void* wl, int ldw, const void* xh, const void* xl,
                         const float* mdt, float* eps, float* partial, int B, int n, int n_pad,
                         int k, int ke, int kp, int KR, int splits, int do_mma, int load_eps,
                         int store_eps, const void* xs_hi, const void* xs_lo,
                         cudaStream_t stream);

/* K6r The ALIF trace PAIR (G_u, G_a) of reset=True carried across chunks on tcgen05
 *     (elig_reset.cu): with (W_u, W_a), M, Dt from K1r and the raw input x (K4, alpha=0)
 *       (E_u, E_a)_end = Dt (E_u, E_a)_0 + sum_rho (W_u, W_a)_rho x_rho   (if do_mma)
 *       partial[z][i][j] = sum_{b in split z} (M_u E_u0 + M_a E_a0)[b,i,j]
 *     eps_u / eps_a [B][n_pad][ke] fp32; coef [B][n][8]; layouts and padding as K6
 *     (tiles of 128 neurons x 64 inputs).  Replaces the reset branch of the ALIF
 *     eprop_trace_update (gradients.py:89-94, neurons.py:266-271). */
int spb_reset_carry_chunk(const void* wu_hi, const void* wu_lo, const void* wa_hi,
                          const void* wa_lo, int ldw, const void* xh, const float* coef,
                          float* eps_u, float* eps_a, float* partial, int B, int n, int n_pad,
                          int k, int ke, int kp, int KR, int splits, int do_mma, int load_eps,
                          int store_eps, cudaStream_t stream);

/* grad[i][j] (+)= sum_{s<splits} partial[s][i][j] in fixed order (fp64); accumulate = 0
 * overwrites. */
int spb_reduce_partials(const float* partial, int splits, int n, int n_pad, int k_pad,
                        int accumulate, double* grad, cudaStream_t stream);

/* Streaming inputs: copy rows of `row_bytes` from pinned host memory (pitch src_pitch)
 * into a device chunk buffer (pitch dst_pitch) with cudaMemcpy2DAsync on `stream`. */
int spb_copy_chunk_h2d(void* dst, long long dst_pitch, const void* src, long long src_pitch,
                       long long row_bytes, int rows, cudaStream_t stream);

/* Real-valued (non-count) inputs, one chunk: x [B][len][k] fp32 (x_is_f64 = 0) / fp64 with
 * sample stride stride_b (elements) -> the raw-input GEMM operand as bf16 hi/lo pairs
 * xh, xl [B*KR][ld] (row b*KR + s + 1 = step s; rows s >= len zero; row b*KR untouched),
 * x = hi + lo to ~2^-16 relative.  The projection of such inputs is an fp64 GEMM (the
 * exact INT8 path needs integer counts). */
int spb_pack_real(const void* x, int x_is_f64, long long stride_b, int B, int k, int len, int KR,
                  int ld, void* xh, void* xl, cudaStream_t stream);

/* HOST helper of the drop-in's staging (host.cu; x and out are HOST pointers, no stream):
 * uint8 counts x [rows][k] -> out [rows][ceil(k/8)] bit-packed like
 * np.packbits(x, axis=-1, bitorder="little").  Returns 0 when every count is 0 or 1, 1
 * when some count is > 1 (out then partial; the caller stages the bytes instead), 2 on
 * bad arguments.  Thread-safe on disjoint row ranges. */
int spb_host_pack_bits(const uint8_t* x, long long rows, int k, uint8_t* out);

/* out[r][c] = acc[r*ld + c] cast to fp32 (out_is_f64=0) or fp64. */
int spb_finalize_grad(const double* acc, int rows, int cols, int ld, void* out, int out_is_f64,
                      cudaStream_t stream);

/* Data-parallel allreduce payload (parallel.py GradPacker) in one launch:
 * out = [acc[:, :k] (n*k) | gwo (m*n) | sum_b loss[b] | sum_b correct[b]] in fp32
 * (out_is_f64=0) or fp64; the two sums in sample order.  Replaces the host-side packing
 * the reference never needed (it is single-process: reference/pkg/src/sparseprop/training.py). */
int spb_pack_grads(const double* acc, int n, int k, int ld, const double* gwo, int m,
                   const double* loss, const int* correct, int B, void* out, int out_is_f64,
                   cudaStream_t stream);

/* On-device synthetic spikes (poisson.cu): out[b*stride_b + t*ceil(k/8) + (j>>3)] bit (j&7)
 * = 1 with probability rates[labels[b]][j] for t < T, global step t0+t, Philox4x32-10
 * keyed by `seed`, counter (byte, step, sample) -- reproducible in any chunking; the
 * distribution of sample_events (datasets.py:65-67), not numpy's bits. */
int spb_poisson_bits(const float* rates, const long long* labels, int B, int T, int k, int t0,
                     unsigned long long seed, uint8_t* out, long long stride_b,
                     cudaStream_t stream);

/* Optimizer steps on device after the gradient / allreduce, restating
 * sgd_update / adam_update (training.py:58-91) operation by operation in the parameter
 * dtype (p_is_f64 ? fp64 : fp32).  p [rows][cols] (and Adam moments m, v, same dtype) are
 * updated in place; the gradient is g [rows][ld_g] (fp64 accumulator or the packed
 * allreduce buffer, g_is_f64), multiplied by g_scale (1/B for a batch mean) and rounded
 * to the parameter dtype first; t >= 1 is the Adam step count after increment; mirror
 * (optional, fp64 [rows][cols]) receives the updated parameter. */
int spb_sgd_update(void* p, int p_is_f64, int rows, int cols, const void* g, int g_is_f64,
                   int ld_g, double g_scale, double lr, double* mirror, cudaStream_t stream);
/* SGD on the input weights fused with their re-slicing (spb_slice_weights) for the next
 * update's projection: w [n][k] (fp32 / fp64 by w_is_f64) <- w - lr*(g_scale*g) exactly as
 * spb_sgd_update, then wq/sexp re-derived from the new w.  One launch instead of two. */
int spb_sgd_slice_update(void* w, int w_is_f64, int n, int k, const void* g, int g_is_f64,
                         int ld_g, double g_scale, double lr, int Kpad, int n_pad32, int P,
                         int8_t* wq, int* sexp, cudaStream_t stream);
int spb_adam_update(void* p, void* m, void* v, int p_is_f64, int rows, int cols, const void* g,
                    int g_is_f64, int ld_g, double g_scale, double lr, double beta1, double beta2,
                    double eps, int t, double* mirror, cudaStream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* SPARSEPROP_B200_H */
