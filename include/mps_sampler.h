/*
 * mps_sampler.h — C ABI of the B200-native displaced-MPS sampler.
 *
 * This is the drop-in boundary for the hot path named by BASELINE.json
 * north_star: the per-mode chain  temp(n x chi) . Gamma(chi x chi D)  ->
 * displacement einsum -> |amplitude|^2 marginal -> inverse-CDF draw ->
 * gather + renormalise.
 *
 * The reference (gbsemu) exposes its samplers through method dispatch in
 * batch_sample(config, ...) (pkg/src/gbsemu/sampler.py:706-723) with a frozen
 * validated config (sampler.py:51-79) and a SampleBatch result
 * (sampler.py:82-95).  It has no native layer; this library is what a new
 * method "mps" in that dispatch binds through ctypes (INTEGRATION.md shows
 * the stub).  Entry points and the reference interface each replaces:
 *
 *   mps_create / mps_destroy  — per-process engine state; replaces the
 *       per-worker initializer _pool_init (sampler.py:658-663): one context
 *       per GPU, one process per GPU.
 *   mps_set_site              — loads Gamma^[m]; replaces "load the stored
 *       MPS from disk" / the read-only table hand-off to
 *       workers (sampler.py:661-663).
 *   mps_set_streams           — seeds the counter-based streams; replaces
 *       SamplerConfig.seed + _stream_uniforms (sampler.py:109-125).
 *   mps_sample                — N-sample batch; replaces _chunk_chain
 *       (sampler.py:628-655) for method "mps".
 *   mps_sample_range          — one pipeline stage (modes [m_begin, m_end)),
 *       state in/out on the device; the mode-pipelined layout.
 *   mps_last_error            — message for the last non-zero status.
 *
 * Status codes mirror gbsemu/errors.py:8-29 (and the CLI exit codes):
 *   0 ok, 1 generic GbsError (CUDA runtime failure), 2 ValidationError,
 *   3 ResourceGuardError (out of memory / budget), 4 NumericalError.
 *
 * Conventions:
 *   * Gamma^[m] is chi_l x chi_r x D complex, C order (d fastest), so its
 *     reshape(chi_l, chi_r*D) is free.
 *   * disp[b][m] is D x D complex indexed [out k][in d];
 *     E[j][k] = sum_d C[j][d] disp[k][d].
 *   * complex numbers are interleaved (re, im) float64 pairs (complex128).
 *   * counts are int32, N x M row-major; uniforms are float64 N x M.
 *   * Any array argument may be a host or a device pointer (detected with
 *     cudaPointerGetAttributes).  When every output is a device pointer the
 *     call is asynchronous on `stream`; otherwise it returns after the
 *     results are on the host.
 *   * The caller owns every buffer; the library borrows pointers for the
 *     call only (sites: see MPS_SITE_*).
 *   * Calls on one context are serialised by the library (a per-context lock
 *     held while a call validates, stages and enqueues its work); distinct
 *     contexts are independent.  ctypes releases the GIL around every call.
 */
#ifndef MPS_SAMPLER_H
#define MPS_SAMPLER_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPS_OK 0
#define MPS_ERR_GENERIC 1
#define MPS_ERR_VALIDATION 2
#define MPS_ERR_RESOURCE 3
#define MPS_ERR_NUMERICAL 4

/* mps_set_site flags */
#define MPS_SITE_HOST 0          /* gamma is host memory: copied into context-owned HBM */
#define MPS_SITE_DEVICE_COPY 1   /* gamma is device memory: copied */
#define MPS_SITE_DEVICE_BORROW 2 /* gamma is device memory: borrowed, caller keeps it alive AND
                                    unchanged -- the context derives private copies from it at
                                    load time (3M sum plane, small-chain layout, INT8 digit planes),
                                    so an in-place edit must be followed by mps_set_site again */
#define MPS_SITE_HOST_STREAM 3   /* gamma is host memory, kept there (pinned via cudaHostRegister
                                    unless already pinned; caller keeps it alive) and streamed
                                    into a 2-slot HBM ring on a copy stream ahead of each GEMM:
                                    for MPS larger than the GPU (complex128 only) */

/* dtype (all sites of a context share it; state_in / state_out use the same type) */
#define MPS_C128 0
#define MPS_C64 1   /* complex64 chain: K1 on tcgen05 (3xTF32), draw in fp64, parity 1e-4 */

/* per-sample status bits written to `status` */
#define MPS_STATUS_FAILED 1      /* step norm sum_k p(k) not finite / not positive */
#define MPS_STATUS_FLAGGED 2     /* some draw had |cdf[k] - u| <= 1e-10 */

typedef struct mps_ctx mps_ctx;

/* Create a context on one device.  n_dev must be 1 (one process per GPU; the
 * multi-GPU layouts run one context per rank).  layout: 0 sample-sharded,
 * 1 mode-pipelined (informational: a stage simply holds a subset of sites). */
int mps_create(int n_dev, const int* dev_ids, int layout, mps_ctx** out);

/* Declare the chain: M sites of physical dimension D.  Must precede set_site. */
int mps_configure(mps_ctx* ctx, int M, int D);

/* Load site m (chi_l x chi_r x D complex128).  chi_l must equal the chi_r of
 * site m-1 when that site is loaded; chi_0 = chi_M = 1 is not enforced so
 * a stage may start mid-chain. */
int mps_set_site(mps_ctx* ctx, int m, int chi_l, int chi_r, int D,
                 const void* gamma, int flags, int dtype);

/* Seed the on-device counter streams (used when uniforms / alpha are NULL):
 * uniforms of sample i are _stream_uniforms(seed, i, M) bit-for-bit
 * (sampler.py:109-125); alpha_sigma >= 0 enables on-device alpha ~ CN(0, sigma^2)
 * from the alpha stream (oracle decision 7); alpha_sigma < 0 disables it.
 * seed must be < 2^63 (MPS_ERR_VALIDATION otherwise): numpy turns larger seeds in a
 * key list into float64, which collapses the alpha stream's block keys; the raw
 * uniform stream (mps_stream_uniforms) keeps numpy's behaviour for any seed. */
int mps_set_streams(mps_ctx* ctx, uint64_t seed, double alpha_sigma);

/* Sample n paths (global sample indices first_index .. first_index+n-1)
 * through all M sites.  uniforms: n x M or NULL (device stream); disp:
 * n x M x D x D complex or NULL; alpha: n x M complex or NULL (if both are
 * NULL the on-device alpha stream is used when enabled, else no displacement).
 * counts: n x M int32 out (failed samples: row of -1); marginals: n x M x D
 * normalised float64 out or NULL; n_flagged: out, may be NULL. */
int mps_sample(mps_ctx* ctx, int64_t first_index, int n,
               const double* uniforms, const void* disp, const void* alpha,
               int32_t* counts, double* marginals, uint64_t* n_flagged);

/* One stage: modes [m_begin, m_end) for n samples.  Arrays are full-width
 * (column = absolute mode index) with row strides ld_u / ld_c (elements);
 * marginals use row stride ld_c * D.  state_in: device n x chi_{m_begin}
 * complex or NULL (= ones, only valid when chi_{m_begin} == 1); state_out:
 * device n x chi_{m_end} complex or NULL.  status: n bytes in/out (bits
 * MPS_STATUS_*), may be NULL.  stream: the cudaStream_t to run on (0 = the
 * legacy default stream); mps_sample runs on the context's own stream. */
int mps_sample_range(mps_ctx* ctx, int m_begin, int m_end, int64_t first_index, int n,
                     const double* uniforms, int64_t ld_u,
                     const void* disp, const void* alpha,
                     const void* state_in, void* state_out,
                     int32_t* counts, int64_t ld_c, double* marginals,
                     uint8_t* status, uint64_t stream);

/* Device launches issued by this context since creation (kernels only). */
uint64_t mps_kernel_launches(const mps_ctx* ctx);

/* Live per-kernel timing: enable is a mask (bit 0: K1 site_gemm, bit 1: K2+K3
 * displace_draw); each selected launch is bracketed by CUDA events on its own stream.  mps_profile_read synchronises on them and
 * returns (and resets) out6 = {site_gemm ms, launches, algorithmic flops,
 * displace_draw ms, launches, algorithmic bytes}. */
int mps_profile(mps_ctx* ctx, int enable);
int mps_profile_read(mps_ctx* ctx, double* out6);

const char* mps_last_error(const mps_ctx* ctx);
void mps_destroy(mps_ctx* ctx);

/* Kernel-level entry points, exposed for unit tests and the bench roofline.
 * All pointers are device pointers; stream 0 = legacy default stream. */

/* C (n x N complex, row stride ldc) = V (n x K complex, row stride K) . G (K x N complex);
 * 3M, autotuned tile config. */
int mps_site_gemm(const void* V, const void* G, void* C, int n, int K, int N,
                  int64_t ldc, uint64_t stream);
/* Same with an explicit K1 tile config (-1 autotune, cached per shape; -2 analytic
 * model; 0..3 fixed tiles) and product mode (3: 3M, three real GEMMs; 4: 4M
 * real-doubled).  Within a mode every config gives bit-identical C. */
int mps_site_gemm_cfg(const void* V, const void* G, void* C, int n, int K, int N,
                      int64_t ldc, uint64_t stream, int cfg, int mode);
/* Pin the K1 tile config of a context (-1 = autotune, the default; -2 = model). */
int mps_set_gemm_config(mps_ctx* ctx, int cfg);
/* Concurrent chains per call (1..8, default 2): the micro-batch is split into contiguous
 * row blocks of >= 64 samples, each run on its own stream (forked from and joined back
 * to the caller's stream) so one block's draw kernels and GEMM tails overlap another's
 * GEMMs.  Per-sample results are identical for any lane count. */
int mps_set_lanes(mps_ctx* ctx, int lanes);
/* Micro-batch size for calls with host arrays (0, the default: a call is one micro-batch).  With
 * micro > 0, a mps_sample / mps_sample_range call of n > micro samples runs as micro-batches of
 * `micro` rows, grouped into chunks of about 2 MB of inputs (at most 64 micro-batches): a chunk's
 * inputs go up in one copy per array on a copy-engine stream while the previous chunk computes,
 * its kernels run back to back (programmatic dependent launch), its outputs come down while the
 * next chunk computes; one host synchronisation per call; results are identical. */
int mps_set_micro_batch(mps_ctx* ctx, int micro);
/* Small chains (complex128, 3M product mode, every site chi_l <= 128 and chi_r * D <= 1024):
 * run the whole mode range of a call as ONE persistent kernel -- clusters of 16 CTAs each own
 * 16 sample rows, exchange C rows and the next state through distributed shared memory and never
 * return to the host between modes (the two-kernels-per-mode chain is latency-bound there).
 * Results are bit-identical to the per-mode kernels.  mode 0: off; 1: whenever eligible;
 * 2 (default): when its latency model beats the per-mode kernels' for the call's n (one to a few
 * waves of 16-row groups); 3: as 1 but never the tiny-chain kernel (mps_small_chain_eligible).
 * MPS_SMALL_CHAIN=0 / =1 / =3 set modes 0 / 1 / 3 at context creation. */
int mps_set_small_chain(mps_ctx* ctx, int mode);
/* Which whole-chain kernel mps_sample_range over [m_begin, m_end) with n samples would take:
 * 0 the per-mode kernels, 1 the 16-CTA cluster kernel, 2 the tiny-chain kernel (one CTA per 8-row
 * group, every site in shared memory: chi_l, chi_r <= 32, chi_r D <= 256; taken in modes 1 and 2
 * whenever eligible -- faster than both other paths at any n).  Mode 3 of mps_set_small_chain is
 * mode 1 without the tiny kernel (A/B and tests).  All paths give the same bits. */
int mps_small_chain_eligible(const mps_ctx* ctx, int m_begin, int m_end, int n);
/* Teacher forcing (the oracle's forced=, the pattern of gbsemu's forced path, sampler.py:394-416):
 * when enabled, mps_sample / mps_sample_range read sample b's outcome at mode m from counts
 * (an INPUT, left unchanged) instead of drawing it, and still return the normalised marginals
 * along that path -- the per-mode conditional probabilities, whose logs sum to the sample's log
 * probability under the chain.  An outcome outside [0, D) marks the sample failed; uniforms
 * are ignored. */
int mps_set_forced(mps_ctx* ctx, int enable);
/* Sum planes for the 3M GEMM (default on): mps_set_site stores Gr+Gi next to each site
 * (+50% of the site's HBM, skipped per site when memory is short) and the draw kernel
 * writes Vr+Vi next to the state, so K1 loads the operand sums instead of forming them
 * on the FP64 pipe.  Results are bit-identical either way.  Set before loading sites. */
int mps_set_sum_planes(mps_ctx* ctx, int enable);
/* K1 complex product: 3 = 3M (default), 4 = 4M, both on the FP64 DMMA pipe; 8 = fp64
 * emulated on the INT8 tcgen05 tensor cores (Ozaki scheme, 7 digits of 7 bits per operand,
 * ~1e-13 of the row scales; opt-in).  Results of the modes differ at rounding level; each is
 * deterministic across batch sizes and GPU counts. */
int mps_set_gemm_mode(mps_ctx* ctx, int mode);
/* Digits per operand of gemm mode 8 (Ozaki): 7 (default, ~1e-13 of the row scales), 6 (25% fewer
 * INT8 products, ~1e-11) or 5. */
int mps_set_ozaki_digits(mps_ctx* ctx, int S);
/* Where gemm mode 8 keeps the sites' digit planes (1.75x the site bytes at 7 digits): 0 resident
 * (built once per site), 1 streamed (sliced per call, column block by column block, into a 2-slot
 * ring on a copy stream that runs ahead of the GEMMs: for stages whose planes do not fit, e.g. C5),
 * 2 auto (default: streamed when the planes would not fit in free memory).  block_cols: complex
 * columns per streamed block (0: ~4 GB of planes per block).  Results are identical in all modes. */
int mps_set_ozaki_site_mode(mps_ctx* ctx, int mode, int block_cols);
/* complex128 K1 emulated on the INT8 tensor cores (Ozaki scheme with S = 5..7 digits):
 * C (n x N) = V (n x K) . G (K x N), all complex128.  Test/benchmark entry (slices per call). */
int mps_site_gemm_ozaki(const void* V, const void* G, void* C, int n, int K, int N, int S, uint64_t stream);
/* Its pieces: int8 digit planes (S planes of rows_pad x ld bytes in the tiled stage layout of
 * ozaki_gemm.cuh; ld = 2K rounded up to a multiple of 32, rows_pad a multiple of 256) and
 * exponents of a state (n x K) and of a site's B_r^T (2N rows), and the GEMM on them. */
int mps_ozaki_state_planes(const void* V, int n, int K, int S, int8_t* planes, int* e, int ld, int n_pad,
                           uint64_t stream);
int mps_ozaki_site_planes(const void* G, int K, int N, int S, int8_t* planes, int* e, int ld, int b_pad,
                          uint64_t stream);
int mps_ozaki_gemm_planes(const int8_t* a_planes, int n_pad, const int* ea, const int8_t* b_planes, int b_pad,
                          const int* eb, int ld, void* C, int n, int K, int N, int S, uint64_t stream);
/* complex64 K1 on the tcgen05 tensor cores (kind::tf32, 3xTF32 split, fp32 accumulate):
 * C (n x N complex64) = V (n x K complex64) . G (K x N complex64).  Test/benchmark entry:
 * builds the hi/lo operand planes in temporary memory on every call. */
int mps_site_gemm_c64(const void* V, const void* G, void* C, int n, int K, int N, uint64_t stream);
/* The pieces of it: tf32 hi / lo planes of a complex64 state (rows x cols -> rows x ld fp32,
 * ld >= 2 cols, ld % 4 == 0) and of a complex64 site (K x N -> B_r^T, 2N x ld), and the
 * GEMM on prepared planes. */
int mps_c64_state_planes(const void* V, int rows, int cols, float* hi, float* lo, int ld, uint64_t stream);
int mps_c64_site_planes(const void* G, int K, int N, float* hi, float* lo, int ld, uint64_t stream);
int mps_c64_gemm_planes(const float* ahi, const float* alo, const float* bhi, const float* blo, int ld, void* C,
                        int n, int K, int N, uint64_t stream);
/* Fused stage hand-off over peer memory (mode-pipelined layout; replaces the NCCL send/recv of
 * the n x chi state).  The receiving stage allocates its input buffers with mps_ipc_alloc and
 * passes the 64-byte handles to the previous stage's process, which maps them with mps_ipc_open
 * (NVLink peer memory) and hands the mapped pointer to mps_sample_range as state_out, so its last
 * draw kernel writes the state into the next GPU directly.  Interprocess events (64-byte
 * handles) order the two sides on the GPU: mps_event_record after the producer's stage,
 * mps_stream_wait_event before the consumer's (and the reverse for buffer reuse). */
int mps_ipc_alloc(uint64_t bytes, void** dptr, void* mem_handle64);
int mps_ipc_free(void* dptr);
int mps_ipc_open(const void* mem_handle64, void** dptr);
int mps_ipc_close(void* dptr);
int mps_ipc_event_create(void** ev, void* ev_handle64);
int mps_ipc_event_open(const void* ev_handle64, void** ev);
int mps_event_record(void* ev, uint64_t stream);
int mps_stream_wait_event(uint64_t stream, void* ev);
int mps_event_destroy(void* ev);
/* D x D truncated displacement matrices for `count` alphas: out[count][D][D] */
int mps_displacement(const void* alpha, int count, int D, void* out, uint64_t stream);
/* Uniforms of samples first..first+count-1 (count x M float64), bit-equal to
 * numpy Philox / _stream_uniforms. */
int mps_stream_uniforms(uint64_t seed, int64_t first, int count, int M, double* out,
                        uint64_t stream);

#ifdef SC_TRACE
/* Debug builds only (-DSC_TRACE, tools/chain_trace.py): copy the small-chain kernel's clock64
 * stamps of CTA 0 (2 x 256 x 8 long long: producer / owner side, per mode) to out. */
int mps_debug_chain_trace(long long* out);
/* (-DSC_TRACE) the pipelined-halves kernel's stamps (4 x 256 x 8 long long), tools/chain2_trace.py */
int mps_debug_chain2_trace(long long* out);
#endif
#ifdef TC_TRACE
/* Debug builds only (-DTC_TRACE, tools/tiny_trace.py): the tiny-chain kernel's clock64 stamps of
 * CTA 0, warp 0 (64 modes x 8 long long). */
int mps_debug_tiny_trace(long long* out);
#endif
#ifdef DRAW_TRACE
/* Debug builds only (-DDRAW_TRACE, tools/draw_trace.py): m >= 0 arms the per-CTA globaltimer trace
 * of the draw kernel for mode m; m < 0 copies it (8192 CTAs x 8 long long: 6 phase stamps, -, smid). */
int mps_debug_draw_trace(int m, long long* out);
#endif

#ifdef __cplusplus
}
#endif

#endif /* MPS_SAMPLER_H */
