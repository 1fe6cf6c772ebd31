/*
 * blade_ms.h — C ABI of the B200 (sm_100a) multiscale BLADE denoiser, inference path.
 *
 * Method: arxiv 1802.06130 (reference text /root/reference/PAPER.md; citations below are
 * "PAPER.md:<lines> (<section>, <equation>)"). The library computes, for each RGB frame z:
 *
 *   pyramid      z^{l+1} = bicubic 2x decimation of z^l          PAPER.md:260-263 (§4)
 *   selector     s^l(i)  = bucket(orientation, strength, coherence of the joint-colour
 *                          structure tensor T_i of z^l)           PAPER.md:131-148 (§3, Eq. 6)
 *   stage        u^l_i   = sum_j f^{l,s(i)}_j u^{l+1}_{i/2+j} + sum_j g^{l,s(i)}_j z^l_{i+j}
 *                                                                 PAPER.md:269-271 (§4, Eq. 9)
 *   cascade      u^{L-1} = z^{L-1}; l = L-2 .. 0                  PAPER.md:284-289 (§4)
 *   single-level (L == 1): u_i = sum_j h^{s(i)}_j z_{i+j}         PAPER.md:81-83 (§3, Eq. 1)
 *
 * Readings of points the paper leaves open (border, gradient, window, quantiser, phase,
 * normalisation, ...) are DESIGN.md R1..R24; the ones that shape this interface are cited
 * inline as [Rn].
 *
 * Conventions
 *   - Images are planar fp32 NCHW with C = 3 (R, G, B), contiguous, values on any scale
 *     (the configs use [0, 1]) [R1]. Row y runs down, column x runs right.
 *   - Border handling is half-sample symmetric (numpy 'symmetric'), periodic for offsets
 *     beyond one period, applied to every level's image [R2].
 *   - Level dims: H_{l+1} = ceil(H_l / 2), W likewise [R16]. "levels" = number of pyramid
 *     images L (L-1 decimations, L-1 stages; L == 1 is fixed-scale Eq. 1).
 *   - All entry points are asynchronous on the caller's CUDA stream (cudaStream_t passed as
 *     void*; NULL = legacy default stream) unless stated; no host synchronisation happens.
 *   - Errors: every argument error is detected BEFORE any launch (no partial writes) and
 *     returned as a blade_status; blade_ms_last_error() returns a thread-local message.
 *     Asynchronous device faults surface at the caller's next synchronisation.
 *   - Thread safety: a handle's bank and plan are immutable after create; concurrent calls
 *     with distinct workspaces/outputs (on any streams) are safe, except while profiling is on
 *     (blade_ms_set_profiling). blade_ms_denoise_pipelined's internal streams and fork/join
 *     events are shared by the handle: concurrent pipelined calls are serialised on the host
 *     (a per-handle mutex held from fork to join), so each call's chunks wait on its own
 *     caller stream; their device work may serialise, and a caller's join may also wait for
 *     another call's chunks queued before its own. destroy must not race pending work.
 *   - Non-finite PIXEL values are not checked (it would cost a pass); outputs are then
 *     unspecified. Non-finite TAPS and thresholds are rejected at create.
 */
#ifndef BLADE_MS_H
#define BLADE_MS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct blade_ms* blade_ms_t; /* opaque handle; immutable after create */

typedef enum {
  BLADE_OK = 0,
  BLADE_EINVAL = 1,       /* bad argument: null pointer, bad size, overlap, ...          */
  BLADE_ENONFINITE = 2,   /* NaN/Inf tap or threshold                      */
  BLADE_ESHAPE = 3,       /* tap count / workspace size / band extent mismatch           */
  BLADE_EDEVICE = 4,      /* pointer not on the handle's device, or bad device ordinal   */
  BLADE_ENOMEM = 5,       /* device allocation failed at create                          */
  BLADE_ECUDA = 6,        /* a CUDA call or launch failed (message in last_error)        */
  BLADE_EUNSUPPORTED = 7  /* valid per the paper but not built (see blade_ms_create)     */
} blade_status;

typedef struct {
  int32_t levels;            /* L >= 1 pyramid images; 1 => fixed-scale Eq. 1; max 12           */
  int32_t fine_size;         /* n_f: odd, 1..9; the g block (and the single-level h)           */
  int32_t coarse_size;       /* n_c: odd, 1..9 if L >= 2; must be 0 if L == 1 (f block)         */
  int32_t n_phases;          /* 4 = pair indexed by (2(y mod 2) + (x mod 2), bucket) [R9];
                                1 = bucket only (SPEC.md reading); must be 1 if L == 1          */
  int32_t n_filter_channels; /* 1 = one filter for R, G and B [R13]; 3 = per-channel Y, Cb, Cr
                                banks with the shared RGB selector (PAPER.md:198-202 footnote 1;
                                full-range BT.601 [R25])                          */
  int32_t window_size;       /* structure-tensor window: 1, 3 or 5 (configs: 5) [R4]            */
  float window_sigma;        /* Gaussian std of the window, > 0 (configs: 1.5) [R4]             */
  int32_t clamp_output;      /* 0 = raw cascade output (parity); 1 = clamp final u^0 to [0,1]
                                (SPEC.md:447 clamps only at the end) [R24]                      */
} blade_ms_config;

typedef struct {
  int32_t n_orient;    /* n_o >= 1 orientation bins over [0, pi) (configs: 16)                 */
  int32_t n_strength;  /* n_s >= 1 (configs: 3)                                                */
  int32_t n_coherence; /* n_c >= 1 (configs: 3); K = n_o * n_s * n_c <= 65536: K <= 256 keeps uint8
                          maps and the bank in shared memory; K > 256 (e.g. the paper's 16 x 16 x
                          16) uses uint16 maps and an L2-resident bank (NEXT f2)     */
  /* Thresholds per stage, stage index = output level l (0 = finest), n_stages = max(L-1, 1):
     strength_thresholds[stage * (n_s - 1) + t], coherence_thresholds[stage * (n_c - 1) + t];
     strictly ascending and finite within a stage. Quantiser [R7]:
       o = floor(theta * n_o / pi) mod n_o, s = #{t <= S}, k = #{t <= C},
       bucket = (o * n_s + s) * n_c + k.
     The device compares fp32 features with fp32 thresholds: pass fp32-representable values
     (a double that is not is rounded UP to the next fp32, which keeps "t <= S" exact for
     fp32 S). May be NULL when the matching count is 1. Copied at create. */
  const double* strength_thresholds;
  const double* coherence_thresholds;
} blade_bucket_layout;

/*
 * Create a handle on CUDA device `device` (ordinal).
 *   taps: HOST fp32, n_taps = n_stages * n_filter_channels * n_phases * K * (n_f^2 + n_c^2),
 *         layout [stage][channel][phase][bucket][ fine n_f*n_f row-major | coarse n_c*n_c ];
 *         tap (dy, dx) (row-major from (-r, -r)) multiplies the sample at (y+dy, x+dx) of z^l
 *         (fine) or (floor(y/2)+dy, floor(x/2)+dx) of u^{l+1} (coarse): correlation, as in
 *         Eq. 1 "z_{i+j}" [R12]. Copied (and re-laid for the kernels) at create; the caller
 *         may free its arrays on return.
 * Every odd fine / coarse size in 1..9 is built. The pairs 5+5, 3+3, 5+3 (whole bank in shared
 * memory), 7+7, 7+5 (two phases per CTA) and 9+9, 9+7 (one phase per CTA) have TMA-staged kernels;
 * the other pairs, widths that are not multiples of 4 and tiny levels run the generic stage
 * kernel. A shared (K <= 256) bank whose two phases do not fit a CTA's shared memory (e.g. 5+9 at
 * K = 256) is read from global memory like the K > 256 banks. K > 256 with per-channel banks (the
 * paper's own 16 x 16 x 16 x {Y, Cb, Cr} layout) runs too. EUNSUPPORTED remains for GPU training
 * (blade_ms_train_*) of footprints with n_f^2 + n_c^2 > 123 (7+9, 9+7, 9+9), of K > 256 banks other
 * than 7, 5+5, 7+5, 7+7, and of per-channel banks.
 * Errors: EINVAL (null/bad config), ESHAPE (n_taps), ENONFINITE, EUNSUPPORTED, EDEVICE,
 *         ENOMEM, ECUDA. On error *out is set to NULL.
 */
blade_status blade_ms_create(const blade_ms_config* cfg, const blade_bucket_layout* buckets,
                             const float* taps, size_t n_taps, int device, blade_ms_t* out);

/* Bytes of device workspace blade_ms_denoise / _selector / _pyramid need for a batch of N
 * frames of H x W (levels >= 1 images, u^l intermediates, bucket maps, 256-B aligned). */
blade_status blade_ms_workspace_size(blade_ms_t h, int32_t N, int32_t H, int32_t W, size_t* bytes);

/*
 * Denoise a batch: in, out DEVICE fp32 [N][3][H][W] on the handle's device; N >= 0 (0 is a
 * no-op), H, W >= 1. `out` must not overlap `in` (EINVAL). workspace: device, >= the size
 * from blade_ms_workspace_size (ESHAPE otherwise), 16-byte aligned; on return it holds the
 * pyramid levels (fp32 hi / lo pairs carrying the fp64 decimation), intermediate stage outputs
 * and bucket maps, with rows padded to 16-byte multiples (so every level can be read by TMA;
 * a level-0 width that is not a multiple of 4 adds a padded copy of the input and a padded
 * staging output). Output equals a per-frame loop bit-exactly.
 */
blade_status blade_ms_denoise(blade_ms_t h, const float* in, float* out, int32_t N, int32_t H,
                              int32_t W, void* workspace, size_t ws_bytes, void* cuda_stream);

/*
 * End-to-end variant with HOST buffers: copies in_host -> d_in, denoises into d_out and copies
 * d_out -> out_host, all on `cuda_stream`, chunk-pipelined (up to 32 frame chunks: the copy in
 * of chunk n+1 and the copy out of chunk n-1 overlap the compute of chunk n) when the host
 * buffers are page-locked. A single frame of >= 4 Mi px is pipelined as 12 row bands instead (each
 * band computed from its input dependency cone, as blade_ms_denoise_rows: bit-identical to the
 * whole frame). d_in / d_out: device staging buffers of N*3*H*W floats each. Synchronises the
 * stream before returning (the output is in out_host on return). Calls on one handle are
 * serialised (the handle keeps its copy streams and events between calls).
 */
blade_status blade_ms_denoise_host(blade_ms_t h, const float* in_host, float* out_host,
                                   int32_t N, int32_t H, int32_t W, float* d_in, float* d_out,
                                   void* workspace, size_t ws_bytes, void* cuda_stream);

/*
 * Frame-chunked schedule (NEXT f3, SURVEY.md §8 "L2-resident band pipeline on 1 GPU", PAPER.md:314
 * "time is linear in pixels"): the batch is cut into chunks of `chunk` frames (the last one may be
 * shorter); chunk i runs the whole cascade of blade_ms_denoise on internal stream i % n_streams,
 * forked from and joined back into `cuda_stream`, in its own slice of the workspace. A chunk's
 * input, pyramid levels, maps and stage outputs (about 48 MB per 1080p frame) then stay resident
 * in the 126 MB L2 between the down pass and the up pass instead of round-tripping through HBM
 * (DESIGN.md §10c). chunk >= 1, n_streams in 1..4 (EINVAL otherwise). Same buffer rules as
 * blade_ms_denoise; the workspace size comes from blade_ms_pipeline_workspace_size (n_streams
 * slices of a chunk-sized workspace). Output equals blade_ms_denoise bit-exactly. Asynchronous
 * on `cuda_stream` (graph-capturable: the fork / join are event waits).
 */
blade_status blade_ms_pipeline_workspace_size(blade_ms_t h, int32_t chunk, int32_t n_streams,
                                              int32_t H, int32_t W, size_t* bytes);
blade_status blade_ms_denoise_pipelined(blade_ms_t h, const float* in, float* out, int32_t N,
                                        int32_t H, int32_t W, int32_t chunk, int32_t n_streams,
                                        void* workspace, size_t ws_bytes, void* cuda_stream);

/*
 * Row bands (one huge image split over GPUs, BASELINE.json configs[4]).
 * blade_ms_band_rows: input rows [*in_row0, *in_row0 + *in_rows) of the full H-row image needed
 * to produce output rows [out_row0, out_row0 + out_rows) bit-identically to the full-image call
 * (the union of the cascade's dependency cone, clamped to [0, H)).
 */
blade_status blade_ms_band_rows(blade_ms_t h, int32_t H, int32_t out_row0, int32_t out_rows,
                                int32_t* in_row0, int32_t* in_rows);

/*
 * Training (NEXT f4): the per-(phase, bucket) least-squares filters of PAPER.md:186-198 (§3,
 * Eqs. 7-8) for one stage, from noisy / clean pairs (readings R27-R30).
 * blade_ms_train_layout: nt = taps per filter (n_f^2 + n_c^2), ntp = pitch of the accumulator
 * matrices (nt + 1 rounded up to 4), n_seg = n_phases * K.
 */
blade_status blade_ms_train_layout(blade_ms_t h, int32_t* nt, int32_t* ntp, int32_t* n_seg);
blade_status blade_ms_train_workspace_size(blade_ms_t h, int32_t N, int32_t H, int32_t W,
                                           size_t* bytes);
/*
 * Accumulate the normal equations of stage `level` over N frames (DEVICE fp32 [N][3][H][W]):
 * z = the noisy image at that level, u_clean = the clean target at that level, u_coarse = the
 * filtered coarser level u^{level+1} ([N][3][ceil(H/2)][ceil(W/2)]; NULL when levels == 1).
 * Every pixel and every channel is one sample x = [fine patch of z ; coarse patch of u_coarse]
 * (ABI tap order) of the (phase, bucket) segment its selector (computed here from z with the
 * thresholds of `level`) picks. E: DEVICE fp64 [n_seg][ntp][ntp], accumulated (the caller zeroes
 * it once): E[s] = sum [x; u][x; u]^T over the segment, in its upper 4 x 4-block triangle (G in
 * [0, nt)^2, m in column nt). count: DEVICE uint64 [n_seg], accumulated. Asynchronous.
 */
blade_status blade_ms_train_accumulate(blade_ms_t h, int32_t level, const float* z,
                                       const float* u_clean, const float* u_coarse, int32_t N,
                                       int32_t H, int32_t W, double* E, uint64_t* count,
                                       void* workspace, size_t ws_bytes, void* cuda_stream);
/*
 * Solve every segment on the host (fp64 Cholesky): h = (G + ridge tr(G)/nt I)^-1 m when
 * count >= min_count, else the centred fine delta with a zero coarse block. E, count: HOST copies
 * of the accumulators; taps: HOST fp32 [n_phases][K][nt] (the stage's block of the create layout).
 */
blade_status blade_ms_train_solve(blade_ms_t h, const double* E, const uint64_t* count,
                                  double ridge, uint64_t min_count, float* taps);

/* Diagnostic (synchronous): after a blade_ms_denoise / _selector call of N x H x W frames with
 * workspace ws has completed, counts[l] (l < n_stages) = the number of pixels of selector level l
 * whose fp32 orientation bin was not certified and was recomputed in fp64 (DESIGN.md §6 H1).
 * Small denoise calls (DESIGN.md §6 "Small calls": <= 16 Ki px, or <= 768 Ki px with the 16 x 3 x 3
 * bucket layout) recompute those pixels inside the down-pass kernel and leave the counts at 0;
 * blade_ms_selector always counts. */
blade_status blade_ms_fallback_count(blade_ms_t h, int32_t N, int32_t H, int32_t W, const void* ws,
                                     size_t ws_bytes, uint32_t* counts);

/* The same halo query from a configuration alone (host-only, no device, no handle): used to plan
 * the row bands of a multi-GPU split (BASELINE.json configs[4]) before any device is touched. */
blade_status blade_ms_band_plan(const blade_ms_config* cfg, int32_t H, int32_t out_row0,
                                int32_t out_rows, int32_t* in_row0, int32_t* in_rows);

/* Workspace bytes for a band call (depends on the band's input extent). */
blade_status blade_ms_band_workspace_size(blade_ms_t h, int32_t H, int32_t W, int32_t out_row0,
                                          int32_t out_rows, size_t* bytes);

/*
 * Denoise output rows [out_row0, out_row0 + out_rows) of ONE frame of H_full x W, given input
 * rows [in_row0, in_row0 + in_rows) (device, [3][in_rows][W]); the band must cover
 * blade_ms_band_rows (ESHAPE otherwise). out_band: device [3][out_rows][W]. Rows equal the
 * same rows of blade_ms_denoise on the full frame bit-exactly (all indices global: phases use
 * global parity, folds happen at the true image border).
 */
blade_status blade_ms_denoise_rows(blade_ms_t h, const float* in_band, int32_t in_row0,
                                   int32_t in_rows, float* out_band, int32_t out_row0,
                                   int32_t out_rows, int32_t H_full, int32_t W, void* workspace,
                                   size_t ws_bytes, void* cuda_stream);

/*
 * NEXT f3 (b): row bands whose neighbours EXCHANGE halo rows between pyramid levels instead of
 * each recomputing its whole dependency cone (§5: time linear in
 * the pixels). Band b owns output rows [out_row0, out_row0 + out_rows) = own^0 and, at every
 * level, own^{l+1} = [ceil(own^l.lo / 2), ceil(own^l.hi / 2)) — so bands that partition the
 * image partition every level — and computes only those rows; the halo_z rows of z^l and halo_u
 * rows of u^l around them come from the neighbour bands.
 *
 * blade_ms_xband_layout (host only, no handle): the band's plan. Steps s = 0 .. n_steps-1 with
 * n = max(levels - 1, 1): s < n is the down pass at level l = s (selector map s^l of own^l and
 * z^{l+1} of own^{l+1}), s >= n the up pass at level l = 2n-1-s (stage l of own^l; l = 0 writes
 * out_band). After step s, for side 0 (the band above, rows < own) and side 1 (below),
 * send[s][side] names this band's own boundary rows the neighbour needs and recv[s][side] the
 * halo rows to be filled from it (rows == 0: nothing to move). A region is `planes` runs of
 * `rows` x `pitch` fp32 values, global rows [row0, row0 + rows), starting `offset` bytes into
 * the band's workspace, `plane_stride` bytes apart. The band's send[s][1] and the band below's
 * recv[s][0] cover the same global rows (likewise send[s][0] / the band above's recv[s][1]).
 * in_row0 / in_rows: the level-0 input rows the band reads (own^0 +- halo_z, clamped);
 * ws_bytes: its workspace. EUNSUPPORTED when some level of a band (other than the whole image)
 * owns fewer than halo_z rows. K = bucket count (map entry size).
 *
 * blade_ms_xband_step: runs step s of the band on `stream` (asynchronous). The caller moves the
 * recv regions of step s-1 in before calling it (NCCL send/recv between GPUs, a device copy
 * between bands on one GPU). Concatenated band outputs equal blade_ms_denoise of the whole
 * frame bit-exactly (the same kernels compute every row from the same inputs). Argument errors
 * as blade_ms_denoise_rows.
 */
#define BLADE_MAX_LEVELS 12
typedef struct {
  int64_t offset;        /* bytes into the band's workspace                                  */
  int64_t plane_stride;  /* bytes between planes                                             */
  int32_t row0, rows;    /* global rows [row0, row0 + rows) of the level                      */
  int32_t pitch, planes; /* fp32 values per row; planes (3 channels; 6 = hi + lo of z^l)       */
} blade_region;
typedef struct {
  int32_t levels, n_steps, halo_z, halo_u;
  int32_t own_lo[BLADE_MAX_LEVELS], own_hi[BLADE_MAX_LEVELS];
  int32_t in_row0, in_rows;
  uint64_t ws_bytes;
  blade_region send[2 * BLADE_MAX_LEVELS][2], recv[2 * BLADE_MAX_LEVELS][2];
} blade_xband_layout;
blade_status blade_ms_xband_layout(const blade_ms_config* cfg, int32_t K, int32_t H, int32_t W,
                                   int32_t out_row0, int32_t out_rows, blade_xband_layout* layout);
blade_status blade_ms_xband_step(blade_ms_t h, int32_t step, const float* in_band, int32_t in_row0,
                                 int32_t in_rows, float* out_band, int32_t out_row0,
                                 int32_t out_rows, int32_t H_full, int32_t W, void* workspace,
                                 size_t ws_bytes, void* cuda_stream);

/*
 * Diagnostic: the bucket maps s^l (device, [N][H_l][W_l]; uint8 entries when K <= 256, uint16
 * when K > 256 — the paper's 16 x 16 x 16 layout, NEXT f2) for every selector level
 * l = 0 .. n_stages-1 (maps_per_level[l]; a NULL entry skips that level). Also leaves the
 * pyramid in the workspace.
 */
blade_status blade_ms_selector(blade_ms_t h, const float* in, int32_t N, int32_t H, int32_t W,
                               void* const* maps_per_level, void* workspace, size_t ws_bytes,
                               void* cuda_stream);

/* Diagnostic: pyramid levels 1..L-1 into levels[l-1] (device fp32 [N][3][H_l][W_l]). */
blade_status blade_ms_pyramid(blade_ms_t h, const float* in, int32_t N, int32_t H, int32_t W,
                              float* const* levels, void* workspace, size_t ws_bytes,
                              void* cuda_stream);

/* Properties of a handle (host query). */
typedef struct {
  int32_t levels, fine_size, coarse_size, n_phases, n_stages, K;
  int32_t device;
  size_t bank_bytes_device;    /* device copy of the relaid bank                          */
  size_t stage_smem_bytes;     /* dynamic shared memory of the stage kernel (K3)          */
  int32_t stage_phase_groups;  /* 1: a CTA holds all phases (TMA kernels; the phase-split kernel
                                  holds one); 2: generic kernel, CTAs specialised by row parity */
} blade_ms_info;
blade_status blade_ms_get_info(blade_ms_t h, blade_ms_info* info);

/* Number of kernel launches one blade_ms_denoise(N, H, W) call issues. */
blade_status blade_ms_launch_count(blade_ms_t h, int32_t N, int32_t H, int32_t W, int32_t* count);

/* Diagnostic: the stage kernel blade_ms_denoise(N, H, W) runs at stage `level` (0 .. n_stages-1)
 * with 16-byte aligned buffers: *kind = 0 generic k_stage, 1 k_stage_tma, 2 k_stage_ph (phase-
 * split), 3 k_stage_p2 (row-parity CTAs with two phases each); *rows_per_thread = output rows per
 * thread of k_stage_tma (2 or 4; 2 otherwise). Used by
 * bench.py's shared-memory roofline model and the tests. EINVAL for a bad level. */
blade_status blade_ms_stage_kernel(blade_ms_t h, int32_t N, int32_t H, int32_t W, int32_t level,
                                   int32_t* kind, int32_t* rows_per_thread);

/*
 * Per-kernel timing (measurement support for bench.py). While enabled, every launch the handle
 * enqueues is bracketed by two CUDA events recorded on the launching stream. blade_ms_profile_read
 * synchronises on those events and returns, per kernel kind (0 = K1 decimate (fused into the
 * selector: unused), 1 = K2 selector (k_down, fused decimation), 2 = K3 stage, 3 = the merged fp64
 * fix-up of all levels, level 0) and level l (< 16), the summed milliseconds ms[kind * 16 + l] and
 * the launch count
 * count[kind * 16 + l] since the last read, then clears the records. Enabling profiling makes the
 * handle stateful: do not enqueue from several threads while it is on.
 */
blade_status blade_ms_set_profiling(blade_ms_t h, int32_t enable);
blade_status blade_ms_profile_read(blade_ms_t h, double* ms /* [64] */, int32_t* count /* [64] */);

/* Release the handle and its device bank. NULL is a no-op. */
blade_status blade_ms_destroy(blade_ms_t h);

const char* blade_ms_status_string(blade_status s);
/* Thread-local description of the last error on this thread ("" if none). */
const char* blade_ms_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* BLADE_MS_H */
