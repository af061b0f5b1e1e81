/*
 * fvv_b200.h -- C ABI of the B200-native dense view-synthesis path.
 *
 * This is the drop-in boundary for the reference's interpolation / tiling
 * path (reference = arxiv/paper_2112_10603, package `fvv`, pure Python).
 * The reference has no FFI of its own; each entry point below replaces one
 * Python function of its public API, with the same argument meaning and the
 * same error classes (mapped back to ValueError / LayoutError by the host
 * shim paper_2112_10603_b200/_lib.py):
 *
 *   fvv_validate_params        <- InterpConfig.__post_init__   interp.py:24-36
 *   fvv_interpolate_pairs      <- interpolate(left, right, cfg) interp.py:97-148 (batched)
 *   fvv_dense_views            <- dense_views(left, right, n)   interp.py:151-170
 *   fvv_rig_views              <- PipelineHandle._interp        server/pipeline.py:254-271
 *   fvv_downscale              <- downscale(frame, factor)      cluster.py:77-89 (batched)
 *   fvv_assemble_cluster       <- assemble_cluster_frame        cluster.py:143-191
 *   fvv_rig_clusters           <- PipelineHandle._stitch        server/pipeline.py:273-292
 *
 * Conventions
 *  - Frames are packed planes in the reference's Frame.raw_planes() order
 *    (frame.py:99-101): GRAY8 = Y (H,W); YUV420 = Y (H,W), U, V (H/2,W/2);
 *    RGB8 = interleaved (H,W,3).  Byte size: fvv_frame_bytes().
 *  - All frame pointers are DEVICE pointers (the caller -- torch -- owns
 *    every buffer); pointer arrays (`const uint8_t* const*`) are HOST arrays
 *    of device pointers.  Work is enqueued on the caller's stream; no call
 *    synchronises the device or allocates memory after fvv_engine_create.
 *  - Return value: FVV_OK (0) or a negative error class; the message is in
 *    fvv_last_error() (thread-local).  Entry points are reentrant per engine
 *    and keep no global mutable state besides that message.
 */
#ifndef FVV_B200_H
#define FVV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FVV_OK 0
#define FVV_EINVAL (-1)       /* ValueError in the reference               */
#define FVV_ELAYOUT (-2)      /* cluster.LayoutError in the reference      */
#define FVV_ECUDA (-3)        /* CUDA launch / runtime failure             */
#define FVV_EUNSUPPORTED (-4) /* valid for the reference, outside this path */

enum { FVV_GRAY8 = 0, FVV_YUV420 = 1, FVV_RGB8 = 2 }; /* frame.py:11-14 */

typedef struct {
    int32_t width;
    int32_t height;
    int32_t format; /* FVV_GRAY8 / FVV_YUV420 / FVV_RGB8 */
} fvv_frame_desc;

/* InterpConfig (interp.py:24-36); `refine` is a host-side hook, not here. */
typedef struct {
    int32_t block_size[3];    /* coarse -> fine, default (8, 8, 8)   */
    int32_t search_radius[3]; /* coarse -> fine, default (12, 4, 2)  */
    double mask_epsilon;      /* default 1e-3                        */
} fvv_interp_params;

typedef struct fvv_engine fvv_engine;

const char* fvv_last_error(void);
const char* fvv_build_info(void);

/* frame.py:22-30 plane_shapes -> total bytes of a packed frame */
size_t fvv_frame_bytes(const fvv_frame_desc* desc);

/* interp.py:32-36 validation (ValueError); mask_epsilon <= 0 is FVV_EUNSUPPORTED.
 * Every block size >= 2 and radius >= 1 the reference accepts is supported:
 * power-of-two blocks with max_span <= 120 run the exact fixed-point fast path
 * (DESIGN.md sec. 3), anything else the literal path (literal_kernels.cu, the
 * reference's f64/f32 arithmetic replayed one pair at a time; same results). */
int fvv_validate_params(const fvv_interp_params* params);

/* Engine = geometry + config + a caller-owned device workspace able to run
 * up to `max_pairs` interpolations per recursion stage. */
size_t fvv_engine_workspace_size(const fvv_frame_desc* desc, const fvv_interp_params* params,
                                 int max_pairs);
int fvv_engine_create(const fvv_frame_desc* desc, const fvv_interp_params* params, int max_pairs,
                      void* workspace, size_t workspace_bytes, fvv_engine** out);
void fvv_engine_destroy(fvv_engine* engine);
int fvv_engine_max_pairs(const fvv_engine* engine);

/* Launch-variant thresholds of an engine (no effect on results: every variant
 * is bit-exact; tests force each one).  value < 0 restores the default.
 *   FVV_TUNE_SCAN_COOP_MIN     cooperative-staging k_scan_carry from this many
 *                              one-warp CTAs per launch (default 600)
 *   FVV_TUNE_SADW_RB_MIN_CTAS  stacked-block k_sadw from this many CTAs
 *                              (default 296 = 2 per SM)
 *   FVV_TUNE_MASK_COLS2        gray / 4:2:0 mask producer: 1 = two-column
 *                              walker k_mask_cols2 (default), 0 = k_mask_cols
 *   FVV_TUNE_PDL               1 = launch the stage kernels with programmatic
 *                              dependent launch, 0 = plain launches (only in
 *                              a library built with -DFVV_PDL=1; off by default)
 * Not thread-safe against a concurrent call on the same engine. */
#define FVV_TUNE_SCAN_COOP_MIN 0
#define FVV_TUNE_SADW_RB_MIN_CTAS 1
#define FVV_TUNE_MASK_COLS2 2
#define FVV_TUNE_PDL 3
int fvv_engine_set_tuning(fvv_engine* engine, int key, int value);

/* interp.py:97-148, batched: out[i] = interpolate(left[i], right[i]).
 * npairs <= max_pairs.  Outputs may not alias inputs. */
int fvv_interpolate_pairs(fvv_engine* engine, const uint8_t* const* left,
                          const uint8_t* const* right, uint8_t* const* out, int npairs,
                          void* stream);

/* Optional diagnostics of the most recent fvv_interpolate_pairs call, pair i:
 * final full-resolution flows (H,W,2) f32 and the blend mask (H,W) f64, as
 * InterpDiagnostics.scales[-1].flow_lr / flow_rl and .mask (interp.py:49-64).
 * Device pointers; pass NULL to skip.  Must be enqueued on the same stream. */
int fvv_interp_diagnostics(fvv_engine* engine, int pair, float* flow_lr, float* flow_rl,
                           double* mask, void* stream);

/* Per-level diagnostics of pair i of the most recent batch, level 0 (1/4),
 * 1 (1/2) or 2 (full): the level's flows (h_s,w_s,2) f32 and match-error maps
 * (h_s,w_s) f64, as InterpDiagnostics.scales[level].flow_lr / flow_rl /
 * match_error_lr / match_error_rl (interp.py:49-56, 114-118).  NULL skips. */
int fvv_interp_level_diagnostics(fvv_engine* engine, int pair, int level, float* flow_lr,
                                 float* flow_rl, double* err_lr, double* err_rl, void* stream);

/* Coarse-scale diagnostics of pair i of the most recent batch (interp.py:119-127,
 * what interpolate(..., diagnostics=True) stores in scales[0..1]): the level's
 * blend mask (e_r + eps) / (e_l + e_r + 2 eps) and blend_luma, (h_s, w_s) f64,
 * replayed literally in f64 (off the hot path).  Needs a device scratch of
 * fvv_interp_level_mask_scratch(engine, level) bytes.  level 0 or 1. */
size_t fvv_interp_level_mask_scratch(const fvv_engine* engine, int level);
int fvv_interp_level_mask(fvv_engine* engine, int pair, int level, void* scratch, size_t scratch_bytes,
                          double* mask, double* blend_luma, void* stream);

/* Per-kernel timing of the stage kernels (bench.py's roofline figure):
 * while enabled, every stage-kernel launch is bracketed by a cudaEvent pair
 * on the launching stream (at most `capacity` launches are recorded).
 * fvv_profile_read synchronises on the recorded events, returns the summed
 * milliseconds and launch counts per kernel class and resets the record.
 * capacity <= 0 disables.  Not for use under CUDA-graph capture. */
#define FVV_NUM_KERNEL_CLASSES 11
int fvv_profile_enable(fvv_engine* engine, int capacity);
int fvv_profile_read(fvv_engine* engine, double* ms, int* launches, int nclasses);
const char* fvv_kernel_class_name(int kernel_class);

/* interp.py:151-170: views = (2^stages - 1) frames, contiguous, left -> right.
 * mode FVV_DENSE_RECURSIVE: the reference's recursive midpoints (bit-exact;
 *   requires max_pairs >= 2^(stages-1); no scratch).
 * mode FVV_DENSE_DIRECT: direct-t -- one interpolation of (left, right), whose
 *   output is the t = 1/2 view bit-exactly (interp.py:131-132), and every other
 *   view t = j / 2^stages from the same flows and mask in one fp32 synthesis
 *   pass (F_t->l = 2t F_m->l, F_t->r = 2(1-t) F_m->r, w_t = (1-t)M/((1-t)M +
 *   t(1-M))); the reference has no such mode, so there is no byte parity off
 *   t = 1/2.  Needs fvv_dense_views_scratch(engine, mode) bytes of device scratch. */
#define FVV_DENSE_RECURSIVE 0
#define FVV_DENSE_DIRECT 1
size_t fvv_dense_views_scratch(const fvv_engine* engine, int mode);
int fvv_dense_views(fvv_engine* engine, const uint8_t* left, const uint8_t* right, int stages, int mode,
                    uint8_t* views, void* scratch, size_t scratch_bytes, void* stream);

/* server/pipeline.py:254-271: one rig frame.  cams = ncams contiguous frames;
 * views = (ncams-1)*2^stages + 1 contiguous frames in global view order
 * (viewmodel.py:23-71: camera c at c*2^stages).  Requires
 * max_pairs >= (ncams-1)*2^(stages-1). */
int fvv_rig_views(fvv_engine* engine, const uint8_t* cams, int ncams, int stages, uint8_t* views,
                  void* stream);

/* fvv_rig_views with a dense-views mode: FVV_DENSE_RECURSIVE is fvv_rig_views;
 * FVV_DENSE_DIRECT interpolates every gap once (all gaps in one launch; the
 * t = 1/2 views are bit-exact) and synthesizes the other views of every gap
 * direct-t from those flows and masks (see fvv_dense_views).  Direct-t needs
 * max_pairs >= ncams - 1 and fvv_rig_views_scratch(engine, ncams, mode) bytes. */
size_t fvv_rig_views_scratch(const fvv_engine* engine, int ncams, int mode);
int fvv_rig_views_mode(fvv_engine* engine, const uint8_t* cams, int ncams, int stages, int mode, uint8_t* views,
                       void* scratch, size_t scratch_bytes, void* stream);

/* cluster.py:77-89, batched over nframes contiguous frames. */
int fvv_downscale(const fvv_frame_desc* desc, const uint8_t* frames, int nframes, int factor,
                  uint8_t* out, void* stream);

/* cluster.py:135-140 cluster_geometry: stitched width for nsmall quarter tiles */
int fvv_cluster_width(int base_width, int nsmall);

/* cluster.py:143-191: anchor (W,H) + nsmall quarter frames (W/4,H/4) ->
 * stitched frame (fvv_cluster_width(W, nsmall), H); GRAY8 / YUV420 only. */
int fvv_assemble_cluster(const fvv_frame_desc* anchor_desc, const uint8_t* anchor,
                         const uint8_t* const* smalls, int nsmall, uint8_t* stitched,
                         void* stream);

/* server/pipeline.py:273-292 + cluster.py:58-74: every cluster frame of one
 * rig frame straight from the global views buffer (downscale fused into the
 * paste).  clusters: ncams stitched frames packed back to back in camera
 * order; cluster c has fvv_rig_cluster_bytes(..., c) bytes. */
size_t fvv_rig_cluster_bytes(const fvv_frame_desc* desc, int ncams, int stages,
                             int views_per_side, int cluster);
int fvv_rig_clusters(const fvv_frame_desc* desc, int ncams, int stages, int views_per_side,
                     const uint8_t* views, uint8_t* clusters, void* stream);

/* The gap-sharded rig (SURVEY.md sec. 8(e) option 2; bench.py --shard gap):
 * clusters [first_cluster, first_cluster + ncluster) of the rig's cluster
 * frames, packed back to back, from a rank's LOCAL views (global indices
 * [view_base, view_base + nviews)) plus halo tiles -- quarter frames
 * (fvv_downscale factor 4) of global views [halo_first, halo_first +
 * halo_count) received from the neighbouring rank.  Cluster c reads views
 * of gaps c-1 and c (cluster.py:58-74), so the rank owning gap c needs the
 * top views_per_side views of gap c-1 as halo.  Byte-identical to the
 * matching clusters of fvv_rig_clusters.  FVV_EINVAL when a needed view is
 * neither local nor in the halo. */
int fvv_rig_clusters_shard(const fvv_frame_desc* desc, int ncams, int stages, int views_per_side,
                           int first_cluster, int ncluster, const uint8_t* views, int view_base,
                           int nviews, const uint8_t* halo, int halo_first, int halo_count,
                           uint8_t* clusters, void* stream);

/* ---------------------------------------------------------------------------
 * VINet (SURVEY.md sec. 8(b) "fvv_vinet_flow",
 * north star): the CNN flow / fusion estimator.  The reference ships no CNN
 * (SPEC.md:18), so its oracle is the fp32 torch module oracle/vinet_ref.py.
 *
 * fvv_conv2d_bf16: one convolution layer on the tcgen05 tensor cores
 * (implicit GEMM, TMA-fed, fp32 accumulation in TMEM, bias + ReLU epilogue).
 *   x    NHWC bf16 [batch][in_h][in_w][in_cpad], in_cpad in {16, 32} or a
 *        multiple of 64 (padding channels zero);
 *   w    bf16, K-major.  Convolution: [npad][k*k*in_cpad] with
 *        K index = (ky*k + kx)*in_cpad + c.  Transposed (k4 s2 p1):
 *        [4 phases][npad][4*in_cpad], phase = (oy&1)*2 + (ox&1), tap
 *        t = ty*2 + tx with input offsets dy = (oy&1) ? {+1, 0} : {0, -1}
 *        (kernel rows ky = (oy&1) ? {0, 2} : {1, 3}), likewise in x;
 *        npad = out_channels rounded up to ntile;
 *   bias fp32 [out_channels];
 *   out  NHWC [batch][out_h][out_w][out_cstride] (bf16, or fp32 when
 *        out_f32), channels [out_coff, out_coff + out_channels).
 * -------------------------------------------------------------------------- */
typedef struct fvv_conv_desc {
    int32_t batch, in_h, in_w, in_cpad;
    int32_t out_h, out_w, out_cstride, out_coff, out_channels;
    int32_t kernel, stride, pad;   /* square kernel; transposed: 4, 2, 1 */
    int32_t transposed;            /* 1: ConvTranspose2d (4 phase GEMMs); 2: the same as one
                                      3x3 sub-pixel GEMM, weights [npad(4 out)][9*in_cpad]
                                      (row = phase*out_channels + c), bias 4*out_channels */
    int32_t relu, out_f32;
    int32_t ntile;                 /* UMMA N tile: 16, 32, 64, 128 or 256 */
} fvv_conv_desc;
int fvv_conv2d_bf16(const fvv_conv_desc* desc, const void* x, const void* w, const float* bias,
                    void* out, void* stream);

/* VINet forward, batched over camera pairs.  Weights: 3 blocks x 10 layers
 * (c0, c1, r1..r6, u0, u1; paper_2112_10603_b200/vinet_params.py), each packed
 * as documented for fvv_conv2d_bf16 with ntile 128 (c0, u0), 256 (c1, r*)
 * and in_cpad 16 / 32 for block 0 / blocks 1-2 c0.  u1 (ConvTranspose2d
 * 128->5) runs as one 3x3 sub-pixel convolution: weights [32][9*128] with row
 * n = phase*5 + c (phase = (oy&1)*2 + (ox&1)) and tap (ty, tx) reading input
 * offset (ty-1, tx-1) (convtc.pack_convT_subpixel); its bias has 20 entries
 * (the 5 biases once per phase).
 * flows: [npairs][5][H][W] fp32 = F_m->l (x, y), F_m->r (x, y), mask logit.
 * The workspace holds fvv_vinet_workspace_size(desc, max_pairs) bytes; larger
 * batches run in chunks of max_pairs. */
typedef struct fvv_vinet_weights {
    const void* w[3][10];
    const float* b[3][10];
} fvv_vinet_weights;
size_t fvv_vinet_workspace_size(const fvv_frame_desc* desc, int max_pairs);
int fvv_vinet_flow(const fvv_frame_desc* desc, const fvv_vinet_weights* weights, const uint8_t* const* left,
                   const uint8_t* const* right, int npairs, float* flows, void* workspace,
                   size_t workspace_bytes, void* stream);
/* Direct-t synthesis: for every pair the nviews views at t = j/(nviews+1),
 * j = 1..nviews, from one flow field in one pass (warp both frames, sigmoid-
 * mask blend, rint/clip).  views: [npairs][nviews][frame_bytes]. */
int fvv_vinet_synth(const fvv_frame_desc* desc, const uint8_t* const* left, const uint8_t* const* right,
                    const float* flows, int npairs, int nviews, uint8_t* views, void* stream);

/* The rig with VINet: ncams cameras (contiguous frames) -> the global views
 * buffer of fvv_rig_views (anchor c at index c*2^stages, the 2^stages-1
 * direct-t views of gap c after it), ready for fvv_rig_clusters. */
int fvv_vinet_rig(const fvv_frame_desc* desc, const fvv_vinet_weights* weights, const uint8_t* cams, int ncams,
                  int stages, uint8_t* views, void* workspace, size_t workspace_bytes, void* stream);

/* fvv_vinet_rig followed by fvv_rig_clusters in one call, with the cluster
 * tiling fused into the synthesis epilogue: each direct-t view's 4x4 box-mean
 * quarter tiles are written into the cluster frames straight from the
 * synthesis kernel (no re-read of the views); a reduced cluster pass adds the
 * anchors and padding.  `views` and `clusters` are byte-identical to the
 * two-call path (PipelineHandle.process_frame + _stitch, server/pipeline.py:
 * 199-292).  At most 8192 global views per rig frame. */
int fvv_vinet_rig_clusters(const fvv_frame_desc* desc, const fvv_vinet_weights* weights, const uint8_t* cams,
                           int ncams, int stages, int views_per_side, uint8_t* views, uint8_t* clusters,
                           void* workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * RefineNet + ContextNet (vinet_params.py), the
 * paper's context-aware residual U-Net after the VIBlocks.  The convolutions
 * run through fvv_conv2d_bf16; these entry points are its other kernels
 * (orchestration: paper_2112_10603_b200/refine.py; fp32 oracle:
 * oracle/vinet_ref.py refine_view).  The network works on the 64-aligned
 * canvas (Wp, Hp) of the frame, edge-replicated.
 *
 * fvv_refine_image     context-net input: canvas images of nsrc frames,
 *                      NHWC bf16 [nsrc][Hp][Wp][16] (3 channels used)
 * fvv_refine_inputs    per view i (t[i] in (0,1), state[i] = VINet flows
 *                      (5,H,W)): U-Net input x0 NHWC bf16 [n][Hp][Wp][32]
 *                      (17 used), merged blend (n,3,H,W) f32, canvas flows
 *                      flow0 (n,4,Hp,Wp) f32 = (F_l,t, F_r,t)
 * fvv_refine_flow_pool next context level's flows: 2x2 mean * 0.5
 * fvv_refine_warp_features  warp channels [0,C) of NHWC bf16 features of
 *                      source (b*src_mul + src_add) with flow channels
 *                      (comp, comp+1) into dst channels [coff, coff+C)
 * fvv_nhwc_copy        U-Net skip: channels [0,C) of src -> dst at coff
 * fvv_refine_output    views = clip(merged + 2 sigmoid(r) - 1, 0, 1) packed
 *                      as uint8 frames (r: NHWC f32 [n][Hp][Wp][rs])
 * At most 64 views (128 sources) per call. */
int fvv_refine_image(const fvv_frame_desc* desc, const uint8_t* const* frames, int nsrc, void* out, void* stream);
int fvv_refine_inputs(const fvv_frame_desc* desc, const uint8_t* const* left, const uint8_t* const* right,
                      const float* const* state, const float* t, int nviews, void* x0, float* merged, float* flow0,
                      void* stream);
int fvv_refine_flow_pool(const float* in, float* out, int w, int h, int nb, void* stream);
int fvv_refine_warp_features(const void* feat, int fs, int channels, int w, int h, const float* flow, int comp,
                             int src_mul, int src_add, void* dst, int ds, int coff, int nb, void* stream);
int fvv_nhwc_copy(const void* src, int ss, int channels, void* dst, int ds, int coff, long long npix, void* stream);
int fvv_refine_output(const fvv_frame_desc* desc, uint8_t* const* out, int nviews, const float* r, int rs,
                      const float* merged, void* stream);

/* ---------------------------------------------------------------------------
 * FVT1 tile encoder, device stage (the hand-off
 * after the tiling; codec.py:138-216 _encode_plane / encode_frame, dct.py).
 * Per (tile, plane) job: edge-padded 8x8 blocks of the plane (minus the
 * previous reconstruction for P records), orthonormal DCT, rint(c / step)
 * (or the lossless lifting transform at quality 100), the committed
 * reconstruction into `recon`, zigzag coefficients (int16, 64 per block) and
 * the block's token count (nonzeros + EOB).  fvv_encode_tokens writes the
 * 3-byte (run, level) token stream at tok_off[block] * 3; the caller DEFLATEs
 * each plane's tokens and frames the record (paper_2112_10603_b200/encoder.py).
 * fvv_encode_set_tables uploads the reference's DCT matrix and zigzag order. */
typedef struct {
    const uint8_t* src;    /* tile plane inside the stitched frame (device)      */
    const uint8_t* prev;   /* previous reconstruction (w x h), NULL for I        */
    uint8_t* recon;        /* committed reconstruction (w x h) out               */
    long long block0;      /* first 8x8 block of the job in the batch (ascending) */
    int32_t pitch, w, h;   /* row pitch of src, plane size (RGB: 3 * width)      */
    int32_t nbx, nby;      /* ceil(w / 8), ceil(h / 8)                           */
    int32_t is_p, step, pad;
} fvv_enc_job;
int fvv_encode_set_tables(const double* dct64, const uint8_t* zigzag64);
int fvv_encode_blocks(const fvv_enc_job* jobs_dev, int njobs, long long total_blocks, int lossless, int16_t* zz,
                      int* ntok, void* stream);
int fvv_encode_tokens(const int16_t* zz, const long long* tok_off, long long nblocks, uint8_t* out, void* stream);

/* DEFLATE of many independent byte streams on the device, byte-identical to
 * zlib.compress(stream, 6)[2:-4] -- the raw DEFLATE data of each plane's token
 * stream that codec.py:148 (_encode_plane) keeps.  zlib 1.3's level-6
 * deflate_slow / trees.c decisions restated in csrc/zdeflate_core.h.
 * offsets (host, nstreams + 1, ascending): stream s = data[offsets[s],
 * offsets[s+1]) (data on the device).  out (device, 8-byte aligned, at least
 * *out_capacity bytes) receives the compressed streams back to back;
 * out_offsets (device, nstreams + 1) their offsets (out_offsets[0] = 0).
 * Stream-ordered; the offsets are read on the host during the call. */
int fvv_deflate_scratch_bytes(const long long* offsets, int nstreams, size_t* scratch_bytes, size_t* out_capacity);
int fvv_deflate(const uint8_t* data, const long long* offsets, int nstreams, uint8_t* out, long long* out_offsets,
                void* scratch, size_t scratch_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * TS packaging (host code; mpegts.py:188-212
 * mux_segment): one cluster's MPEG-TS segment from the tile records of its
 * frames.  records[f * ntiles + k] / record_lens[...] are HOST pointers; pts[f]
 * the frame's 90 kHz PTS.  0 ok, -1 bad arguments / short buffer, -2 frame 0
 * is not intra on every tile.  Thread-safe (no shared state). */
size_t fvv_ts_segment_bytes(const uint32_t* record_lens, int ntiles, int nframes);
int fvv_ts_mux_segment(const uint8_t* const* records, const uint32_t* record_lens, int ntiles, int nframes,
                       const int64_t* pts, uint8_t* out, size_t out_cap, size_t* written);

#ifdef __cplusplus
}
#endif
#endif /* FVV_B200_H */
