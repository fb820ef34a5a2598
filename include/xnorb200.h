/*
 * xnorb200.h -- C-ABI of libxnorb200.so, the B200 (sm_100a) XNOR-conv forward path.
 *
 * Conventions (mirroring the reference kernel seam, _backend.py:28-41 and
 * _kernels_py.py:3-4): the CALLER allocates every output and passes it in;
 * functions fill in place.  Every pointer is a DEVICE pointer (cudaMalloc /
 * torch CUDA storage) unless stated otherwise; `stream` is a cudaStream_t
 * (NULL = legacy default stream).  Calls only enqueue work: no allocation, no
 * synchronisation, no host<->device copies.  The only library state is a cache,
 * keyed by (device, kernel) and guarded by a mutex, of the dynamic shared-memory
 * opt-in and each device's SM count: calls are thread-safe and may target any
 * device (the current one at call time).  Return value: 0 (XNC_OK) or an
 * XNC_E* code below / a cudaError_t launch error (>= 1000 + cudaError_t).
 * Shape validation lives in the Python layer (which raises the reference's
 * exception types); the C layer re-checks cheaply and returns XNC_EINVAL.
 *
 * Data layouts in HBM (the B200 build's choice):
 *   x      f32  [N][C][H][W]            activations (NCHW, as the reference's
 *                                        (C,H,W) Tensor3 per image)
 *   bits   u32  [N][H][W][Cw]           channel-packed signs, Cw = ceil(C/32);
 *                                        bit (c % 32) of word c/32 = (x >= 0),
 *                                        tail bits (c >= C) are 0
 *   A      f32  [N][H][W]               channel mean |x|, sequential f32 order
 *   K      f32  [N][H'][W']             box-filtered A (the K map)
 *   wbits  u32  [Cw][kh][kw][O]         packed filter signs, filters contiguous
 *   alpha  f32  [O]                     (float)(sum |w| f64 sequential / n)
 *   y      f32  [N][O][H'][W']          output; y[n][o] == xnor_conv(x[n], w[o])
 *   acc    i32  [N][O][H'][W']          optional integer XNOR sums (or NULL)
 *   H' = H + 2*pad - kh + 1, W' = W + 2*pad - kw + 1; 1 <= kh, kw <= 8.
 */
#ifndef XNORB200_H
#define XNORB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define XNC_DTYPE_F32 0
#define XNC_DTYPE_F64 1
#define XNC_DTYPE_I8 2

#define XNC_OK 0
#define XNC_EINVAL 1      /* bad shape / argument */
#define XNC_ENOTSUP 2     /* shape outside what the kernels support */
#define XNC_ECUDA_BASE 1000

/* Version of the ABI (bumped on any signature change). */
int xnc_abi_version(void);
/* Static string for an error code. */
const char* xnc_strerror(int code);

/* ---- K1: fused sign + channel bit-pack + channel-mean |x| ------------------
 * Replaces the float->bit half of pack_plane (_kernels_cy.pyx:42-73, per
 * channel, per filter) and the channel abs-mean of scale_rows/_window_row
 * (_kernels_cy.pyx:151-186, :207-230): one pass over x per image instead of
 * one per (image, filter).  A may be NULL. */
int xnc_pack_input(const float* x, int N, int C, int H, int W,
                   uint32_t* bits, float* A, void* stream);

/* ---- filter binarization (build_filter, engine.py:102-120 + sign_binarize,
 * binarize.py:65-75): signs -> wbits, alpha in float64 sequential order.
 * w: f32 [O][C][kh][kw]; alpha64 (optional, may be NULL) receives the float64
 * alpha the reference keeps in BinaryFilter.scale. */
int xnc_pack_weights(const float* w, int O, int C, int kh, int kw,
                     uint32_t* wbits, float* alpha, double* alpha64, void* stream);

/* Same, from float64 weights (the reference's Tensor3 values, unrounded). */
int xnc_pack_weights_f64(const double* w, int O, int C, int kh, int kw,
                         uint32_t* wbits, float* alpha, double* alpha64, void* stream);

/* ---- K2: K map = box filter of A with zero padding ----------------------------
 * Float32 op order of xnor_reconstruct's ring/map rows (_kernels_cy.pyx:231-239,
 * :299-311): row sums left->right, column sums top->bottom, * f32(1/(kh*kw)). */
int xnc_scale_map(const float* A, int N, int H, int W, int kh, int kw, int pad,
                  float* K, void* stream);

/* ---- K3+K4: XNOR-popcount implicit-GEMM conv with the alpha*K epilogue -------
 * Replaces xnor_accumulate (_kernels_cy.pyx:76-104) + scale_join (:189-204)
 * and the decode loop of xnor_reconstruct (:335-349), for all (n, o) at once.
 * acc may be NULL; y may be NULL when only acc is wanted. */
int xnc_xnor_conv(const uint32_t* bits, const uint32_t* wbits, const float* K,
                  const float* alpha, int N, int C, int H, int W, int O,
                  int kh, int kw, int pad, float* y, int32_t* acc, void* stream);

/* Variant selector for xnc_xnor_conv (benchmarking the north star's
 * popc vs. b1 mma.sync comparison).  0 = popc (default). */
#define XNC_CONV_POPC 0
#define XNC_CONV_B1MMA 1
int xnc_xnor_conv_variant(int variant, const uint32_t* bits, const uint32_t* wbits,
                          const float* K, const float* alpha, int N, int C, int H,
                          int W, int O, int kh, int kw, int pad, float* y,
                          int32_t* acc, void* stream);

/* ---- K3 on the tcgen05 tensor cores (kind::i8, TMEM accumulators, CTA pairs) --
 * The XNOR sum as an exact u8 x s8 GEMM: acc = S_w[o] - 2 * sum_taps d * s_w, with
 * d = 1 for a negative input sign and s_w = +-1 the filter sign.
 * Input: the same packed bits as xnc_xnor_conv (u32 [N][H][W][Cw], from
 * xnc_pack_input); the kernel expands them to its byte operand in shared memory.
 * Weights in the tensor-core layout: wq (xnc_umma_weight_bytes bytes, s8 signs
 * in 128-byte rows) and sw i32 [O] (sum of each filter's signs), produced by
 * xnc_pack_weights_umma from f32 (dtype 0) or f64 (dtype 1) weights.
 * xnc_umma_supported() == 0 means the shape does not fit the kernel's shared
 * memory plan (then use xnc_xnor_conv). */
size_t xnc_umma_weight_bytes(int O, int C, int kh, int kw);
int xnc_umma_supported(int N, int C, int H, int W, int O, int kh, int kw, int pad);
int xnc_pack_weights_umma(const void* w, int dtype, int O, int C, int kh, int kw,
                          uint8_t* wq, int32_t* sw, void* stream);
/* Optional per-channel affines (a bias or a folded batch norm, y' = (y * scale) +
 * shift with one rounding per op): on the input of K1 before the sign and |.|
 * (scale/shift f32 [C]), or on the output of the tcgen05 conv after alpha*K
 * (f32 [O]; "optional bias/BN for the next binary layer").  Both NULL = none. */
int xnc_pack_input_affine(const float* x, int N, int C, int H, int W, const float* in_scale,
                          const float* in_shift, uint32_t* bits, float* A, void* stream);
int xnc_xnor_conv_umma_affine(const uint32_t* bits, const uint8_t* wq, const int32_t* sw,
                              const float* K, const float* alpha, int N, int C, int H, int W,
                              int O, int kh, int kw, int pad, const float* out_scale,
                              const float* out_shift, float* y, int32_t* acc, void* stream);
/* ---- network data movement (XNOR-Net AlexNet forward, network.py) ----------
 * Max-pool in front of a binary layer (XNOR-Net: pool -> BN -> sign): out f32
 * [N][C][H][W] = max over pool_k x pool_k windows (stride pool_s, no padding) of
 * x [N][C][Hin][Win], H = (Hin - pool_k) / pool_s + 1; the values of
 * torch.max_pool2d (NaN propagates).  bias f32 [C] (or NULL): pool of (x + bias),
 * added after the max (max(v + b) == max(v) + b exactly: a conv's bias folded into
 * the pool); relu != 0: torch.relu before the pool, in the same pass.  pool_k <= 8. */
int xnc_max_pool(const float* x, int N, int C, int Hin, int Win, int pool_k, int pool_s, int relu,
                 int nhwc, const float* bias, float* out, void* stream);
/* y f32 [N][O][plane] in place: y[n][o][i] = y[n][o][i] * scale[o] + shift[o], one
 * rounding per op (the fused tcgen05 epilogue's out_affine, for the popc / b1mma
 * kernels, whose epilogues do not carry it). */
int xnc_plane_affine(float* y, int N, int O, long plane, const float* scale, const float* shift,
                     void* stream);
/* F.pixel_unshuffle(F.pad(x, pad on all sides), r) in one pass: out f32
 * [N][C*r*r][(H+2pad)/r][(W+2pad)/r] (conv1 11x11/4 as a 3x3 conv, network.py).
 * nhwc != 0 (xnc_max_pool too): the map is stored channels-last, [N][H][W][C]. */
int xnc_pad_space_to_depth(const float* x, int N, int C, int H, int W, int pad, int r, int nhwc,
                           float* out, void* stream);
/* K1 of max_pool(x) without materialising it: x f32 [N][C][Hin][Win] is the
 * PRE-pool map; bits / A describe the pooled map [N][Ho][Wo] (Ho = (Hin - pool_k) /
 * pool_s + 1), bit-identical to xnc_max_pool followed by xnc_pack_input_affine
 * (in_scale / in_shift may be NULL).  Returns XNC_ENOTSUP for shapes the fused
 * kernel does not take (pool_k != 3; unless pool_s == 2 and Win <= 32, also
 * fewer than 32 pooled pixels per image or C outside 32..768): pool, then pack. */
int xnc_pack_input_pool(const float* x, int N, int C, int Hin, int Win, int pool_k, int pool_s,
                        const float* in_scale, const float* in_shift, uint32_t* bits, float* A, void* stream);
/* The channels-last form with the pool's bias and ReLU: bits / A of
 * xnc_max_pool(x, pool_k, pool_s, relu, bias, nhwc = 1) followed by
 * xnc_pack_input_nhwc(in_scale, in_shift), bit-identical, the pooled map never
 * written (the XNOR-Net front end: conv1 -> bias -> ReLU -> pool -> conv2's BN ->
 * sign; reference xnor_conv pipeline.py:176-201 takes one image's binarized input,
 * this is that input's K1 for a whole batch).  x f32 [N][Hin][Win][C], 16-byte
 * aligned; bias may be NULL.  XNC_ENOTSUP unless pool_k == 3 and C % 32 == 0, C <=
 * 256: pool, then pack. */
int xnc_pack_input_pool_nhwc(const float* x, int N, int C, int Hin, int Win, int pool_k, int pool_s, int relu,
                             const float* bias, const float* in_scale, const float* in_shift, uint32_t* bits,
                             float* A, void* stream);
/* K1 (xnc_pack_input_affine) for a channels-last input x f32 [N][H][W][C]: same
 * bits / A, a thread per pixel walking its contiguous channels. */
int xnc_pack_input_nhwc(const float* x, int N, int C, int H, int W, const float* in_scale,
                        const float* in_shift, uint32_t* bits, float* A, void* stream);
/* Binary -> binary: the conv epilogue writes the NEXT binary layer's K1 output
 * instead of y (north star item 4, "sign for the next binary layer"): with
 * y' = ((f32(acc) * K) * alpha) [* out_scale + out_shift], next_bits u32
 * [N][H'][W'][ceil(O/32)] = sign words of y' (bit c = y'_c >= 0, tail bits 0) and
 * next_A f32 [N][H'][W'] = (sequential f32 sum over c of |y'_c|) * f32(1/O) (NULL
 * = not written), bit-identical to xnc_pack_input_affine run on the materialised
 * y'.  The 822 MB float map of a C3 layer is never written nor re-read.  Any O the
 * tcgen05 plan supports: with several filter blocks (O > 256) each CTA pair takes
 * whole pixel tiles and runs their blocks back to back (tile-major), so a pixel's
 * channels reach one thread in order; xnc_umma_emit_supported() says whether the
 * shape's plan fits. */
int xnc_umma_emit_supported(int N, int C, int H, int W, int O, int kh, int kw, int pad);
int xnc_xnor_conv_umma_emit(const uint32_t* bits, const uint8_t* wq, const int32_t* sw,
                            const float* K, const float* alpha, int N, int C, int H, int W,
                            int O, int kh, int kw, int pad, const float* out_scale,
                            const float* out_shift, uint32_t* next_bits, float* next_A,
                            void* stream);
/* K split for shapes with fewer (pixel tile, 256-filter block) work units than CTA
 * pairs -- fully connected layers viewed as one 1 x N image.  Units of one output
 * tile take disjoint K ranges and store their raw partial sums into their own
 * slice of split_ws (s32, xnc_umma_split_ws_bytes() bytes = S slices of N*O*H'*W';
 * any contents on entry -- every slice entry is written); a finalize kernel then
 * adds the slices and writes y / acc with the same arithmetic as the unsplit
 * epilogue (integer sums: exact in any order).  xnc_umma_split_ws_bytes()
 * == 0: no split for this shape, split_ws is ignored (may be NULL).  Otherwise
 * the same contract as xnc_xnor_conv_umma_affine (which never splits). */
size_t xnc_umma_split_ws_bytes(int N, int C, int H, int W, int O, int kh, int kw, int pad);
int xnc_xnor_conv_umma_ws(const uint32_t* bits, const uint8_t* wq, const int32_t* sw,
                          const float* K, const float* alpha, int N, int C, int H, int W,
                          int O, int kh, int kw, int pad, const float* out_scale,
                          const float* out_shift, int32_t* split_ws, float* y, int32_t* acc,
                          void* stream);
/* xnc_xnor_conv_umma_ws with y written CHANNELS-LAST, f32 [N][H'][W'][O] (the
 * epilogue's 16 filters of a pixel are 64 contiguous bytes; the K-split finalize
 * transposes through shared memory).  A fully connected layer (network.py's fc6 /
 * fc7: the batch as one 1 x P image, kernel 1 x 1) gets its [batch][filters]
 * output without a transpose pass; a conv gets an NHWC map for the channels-last
 * pool + K1 that follow it.  Float output only; O % 4 == 0, y 16-byte aligned. */
int xnc_xnor_conv_umma_nhwc(const uint32_t* bits, const uint8_t* wq, const int32_t* sw, const float* K,
                            const float* alpha, int N, int C, int H, int W, int O, int kh, int kw, int pad,
                            const float* out_scale, const float* out_shift, int32_t* split_ws, float* y,
                            void* stream);
/* xnc_xnor_conv_umma_nhwc followed by the NEXT binary layer's K1 of y: next_bits
 * [pixels][O/32] and next_A [pixels] = xnc_pack_input of y viewed as pixels 1 x 1 maps
 * of O channels (the fc6 -> fc7 hand-off of the XNOR-Net forward; reference: the next
 * layer's xnor_conv input binarization, pipeline.py:176-201), bit-identical.  With a
 * K split the finalize builds them in the same pass (one block per pixel runs the
 * sequential |.| chain); unsplit, K1 runs on y after the conv.  y is still written.
 * O % 32 == 0, O <= 4096, y 16-byte aligned. */
int xnc_xnor_conv_umma_nhwc_emit(const uint32_t* bits, const uint8_t* wq, const int32_t* sw, const float* K,
                                 const float* alpha, int N, int C, int H, int W, int O, int kh, int kw, int pad,
                                 const float* out_scale, const float* out_shift, int32_t* split_ws, float* y,
                                 uint32_t* next_bits, float* next_A, void* stream);
/* Profiling only: per-CTA cycle counters of the last tcgen05 conv launched with
 * XNC_UMMA_DEBUG bit 7 set (16 u64 slots per CTA, host memory; blocking copy). */
int xnc_umma_profile(unsigned long long* host_out, int n_ctas);
int xnc_xnor_conv_umma(const uint32_t* bits, const uint8_t* wq, const int32_t* sw,
                       const float* K, const float* alpha, int N, int C, int H, int W,
                       int O, int kh, int kw, int pad, float* y, int32_t* acc, void* stream);

/* ---- whole layer: K1 -> K2 -> K3+K4 on one stream ------------------------------
 * The batched equivalent of ConvWorkspace.run() (pipeline.py:124-151) over
 * every (image, filter) pair.  workspace: device scratch of at least
 * xnc_layer_workspace_bytes(...) bytes (holds bits, A, K). */
size_t xnc_layer_workspace_bytes(int N, int C, int H, int W, int kh, int kw, int pad);
int xnc_layer_forward(const float* x, const uint32_t* wbits, const float* alpha,
                      int N, int C, int H, int W, int O, int kh, int kw, int pad,
                      void* workspace, float* y, int32_t* acc, void* stream);
/* The same layer on the tcgen05 pair kernel (weights from xnc_pack_weights_umma;
 * alpha from xnc_pack_weights).  XNC_ENOTSUP when xnc_umma_supported() is 0. */
int xnc_layer_forward_umma(const float* x, const uint8_t* wq, const int32_t* sw,
                           const float* alpha, int N, int C, int H, int W, int O, int kh,
                           int kw, int pad, void* workspace, float* y, int32_t* acc,
                           void* stream);

/* ======================================================================
 * The reference kernel seam on the device (interop surface).
 * One entry point per function of the module returned by the reference's
 * _backend.get_kernels() (_backend.py:28-41), same argument meaning, same
 * reference TILE-WORD layout (PackedTileGrid, pack.py:1-20) and float order;
 * plus the float64 module-level operators of the reference's Python API.
 * Device pointers; caller allocates outputs; enqueue only (except
 * xnc_xnor_reconstruct, which takes stream-ordered scratch with
 * cudaMallocAsync, as the reference mallocs per band, _kernels_cy.pyx:285).
 * ====================================================================== */
/* pack_plane (_kernels_cy.pyx:42-73): plane [h][w] of f32/f64/int8 -> tile
 * words [tiles_y][tiles_x], bit r*tile_w+c = (plane[ty*sy+r][tx*sx+c] >= 0). */
int xnc_pack_plane(const void* plane, int dtype, int h, int w, int tiles_y, int tiles_x,
                   int tile_h, int tile_w, int stride_y, int stride_x, uint64_t* out_words,
                   void* stream);
/* unpack (pack.py:123-154): tile words -> +-1 plane over the whole covered
 * region [cov_h][cov_w]; *mismatch |= 1 when overlapping tiles disagree. */
int xnc_unpack_plane(const uint64_t* words, int tiles_y, int tiles_x, int tile_h, int tile_w,
                     int stride_y, int stride_x, int8_t* plane_cov, int* mismatch, void* stream);
/* sign_plane / _signs_of (binarize.py:56-60): float64 -> int8 +-1, sign(0) = +1. */
int xnc_sign_plane(const double* x, long n, int8_t* out, void* stream);
/* xnor_accumulate (_kernels_cy.pyx:76-104): words [C][tiles_y][tiles_x]. */
int xnc_xnor_accumulate(const uint64_t* words, int channels, int tiles_y, int tiles_x,
                        const uint64_t* weight_words, uint64_t mask, int tile_w, int stride_y,
                        int stride_x, int k_area, int32_t* out, int out_h, int out_w,
                        void* stream);
/* build_filter (engine.py:102-120) for O filters: w f64 [O][C][kh][kw] ->
 * tile-layout words [O][C] and float64 alpha [O]. */
int xnc_filter_words(const double* w, int O, int C, int kh, int kw, int tile_w, uint64_t* words,
                     double* alpha, void* stream);
/* box_mean (_kernels_cy.pyx:126-148), f32 or f64: a [h][w] -> tmp [h][w-kw+1],
 * out [h-kh+1][w-kw+1]. */
int xnc_box_mean(const void* a, int dtype, int h, int w, int kh, int kw, double scale, void* tmp,
                 void* out, void* stream);
/* scale_rows (_kernels_cy.pyx:151-186): padded [C][h][w] -> tmp [h][w-kw+1]. */
int xnc_scale_rows(const void* padded, int dtype, int channels, int h, int w, int kw, void* tmp,
                   void* stream);
/* scale_join (_kernels_cy.pyx:189-204): tmp [out_h+kh-1][out_w], ints [out_h][out_w]. */
int xnc_scale_join(const void* tmp, int dtype, const int32_t* ints, int kh, double scale,
                   double weight_scale, int out_h, int out_w, void* out, void* stream);
/* xnor_reconstruct (_kernels_cy.pyx:242-354): one (padded image, filter) pair,
 * padded [C][ph][pw] f32/f64 -> out [ph-kh+1][pw-kw+1]; race-free. */
int xnc_xnor_reconstruct(const uint64_t* weight_words, uint64_t mask, int tile_h, int tile_w,
                         int stride_y, int stride_x, int k_area, const void* padded, int dtype,
                         int channels, int ph, int pw, int kh, int kw, double scale,
                         double weight_scale, void* out, void* stream);
/* channel_abs_mean (tensor.py:103-105): x f64 [C][H][W] -> A f64 [H][W]. */
int xnc_channel_abs_mean_f64(const double* x, int C, int H, int W, double* A, void* stream);
/* apply_scaling (scaling.py:91-98): out = ints * K * alpha, float64. */
int xnc_apply_scaling_f64(const int32_t* ints, const double* K, double alpha, long n, double* out,
                          void* stream);

/* ---- XNOR-Net AlexNet conv1 on the tensor cores (network.py front end) -----
 * The network's full-precision first layer (11x11, stride 4, pad 2, 3 -> 96,
 * 224 x 224 -> 55 x 55) as one tcgen05 kind::tf32 kernel on CTA pairs, reading the
 * raw images (no space-to-depth pass).  Operands are rounded to TF32 (cvt.rna, as
 * cuDNN's TF32 mode), products accumulate in f32.  Not on the binary path.
 * xnc_conv1_pack_weights: w f32 [96][3][11][11] -> wq f32, xnc_conv1_weight_bytes()
 * bytes (27 (c, tap) blocks x 96 filters x 16 phases, TF32-rounded).
 * xnc_conv1_forward: x f32 [N][3][224][224] (8-byte aligned) -> y f32
 * [N][55][55][96] channels-last (16-byte aligned), the raw conv (no bias: the
 * caller's xnc_max_pool adds it with the ReLU). */
size_t xnc_conv1_weight_bytes(void);
int xnc_conv1_pack_weights(const float* w, float* wq, void* stream);
int xnc_conv1_forward(const float* x, int N, const float* wq, float* y, void* stream);

/* ---- the reference's naive truth (reference.py) and vanilla_conv ---------
 * Not on the hot path: the checkers of paper_2007_14178_b200.verify (the
 * reference's verify.py:42-145 gates) and the float baseline of its bench
 * (bench.py:196-256).  One thread per output, the reference's (ch, ky, kx)
 * order, one rounding per operation (no FMA).  Independent of the packed engine.
 * sign_conv2d_int (reference.py:57-90): signs / wsigns int8 +-1 [C][h][w] /
 * [C][kh][kw], taps outside the plane count +1 -> out i32 [h+2p-kh+1][w+2p-kw+1]. */
int xnc_ref_sign_conv2d(const int8_t* signs, const int8_t* wsigns, int C, int h, int w, int kh, int kw,
                        int pad, int32_t* out, void* stream);
/* conv2d_float (reference.py:30-54), bwn == 0: f64 cross-correlation with zero
 * padding.  bwn_conv (reference.py:93-122), bwn != 0: +-x by sign(w > 0), then
 * * scale.  x [C][h][w], w [C][kh][kw] f64 -> out f64 [h+2p-kh+1][w+2p-kw+1]. */
int xnc_ref_conv2d_f64(const double* x, const double* wt, int C, int h, int w, int kh, int kw, int pad,
                       int bwn, double scale, double* out, void* stream);
/* vanilla_conv (_kernels_cy.pyx:107-123): padded [C][ph][pw] against weights
 * [C][kh][kw], both f32 (dtype 0) or f64 (dtype 1) -> out [ph-kh+1][pw-kw+1]. */
int xnc_vanilla_conv(const void* padded, int dtype, int C, int ph, int pw, const void* weights, int kh,
                     int kw, void* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* XNORB200_H */
