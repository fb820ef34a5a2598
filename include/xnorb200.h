/*
 * xnorb200.h -- C-ABI of libxnorb200.so, the B200 (sm_100a) XNOR-conv forward path.
 *
 * Conventions (mirroring the reference kernel seam, _backend.py:28-41 and
 * _kernels_py.py:3-4): the CALLER allocates every output and passes it in;
 * functions fill in place.  Every pointer is a DEVICE pointer (cudaMalloc /
 * torch CUDA storage) unless stated otherwise; `stream` is a cudaStream_t
 * (NULL = legacy default stream).  Calls only enqueue work: no allocation, no
 * synchronisation, no host<->device copies, no global mutable state beyond a
 * one-time per-kernel shared-memory opt-in.  Return value: 0 (XNC_OK) or an
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

/* ---- whole layer: K1 -> K2 -> K3+K4 on one stream ------------------------------
 * The batched equivalent of ConvWorkspace.run() (pipeline.py:124-151) over
 * every (image, filter) pair.  workspace: device scratch of at least
 * xnc_layer_workspace_bytes(...) bytes (holds bits, A, K). */
size_t xnc_layer_workspace_bytes(int N, int C, int H, int W, int kh, int kw, int pad);
int xnc_layer_forward(const float* x, const uint32_t* wbits, const float* alpha,
                      int N, int C, int H, int W, int O, int kh, int kw, int pad,
                      void* workspace, float* y, int32_t* acc, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* XNORB200_H */
