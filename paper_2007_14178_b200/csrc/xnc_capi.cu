// extern "C" surface of libxnorb200.so (declared in include/xnorb200.h).
// Cheap argument checks, then enqueue on the caller's stream.  No allocation,
// no synchronisation.
#include <cstdio>

#include "xnc_common.cuh"

using namespace xnc;

namespace {

bool conv_shape_ok(int N, int C, int H, int W, int kh, int kw, int pad) {
  if (N < 1 || C < 1 || H < 1 || W < 1 || pad < 0) return false;
  if (kh < 1 || kw < 1 || kh > kMaxK || kw > kMaxK) return false;
  if (H + 2 * pad - kh + 1 < 1 || W + 2 * pad - kw + 1 < 1) return false;
  // integer decode bound: |acc| <= C*kh*kw must be exact in f32 (2^24)
  if ((long)C * kh * kw > (1L << 24)) return false;
  return true;
}

size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

}  // namespace

extern "C" {

int xnc_abi_version(void) { return 1; }

const char* xnc_strerror(int code) {
  if (code == XNC_OK) return "ok";
  if (code == XNC_EINVAL) return "invalid argument or shape";
  if (code == XNC_ENOTSUP) return "shape not supported by the sm_100a kernels";
  if (code >= XNC_ECUDA_BASE) return cudaGetErrorString((cudaError_t)(code - XNC_ECUDA_BASE));
  return "unknown error";
}

int xnc_pack_input(const float* x, int N, int C, int H, int W, uint32_t* bits, float* A,
                   void* stream) {
  if (!x || !bits || N < 1 || C < 1 || H < 1 || W < 1) return XNC_EINVAL;
  return launch_pack_input(x, N, C, H, W, bits, A, as_stream(stream));
}

int xnc_pack_weights(const float* w, int O, int C, int kh, int kw, uint32_t* wbits,
                     float* alpha, double* alpha64, void* stream) {
  if (!w || !wbits || !alpha || O < 1 || C < 1 || kh < 1 || kw < 1 || kh > kMaxK ||
      kw > kMaxK)
    return XNC_EINVAL;
  return launch_pack_weights(w, O, C, kh, kw, wbits, alpha, alpha64, as_stream(stream));
}

int xnc_pack_weights_f64(const double* w, int O, int C, int kh, int kw, uint32_t* wbits,
                         float* alpha, double* alpha64, void* stream) {
  if (!w || !wbits || !alpha || O < 1 || C < 1 || kh < 1 || kw < 1 || kh > kMaxK ||
      kw > kMaxK)
    return XNC_EINVAL;
  return launch_pack_weights_f64(w, O, C, kh, kw, wbits, alpha, alpha64, as_stream(stream));
}

int xnc_scale_map(const float* A, int N, int H, int W, int kh, int kw, int pad, float* K,
                  void* stream) {
  if (!A || !K || !conv_shape_ok(N, 1, H, W, kh, kw, pad)) return XNC_EINVAL;
  return launch_scale_map(A, N, H, W, kh, kw, pad, K, as_stream(stream));
}

int xnc_xnor_conv_variant(int variant, const uint32_t* bits, const uint32_t* wbits,
                          const float* K, const float* alpha, int N, int C, int H, int W, int O,
                          int kh, int kw, int pad, float* y, int32_t* acc, void* stream) {
  if (!bits || !wbits || O < 1 || !conv_shape_ok(N, C, H, W, kh, kw, pad)) return XNC_EINVAL;
  if (!y && !acc) return XNC_EINVAL;
  if (y && (!K || !alpha)) return XNC_EINVAL;
  switch (variant) {
    case XNC_CONV_POPC:
      return launch_conv_popc(bits, wbits, K, alpha, N, C, H, W, O, kh, kw, pad, y, acc,
                              as_stream(stream));
    case XNC_CONV_B1MMA:
      return launch_conv_b1mma(bits, wbits, K, alpha, N, C, H, W, O, kh, kw, pad, y, acc,
                               as_stream(stream));
    default:
      return XNC_EINVAL;
  }
}

int xnc_xnor_conv(const uint32_t* bits, const uint32_t* wbits, const float* K,
                  const float* alpha, int N, int C, int H, int W, int O, int kh, int kw,
                  int pad, float* y, int32_t* acc, void* stream) {
  return xnc_xnor_conv_variant(XNC_CONV_POPC, bits, wbits, K, alpha, N, C, H, W, O, kh, kw, pad,
                               y, acc, stream);
}

size_t xnc_umma_weight_bytes(int O, int C, int kh, int kw) {
  if (O < 1 || C < 1 || kh < 1 || kw < 1 || kh > kMaxK || kw > kMaxK) return 0;
  return umma_weight_bytes(O, C, kh, kw);
}

int xnc_umma_supported(int N, int C, int H, int W, int O, int kh, int kw, int pad) {
  if (O < 1 || !conv_shape_ok(N, C, H, W, kh, kw, pad)) return 0;
  return umma_supported(N, C, H, W, O, kh, kw, pad) ? 1 : 0;
}

int xnc_pack_weights_umma(const void* w, int dtype, int O, int C, int kh, int kw, uint8_t* wq,
                          int32_t* sw, void* stream) {
  if (!w || !wq || !sw || O < 1 || C < 1 || kh < 1 || kw < 1 || kh > kMaxK || kw > kMaxK ||
      (dtype != XNC_DTYPE_F32 && dtype != XNC_DTYPE_F64))
    return XNC_EINVAL;
  return launch_pack_weights_umma(w, dtype, O, C, kh, kw, wq, sw, as_stream(stream));
}

int xnc_pack_input_affine(const float* x, int N, int C, int H, int W, const float* in_scale,
                          const float* in_shift, uint32_t* bits, float* A, void* stream) {
  if (!x || !bits || N < 1 || C < 1 || H < 1 || W < 1 || (!in_scale != !in_shift)) return XNC_EINVAL;
  return launch_pack_input(x, N, C, H, W, bits, A, as_stream(stream), in_scale, in_shift);
}

int xnc_pack_input_pool(const float* x, int N, int C, int Hin, int Win, int pool_k, int pool_s,
                        const float* in_scale, const float* in_shift, uint32_t* bits, float* A, void* stream) {
  if (!x || !bits || N < 1 || C < 1 || Hin < 1 || Win < 1 || pool_k < 1 || pool_s < 1 || (!in_scale != !in_shift))
    return XNC_EINVAL;
  return launch_pack_input_pool(x, N, C, Hin, Win, pool_k, pool_s, bits, A, as_stream(stream), in_scale, in_shift);
}

int xnc_pack_input_pool_nhwc(const float* x, int N, int C, int Hin, int Win, int pool_k, int pool_s, int relu,
                             const float* bias, const float* in_scale, const float* in_shift, uint32_t* bits,
                             float* A, void* stream) {
  if (!x || !bits || N < 1 || C < 1 || Hin < 1 || Win < 1 || pool_k < 1 || pool_s < 1 || (!in_scale != !in_shift))
    return XNC_EINVAL;
  return launch_pack_input_pool_nhwc(x, N, C, Hin, Win, pool_k, pool_s, relu, bias, bits, A, as_stream(stream),
                                     in_scale, in_shift);
}

int xnc_xnor_conv_umma_affine(const uint32_t* bits, const uint8_t* wq, const int32_t* sw, const float* K,
                              const float* alpha, int N, int C, int H, int W, int O, int kh, int kw, int pad,
                              const float* out_scale, const float* out_shift, float* y, int32_t* acc,
                              void* stream) {
  if (!bits || !wq || !sw || O < 1 || !conv_shape_ok(N, C, H, W, kh, kw, pad)) return XNC_EINVAL;
  if (!y && !acc) return XNC_EINVAL;
  if (y && (!K || !alpha)) return XNC_EINVAL;
  if (!out_scale != !out_shift) return XNC_EINVAL;
  return launch_conv_umma(bits, wq, sw, K, alpha, N, C, H, W, O, kh, kw, pad, y, acc, as_stream(stream),
                          out_scale, out_shift);
}

int xnc_xnor_conv_umma(const uint32_t* bits, const uint8_t* wq, const int32_t* sw, const float* K,
                       const float* alpha, int N, int C, int H, int W, int O, int kh, int kw, int pad,
                       float* y, int32_t* acc, void* stream) {
  if (!bits || !wq || !sw || O < 1 || !conv_shape_ok(N, C, H, W, kh, kw, pad)) return XNC_EINVAL;
  if (!y && !acc) return XNC_EINVAL;
  if (y && (!K || !alpha)) return XNC_EINVAL;
  return launch_conv_umma(bits, wq, sw, K, alpha, N, C, H, W, O, kh, kw, pad, y, acc,
                          as_stream(stream));
}

int xnc_max_pool(const float* x, int N, int C, int Hin, int Win, int pool_k, int pool_s, int relu, int nhwc,
                 const float* bias, float* out, void* stream) {
  if (!x || !out || N < 1 || C < 1 || pool_k < 1 || pool_k > 8 || pool_s < 1 || Hin < pool_k || Win < pool_k)
    return XNC_EINVAL;
  return nhwc ? launch_max_pool_nhwc(x, N, C, Hin, Win, pool_k, pool_s, relu, bias, out, as_stream(stream))
              : launch_max_pool(x, N, C, Hin, Win, pool_k, pool_s, relu, bias, out, as_stream(stream));
}

int xnc_plane_affine(float* y, int N, int O, long plane, const float* scale, const float* shift, void* stream) {
  if (!y || !scale || !shift || N < 0 || O < 1 || plane < 0) return XNC_EINVAL;
  return launch_plane_affine(y, N, O, plane, scale, shift, as_stream(stream));
}

int xnc_pad_space_to_depth(const float* x, int N, int C, int H, int W, int pad, int r, int nhwc, float* out,
                           void* stream) {
  if (!x || !out || N < 1 || C < 1 || H < 1 || W < 1 || pad < 0 || r < 1 || (H + 2 * pad) % r ||
      (W + 2 * pad) % r)
    return XNC_EINVAL;
  return launch_pad_s2d(x, N, C, H, W, pad, r, nhwc, out, as_stream(stream));
}

int xnc_pack_input_nhwc(const float* x, int N, int C, int H, int W, const float* in_scale, const float* in_shift,
                        uint32_t* bits, float* A, void* stream) {
  if (!x || !bits || N < 1 || C < 1 || H < 1 || W < 1 || (!in_scale != !in_shift)) return XNC_EINVAL;
  return launch_pack_input_nhwc(x, N, C, H, W, bits, A, as_stream(stream), in_scale, in_shift);
}

int xnc_umma_emit_supported(int N, int C, int H, int W, int O, int kh, int kw, int pad) {
  if (O < 1 || !conv_shape_ok(N, C, H, W, kh, kw, pad)) return 0;
  return umma_emit_supported(N, C, H, W, O, kh, kw, pad) ? 1 : 0;
}

int xnc_xnor_conv_umma_emit(const uint32_t* bits, const uint8_t* wq, const int32_t* sw, const float* K,
                            const float* alpha, int N, int C, int H, int W, int O, int kh, int kw, int pad,
                            const float* out_scale, const float* out_shift, uint32_t* next_bits, float* next_A,
                            void* stream) {
  if (!bits || !wq || !sw || !K || !alpha || !next_bits || O < 1 || !conv_shape_ok(N, C, H, W, kh, kw, pad))
    return XNC_EINVAL;
  if (!out_scale != !out_shift) return XNC_EINVAL;
  return launch_conv_umma(bits, wq, sw, K, alpha, N, C, H, W, O, kh, kw, pad, nullptr, nullptr, as_stream(stream),
                          out_scale, out_shift, nullptr, next_bits, next_A);
}

size_t xnc_umma_split_ws_bytes(int N, int C, int H, int W, int O, int kh, int kw, int pad) {
  if (O < 1 || !conv_shape_ok(N, C, H, W, kh, kw, pad)) return 0;
  return umma_split_ws_bytes(N, C, H, W, O, kh, kw, pad);
}

int xnc_xnor_conv_umma_ws(const uint32_t* bits, const uint8_t* wq, const int32_t* sw, const float* K,
                          const float* alpha, int N, int C, int H, int W, int O, int kh, int kw, int pad,
                          const float* out_scale, const float* out_shift, int32_t* split_ws, float* y,
                          int32_t* acc, void* stream) {
  if (!bits || !wq || !sw || O < 1 || !conv_shape_ok(N, C, H, W, kh, kw, pad)) return XNC_EINVAL;
  if (!y && !acc) return XNC_EINVAL;
  if (y && (!K || !alpha)) return XNC_EINVAL;
  if (!out_scale != !out_shift) return XNC_EINVAL;
  return launch_conv_umma(bits, wq, sw, K, alpha, N, C, H, W, O, kh, kw, pad, y, acc, as_stream(stream),
                          out_scale, out_shift, split_ws);
}

int xnc_xnor_conv_umma_nhwc(const uint32_t* bits, const uint8_t* wq, const int32_t* sw, const float* K,
                            const float* alpha, int N, int C, int H, int W, int O, int kh, int kw, int pad,
                            const float* out_scale, const float* out_shift, int32_t* split_ws, float* y,
                            void* stream) {
  if (!bits || !wq || !sw || !K || !alpha || !y || O < 1 || (O & 3) || !conv_shape_ok(N, C, H, W, kh, kw, pad) ||
      (reinterpret_cast<uintptr_t>(y) & 15) || (!out_scale != !out_shift))
    return XNC_EINVAL;
  return launch_conv_umma(bits, wq, sw, K, alpha, N, C, H, W, O, kh, kw, pad, y, nullptr, as_stream(stream),
                          out_scale, out_shift, split_ws, nullptr, nullptr, 1);
}

int xnc_xnor_conv_umma_nhwc_emit(const uint32_t* bits, const uint8_t* wq, const int32_t* sw, const float* K,
                                 const float* alpha, int N, int C, int H, int W, int O, int kh, int kw, int pad,
                                 const float* out_scale, const float* out_shift, int32_t* split_ws, float* y,
                                 uint32_t* next_bits, float* next_A, void* stream) {
  if (!bits || !wq || !sw || !K || !alpha || !y || !next_bits || !next_A || O < 1 || (O & 31) ||
      !conv_shape_ok(N, C, H, W, kh, kw, pad) || (reinterpret_cast<uintptr_t>(y) & 15) || (!out_scale != !out_shift))
    return XNC_EINVAL;
  return launch_conv_umma(bits, wq, sw, K, alpha, N, C, H, W, O, kh, kw, pad, y, nullptr, as_stream(stream),
                          out_scale, out_shift, split_ws, next_bits, next_A, 1);
}

int xnc_umma_profile(unsigned long long* host_out, int n_ctas) {
  if (!host_out || n_ctas < 1) return XNC_EINVAL;
  return umma_profile_read(host_out, n_ctas);
}

size_t xnc_layer_workspace_bytes(int N, int C, int H, int W, int kh, int kw, int pad) {
  if (!conv_shape_ok(N, C, H, W, kh, kw, pad)) return 0;
  const size_t oh = H + 2 * pad - kh + 1, ow = W + 2 * pad - kw + 1;
  const size_t Cw = (C + 31) / 32;
  return align256((size_t)N * H * W * Cw * 4) + align256((size_t)N * H * W * 4) +
         align256((size_t)N * oh * ow * 4);
}

int xnc_layer_forward(const float* x, const uint32_t* wbits, const float* alpha, int N, int C,
                      int H, int W, int O, int kh, int kw, int pad, void* workspace, float* y,
                      int32_t* acc, void* stream) {
  if (!x || !wbits || !alpha || !workspace || O < 1 || !conv_shape_ok(N, C, H, W, kh, kw, pad))
    return XNC_EINVAL;
  const size_t Cw = (C + 31) / 32;
  char* ws = static_cast<char*>(workspace);
  uint32_t* bits = reinterpret_cast<uint32_t*>(ws);
  float* A = reinterpret_cast<float*>(ws + align256((size_t)N * H * W * Cw * 4));
  float* K = reinterpret_cast<float*>(reinterpret_cast<char*>(A) + align256((size_t)N * H * W * 4));
  cudaStream_t s = as_stream(stream);
  int rc = launch_pack_input(x, N, C, H, W, bits, A, s);
  if (rc) return rc;
  rc = launch_scale_map(A, N, H, W, kh, kw, pad, K, s);
  if (rc) return rc;
  return launch_conv_popc(bits, wbits, K, alpha, N, C, H, W, O, kh, kw, pad, y, acc, s);
}

int xnc_layer_forward_umma(const float* x, const uint8_t* wq, const int32_t* sw, const float* alpha,
                           int N, int C, int H, int W, int O, int kh, int kw, int pad, void* workspace,
                           float* y, int32_t* acc, void* stream) {
  if (!x || !wq || !sw || !alpha || !workspace || O < 1 || !conv_shape_ok(N, C, H, W, kh, kw, pad))
    return XNC_EINVAL;
  if (!umma_supported(N, C, H, W, O, kh, kw, pad)) return XNC_ENOTSUP;
  const size_t Cw = (C + 31) / 32;
  char* ws = static_cast<char*>(workspace);
  uint32_t* bits = reinterpret_cast<uint32_t*>(ws);
  float* A = reinterpret_cast<float*>(ws + align256((size_t)N * H * W * Cw * 4));
  float* K = reinterpret_cast<float*>(reinterpret_cast<char*>(A) + align256((size_t)N * H * W * 4));
  cudaStream_t s = as_stream(stream);
  int rc = launch_pack_input(x, N, C, H, W, bits, A, s);
  if (rc) return rc;
  rc = launch_scale_map(A, N, H, W, kh, kw, pad, K, s);
  if (rc) return rc;
  return launch_conv_umma(bits, wq, sw, K, alpha, N, C, H, W, O, kh, kw, pad, y, acc, s);
}

}  // extern "C"
