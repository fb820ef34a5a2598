// The reference's naive convolutions on the device: the "slow, obviously-correct"
// truth of its verify / bench gates (reference.py:30-122) and its float
// comparison kernel vanilla_conv (_kernels_cy.pyx:107-123, _kernels_py.py:90-108).
//
// One thread per output, every term visited in the reference's (ch, ky, kx)
// order with one rounding per multiply and per add (__fmul_rn / __dadd_rn: no
// FMA contraction, as Python floats and numpy evaluate them).  These kernels
// share nothing with the packed engine (no bit packing, no popcount, no K map),
// which is the point: paper_2007_14178_b200.verify checks the engine against
// them, as verify.py checks the reference's engine against reference.py.
// Not on the hot path.
#include "xnc_common.cuh"

namespace xnc {

// sign_conv2d_int (reference.py:57-90): +-1 int8 planes [C][h][w] against +-1
// int8 filter signs [C][kh][kw]; out-of-plane taps count as +1.
__global__ void k_ref_sign_conv(const int8_t* __restrict__ s, const int8_t* __restrict__ ws, int C,
                                int h, int w, int kh, int kw, int pad, int oh, int ow,
                                int32_t* __restrict__ out) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long)oh * ow) return;
  int y = (int)(i / ow), x = (int)(i - (long)y * ow);
  int acc = 0;
  for (int ch = 0; ch < C; ++ch)
    for (int ky = 0; ky < kh; ++ky) {
      int iy = y + ky - pad;
      for (int kx = 0; kx < kw; ++kx) {
        int ix = x + kx - pad;
        int v = (iy >= 0 && iy < h && ix >= 0 && ix < w) ? s[((long)ch * h + iy) * w + ix] : 1;
        acc += v * ws[(ch * kh + ky) * kw + kx];
      }
    }
  out[i] = acc;
}

// conv2d_float (reference.py:30-54): float64 cross-correlation, zero padding
// (out-of-plane taps skipped), acc += x * w in (ch, ky, kx) order from 0.0.
// bwn != 0: bwn_conv (reference.py:93-122) -- add or subtract x by the sign of
// w (w > 0 adds), then one final multiply by `scale`.
__global__ void k_ref_conv_f64(const double* __restrict__ x, const double* __restrict__ wt, int C,
                               int h, int w, int kh, int kw, int pad, int oh, int ow, int bwn,
                               double scale, double* __restrict__ out) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long)oh * ow) return;
  int y = (int)(i / ow), xo = (int)(i - (long)y * ow);
  double acc = 0.0;
  for (int ch = 0; ch < C; ++ch)
    for (int ky = 0; ky < kh; ++ky) {
      int iy = y + ky - pad;
      if (iy < 0 || iy >= h) continue;
      for (int kx = 0; kx < kw; ++kx) {
        int ix = xo + kx - pad;
        if (ix < 0 || ix >= w) continue;
        double v = x[((long)ch * h + iy) * w + ix], c = wt[(ch * kh + ky) * kw + kx];
        if (bwn) acc = c > 0.0 ? __dadd_rn(acc, v) : __dsub_rn(acc, v);
        else acc = __dadd_rn(acc, __dmul_rn(v, c));
      }
    }
  out[i] = bwn ? __dmul_rn(acc, scale) : acc;
}

// vanilla_conv (_kernels_cy.pyx:107-123): pre-padded [C][ph][pw] against
// weights [C][kh][kw], valid mode, acc = acc + p * w from 0 in (ch, ky, kx)
// order, in the arrays' type (f32 or f64), one rounding per op.
template <typename T>
__device__ inline T mul_rn(T a, T b);
template <>
__device__ inline float mul_rn<float>(float a, float b) { return __fmul_rn(a, b); }
template <>
__device__ inline double mul_rn<double>(double a, double b) { return __dmul_rn(a, b); }
template <typename T>
__device__ inline T add_rn(T a, T b);
template <>
__device__ inline float add_rn<float>(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ inline double add_rn<double>(double a, double b) { return __dadd_rn(a, b); }

template <typename T>
__global__ void k_vanilla_conv(const T* __restrict__ p, const T* __restrict__ wt, int C, int ph,
                               int pw, int kh, int kw, int oh, int ow, T* __restrict__ out) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long)oh * ow) return;
  int y = (int)(i / ow), x = (int)(i - (long)y * ow);
  T acc = T(0);
  for (int ch = 0; ch < C; ++ch)
    for (int ky = 0; ky < kh; ++ky)
      for (int kx = 0; kx < kw; ++kx)
        acc = add_rn(acc, mul_rn(p[((long)ch * ph + y + ky) * pw + x + kx], wt[(ch * kh + ky) * kw + kx]));
  out[i] = acc;
}

inline unsigned grid_for(long n) { return (unsigned)((n + 255) / 256); }

}  // namespace xnc

using namespace xnc;

extern "C" {

int xnc_ref_sign_conv2d(const int8_t* signs, const int8_t* wsigns, int C, int h, int w, int kh, int kw,
                        int pad, int32_t* out, void* stream) {
  if (!signs || !wsigns || !out || C < 1 || h < 1 || w < 1 || kh < 1 || kw < 1 || pad < 0) return XNC_EINVAL;
  int oh = h + 2 * pad - kh + 1, ow = w + 2 * pad - kw + 1;
  if (oh < 1 || ow < 1) return XNC_EINVAL;
  k_ref_sign_conv<<<grid_for((long)oh * ow), 256, 0, as_stream(stream)>>>(signs, wsigns, C, h, w, kh, kw, pad,
                                                                         oh, ow, out);
  return launch_status();
}

int xnc_ref_conv2d_f64(const double* x, const double* wt, int C, int h, int w, int kh, int kw, int pad,
                       int bwn, double scale, double* out, void* stream) {
  if (!x || !wt || !out || C < 1 || h < 1 || w < 1 || kh < 1 || kw < 1 || pad < 0) return XNC_EINVAL;
  int oh = h + 2 * pad - kh + 1, ow = w + 2 * pad - kw + 1;
  if (oh < 1 || ow < 1) return XNC_EINVAL;
  k_ref_conv_f64<<<grid_for((long)oh * ow), 256, 0, as_stream(stream)>>>(x, wt, C, h, w, kh, kw, pad, oh, ow,
                                                                        bwn, scale, out);
  return launch_status();
}

int xnc_vanilla_conv(const void* padded, int dtype, int C, int ph, int pw, const void* weights, int kh,
                     int kw, void* out, void* stream) {
  if (!padded || !weights || !out || C < 1 || kh < 1 || kw < 1 || ph < kh || pw < kw) return XNC_EINVAL;
  int oh = ph - kh + 1, ow = pw - kw + 1;
  cudaStream_t s = as_stream(stream);
  if (dtype == XNC_DTYPE_F32)
    k_vanilla_conv<float><<<grid_for((long)oh * ow), 256, 0, s>>>(
        (const float*)padded, (const float*)weights, C, ph, pw, kh, kw, oh, ow, (float*)out);
  else if (dtype == XNC_DTYPE_F64)
    k_vanilla_conv<double><<<grid_for((long)oh * ow), 256, 0, s>>>(
        (const double*)padded, (const double*)weights, C, ph, pw, kh, kw, oh, ow, (double*)out);
  else
    return XNC_EINVAL;
  return launch_status();
}

}  // extern "C"
