// K1: fused sign + channel bit-pack + channel-mean |x|, and filter binarization.
//
// Reference behaviour restated (not translated):
//  * sign bit = (v >= 0.0f): binarize.py:56-57, _kernels_cy.pyx:61,326
//    (sign(0) = sign(-0.0) = +1; NaN -> 0, the reference would have rejected it).
//  * A = (sequential f32 sum of |x| over c = 0..C-1) * f32(1/C):
//    _kernels_cy.pyx:207-230 (`m = m + fabsf(...)`, `mean_row[x] = m * inv`), :258.
//  * alpha = (sequential f64 sum of |w| in (c,ky,kx) order) / n: binarize.py:72-75,
//    then (float)alpha as xnor_reconstruct's wscale (_kernels_cy.pyx:260).
//
// HBM design: x is NCHW, so for a fixed channel the pixels of one image are
// contiguous.  Each thread owns VEC=4 consecutive pixels and walks the C
// channels with 16-byte loads; a warp's load is 512 contiguous bytes per
// channel (fully coalesced), and x is read exactly once.  The bits for 32
// channels are built in registers and written as one word per pixel.
#include "xnc_common.cuh"

namespace xnc {

// 32 sign bits -> 32 d-bytes, d = 1 for a negative sign (the tcgen05 operand).
__device__ __forceinline__ void store_d32(uint8_t* dst, uint32_t d) {
  uint32_t w[8];
#pragma unroll
  for (int b = 0; b < 8; ++b) w[b] = (((d >> (4 * b)) & 0xFu) * 0x00204081u) & 0x01010101u;
  reinterpret_cast<uint4*>(dst)[0] = make_uint4(w[0], w[1], w[2], w[3]);
  reinterpret_cast<uint4*>(dst)[1] = make_uint4(w[4], w[5], w[6], w[7]);
}

// bits (u32 [N][HW][Cw]) and/or dbytes (u8 [N][HW][Cpad], d = 1 for x < 0, zero
// for c >= C) -- the popc kernels read bits, the tcgen05 kernel reads d-bytes.
template <int VEC>
__global__ void __launch_bounds__(256) k_pack_input(const float* __restrict__ x, int C, int HW,
                                                    int Cw, float inv, long groups_per_img,
                                                    long total_groups,
                                                    uint32_t* __restrict__ bits,
                                                    float* __restrict__ A,
                                                    uint8_t* __restrict__ dbytes, int Cpad) {
  long gid = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= total_groups) return;
  const long n = gid / groups_per_img;
  const int p0 = (int)(gid - n * groups_per_img) * VEC;
  const float* xp = x + (long)n * C * HW + p0;
  uint32_t* bp = bits ? bits + ((long)n * HW + p0) * Cw : nullptr;
  uint8_t* dp = dbytes ? dbytes + ((long)n * HW + p0) * Cpad : nullptr;

  float s[VEC];
#pragma unroll
  for (int i = 0; i < VEC; ++i) s[i] = 0.0f;

  for (int j = 0; j < Cw; ++j) {
    uint32_t word[VEC];
#pragma unroll
    for (int i = 0; i < VEC; ++i) word[i] = 0u;
    const int cend = min(32, C - 32 * j);
    if (cend == 32) {
#pragma unroll 8
      for (int cc = 0; cc < 32; ++cc) {
        const float* src = xp + (long)(32 * j + cc) * HW;
        float v[VEC];
        if constexpr (VEC == 4) {
          float4 t = __ldcs(reinterpret_cast<const float4*>(src));  // streamed once
          v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
        } else {
#pragma unroll
          for (int i = 0; i < VEC; ++i) v[i] = __ldcs(src + i);
        }
#pragma unroll
        for (int i = 0; i < VEC; ++i) {
          s[i] = __fadd_rn(s[i], fabsf(v[i]));
          word[i] |= (v[i] >= 0.0f ? 1u : 0u) << cc;
        }
      }
    } else {
      for (int cc = 0; cc < cend; ++cc) {
        const float* src = xp + (long)(32 * j + cc) * HW;
        float v[VEC];
        if constexpr (VEC == 4) {
          float4 t = __ldcs(reinterpret_cast<const float4*>(src));
          v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
        } else {
#pragma unroll
          for (int i = 0; i < VEC; ++i) v[i] = __ldcs(src + i);
        }
#pragma unroll
        for (int i = 0; i < VEC; ++i) {
          s[i] = __fadd_rn(s[i], fabsf(v[i]));
          word[i] |= (v[i] >= 0.0f ? 1u : 0u) << cc;
        }
      }
    }
    if (bp) {
#pragma unroll
      for (int i = 0; i < VEC; ++i) bp[(long)i * Cw + j] = word[i];
    }
    if (dp) {
      const uint32_t valid = cend == 32 ? 0xFFFFFFFFu : ((1u << cend) - 1u);
#pragma unroll
      for (int i = 0; i < VEC; ++i) store_d32(dp + (long)i * Cpad + 32 * j, ~word[i] & valid);
    }
  }
  if (dp) {
    for (int c = 32 * Cw; c < Cpad; c += 16)
#pragma unroll
      for (int i = 0; i < VEC; ++i) *reinterpret_cast<uint4*>(dp + (long)i * Cpad + c) = make_uint4(0, 0, 0, 0);
  }
  if (A != nullptr) {
    float* ap = A + (long)n * HW + p0;
    if constexpr (VEC == 4) {
      *reinterpret_cast<float4*>(ap) =
          make_float4(__fmul_rn(s[0], inv), __fmul_rn(s[1], inv), __fmul_rn(s[2], inv),
                      __fmul_rn(s[3], inv));
    } else {
#pragma unroll
      for (int i = 0; i < VEC; ++i) ap[i] = __fmul_rn(s[i], inv);
    }
  }
}

int launch_pack_input(const float* x, int N, int C, int H, int W, uint32_t* bits, float* A,
                      cudaStream_t s, uint8_t* dbytes) {
  const int HW = H * W;
  const int Cw = cdiv(C, 32);
  const float inv = (float)(1.0 / (double)C);  // <real_t>(1.0 / channels), _kernels_cy.pyx:258
  const bool vec4 = (HW % 4 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0) &&
                    (A == nullptr || (reinterpret_cast<uintptr_t>(A) & 15) == 0);
  if (vec4) {
    long gpi = HW / 4, total = gpi * N;
    long blocks = cdivl(total, 256);
    k_pack_input<4><<<(unsigned)blocks, 256, 0, s>>>(x, C, HW, Cw, inv, gpi, total, bits, A, dbytes,
                                                     round_up(C, 128));
  } else {
    long gpi = HW, total = gpi * N;
    long blocks = cdivl(total, 256);
    k_pack_input<1><<<(unsigned)blocks, 256, 0, s>>>(x, C, HW, Cw, inv, gpi, total, bits, A, dbytes,
                                                     round_up(C, 128));
  }
  return launch_status();
}

// One thread per filter.  wbits layout [Cw][kh][kw][O] (filters contiguous) so
// the conv kernel stages a filter block with coalesced row copies.  Templated
// on the weight dtype: the drop-in API passes the reference's float64 Tensor3
// values unrounded (sign and alpha are taken from them, binarize.py:65-75).
template <typename T>
__global__ void k_pack_weights(const T* __restrict__ w, int O, int C, int kh, int kw,
                               uint32_t* __restrict__ wbits, float* __restrict__ alpha,
                               double* __restrict__ alpha64) {
  int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= O) return;
  const int kk = kh * kw;
  const long n = (long)C * kk;
  const T* wp = w + (long)o * n;
  double total = 0.0;
  for (long i = 0; i < n; ++i) total = __dadd_rn(total, fabs((double)wp[i]));
  const double a = __ddiv_rn(total, (double)n);
  alpha[o] = __double2float_rn(a);
  if (alpha64) alpha64[o] = a;
  const int Cw = cdiv(C, 32);
  for (int j = 0; j < Cw; ++j)
    for (int t = 0; t < kk; ++t) {
      uint32_t word = 0u;
      const int cend = min(32, C - 32 * j);
      for (int cc = 0; cc < cend; ++cc)
        word |= (wp[(long)(32 * j + cc) * kk + t] >= T(0) ? 1u : 0u) << cc;
      wbits[((long)j * kk + t) * O + o] = word;
    }
}

int launch_pack_weights(const float* w, int O, int C, int kh, int kw, uint32_t* wbits,
                        float* alpha, double* alpha64, cudaStream_t s) {
  k_pack_weights<float><<<cdiv(O, 64), 64, 0, s>>>(w, O, C, kh, kw, wbits, alpha, alpha64);
  return launch_status();
}

int launch_pack_weights_f64(const double* w, int O, int C, int kh, int kw, uint32_t* wbits,
                            float* alpha, double* alpha64, cudaStream_t s) {
  k_pack_weights<double><<<cdiv(O, 64), 64, 0, s>>>(w, O, C, kh, kw, wbits, alpha, alpha64);
  return launch_status();
}

}  // namespace xnc
