// The reference kernel seam on the device: one C-ABI entry point per function
// of the module `_backend.get_kernels()` returns (_backend.py:28-41,
// _kernels_cy.pyx), plus the module-level float64 operators of the reference's
// Python API (tensor.py:103-105, scaling.py:91-98, engine.py:102-120,
// pack.py:123-154).  These keep the reference's TILE-WORD layout (PackedTileGrid)
// and its float order, so a reference build can bind them as a device backend
// and the drop-in Python API (paper_2007_14178_b200.pack /
// engine / scaling / pipeline) runs on them.  The batched hot path (K1-K4) does
// not use the tile layout; this file is the interop surface.
//
// Every kernel writes each output element from exactly one thread in the
// reference's fixed order -- deterministic, no atomics except the overlap flag.
#include "xnc_common.cuh"

namespace xnc {

typedef unsigned long long u64;

// ---------------------------------------------------------------- sign / pack
template <typename T>
__device__ inline bool nonneg(T v) { return v >= T(0); }

template <typename T>
__global__ void k_pack_plane(const T* __restrict__ plane, int h, int w, int tiles_y, int tiles_x,
                             int tile_h, int tile_w, int sy, int sx, u64* __restrict__ out) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= tiles_y * tiles_x) return;
  int ty = t / tiles_x, tx = t - ty * tiles_x;
  u64 word = 0;
  for (int r = 0; r < tile_h; ++r) {
    int y = ty * sy + r;
    if (y >= h) break;
    for (int c = 0; c < tile_w; ++c) {
      int x = tx * sx + c;
      if (x < w && nonneg(plane[(long)y * w + x])) word |= 1ull << (r * tile_w + c);
    }
  }
  out[t] = word;
}

// unpack (pack.py:123-154): every covered pixel takes its value from the tiles
// covering it; any disagreement sets *mismatch (the OverlapMismatchError case).
__global__ void k_unpack_plane(const u64* __restrict__ words, int tiles_y, int tiles_x,
                               int tile_h, int tile_w, int sy, int sx, int cov_h, int cov_w,
                               int8_t* __restrict__ plane, int* __restrict__ mismatch) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= cov_h * cov_w) return;
  int y = p / cov_w, x = p - y * cov_w;
  int ty_lo = max(0, (y - tile_h + sy) / sy), ty_hi = min(tiles_y - 1, y / sy);
  int tx_lo = max(0, (x - tile_w + sx) / sx), tx_hi = min(tiles_x - 1, x / sx);
  int val = -1;
  bool bad = false;
  for (int ty = ty_lo; ty <= ty_hi; ++ty) {
    int r = y - ty * sy;
    if (r < 0 || r >= tile_h) continue;
    for (int tx = tx_lo; tx <= tx_hi; ++tx) {
      int c = x - tx * sx;
      if (c < 0 || c >= tile_w) continue;
      int b = (int)((words[(long)ty * tiles_x + tx] >> (r * tile_w + c)) & 1ull);
      if (val < 0) val = b; else if (val != b) bad = true;
    }
  }
  plane[p] = (val == 1) ? 1 : -1;
  if (bad) atomicOr(mismatch, 1);
}

__global__ void k_sign_f64(const double* __restrict__ x, long n, int8_t* __restrict__ out) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = x[i] >= 0.0 ? 1 : -1;
}

// ---------------------------------------------------------------- xnor decode
// xnor_accumulate (_kernels_cy.pyx:76-104): one thread per output pixel.
__global__ void k_xnor_accumulate(const u64* __restrict__ words, int channels, int tiles_y,
                                  int tiles_x, const u64* __restrict__ ww, u64 mask, int tile_w,
                                  int sy, int sx, int k_area, int32_t* __restrict__ out,
                                  int out_h, int out_w) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= out_h * out_w) return;
  int row = p / out_w, col = p - row * out_w;
  int ty = row / sy, tx = col / sx;
  int shift = (row - ty * sy) * tile_w + (col - tx * sx);
  const u64* wp = words + (long)ty * tiles_x + tx;
  const long plane = (long)tiles_y * tiles_x;
  int acc = 0;
  for (int ch = 0; ch < channels; ++ch) {
    u64 diff = ((wp[ch * plane] >> shift) ^ ww[ch]) & mask;
    acc += k_area - 2 * __popcll(diff);
  }
  out[p] = acc;
}

// build_filter (engine.py:102-120) for O filters at once: tile-layout words and
// the float64 alpha (sequential |w| sum in (c,ky,kx) order, binarize.py:72-75).
__global__ void k_filter_words(const double* __restrict__ w, int O, int C, int kh, int kw,
                               int tile_w, u64* __restrict__ words, double* __restrict__ alpha) {
  int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= O) return;
  const long n = (long)C * kh * kw;
  const double* wp = w + (long)o * n;
  double total = 0.0;
  for (long i = 0; i < n; ++i) total = __dadd_rn(total, fabs(wp[i]));
  alpha[o] = __ddiv_rn(total, (double)n);
  for (int ch = 0; ch < C; ++ch) {
    u64 word = 0;
    for (int r = 0; r < kh; ++r)
      for (int c = 0; c < kw; ++c)
        if (wp[((long)ch * kh + r) * kw + c] >= 0.0) word |= 1ull << (r * tile_w + c);
    words[(long)o * C + ch] = word;
  }
}

// ---------------------------------------------------------------- float side
template <typename T> __device__ inline T add_rn(T a, T b);
template <> __device__ inline float add_rn(float a, float b) { return __fadd_rn(a, b); }
template <> __device__ inline double add_rn(double a, double b) { return __dadd_rn(a, b); }
template <typename T> __device__ inline T mul_rn(T a, T b);
template <> __device__ inline float mul_rn(float a, float b) { return __fmul_rn(a, b); }
template <> __device__ inline double mul_rn(double a, double b) { return __dmul_rn(a, b); }

// box_mean (_kernels_cy.pyx:126-148): valid row sums into tmp, column sums * scale.
template <typename T>
__global__ void k_box_rows(const T* __restrict__ a, int h, int w, int kw, T* __restrict__ tmp,
                           int tmp_w) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= h * tmp_w) return;
  int y = p / tmp_w, x = p - y * tmp_w;
  T acc = T(0);
  for (int d = 0; d < kw; ++d) acc = add_rn(acc, a[(long)y * w + x + d]);
  tmp[p] = acc;
}

template <typename T>
__global__ void k_box_cols(const T* __restrict__ tmp, int tmp_w, int kh, T scale, int out_h,
                           T* __restrict__ out) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= out_h * tmp_w) return;
  int y = p / tmp_w, x = p - y * tmp_w;
  T acc = T(0);
  for (int d = 0; d < kh; ++d) acc = add_rn(acc, tmp[(long)(y + d) * tmp_w + x]);
  out[p] = mul_rn(acc, scale);
}

// scale_rows (_kernels_cy.pyx:151-186): tmp[y][x] = sum_d (sum_ch |p[ch][y][x+d]|) * inv
template <typename T>
__global__ void k_scale_rows(const T* __restrict__ padded, int channels, int h, int w, int kw,
                             T inv, T* __restrict__ tmp, int tmp_w) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= h * tmp_w) return;
  int y = p / tmp_w, x = p - y * tmp_w;
  const long plane = (long)h * w;
  T acc = T(0);
  for (int d = 0; d < kw; ++d) {
    T m = T(0);
    for (int ch = 0; ch < channels; ++ch) m = add_rn(m, (T)fabs(padded[ch * plane + (long)y * w + x + d]));
    acc = add_rn(acc, mul_rn(m, inv));
  }
  tmp[p] = acc;
}

// scale_join (_kernels_cy.pyx:189-204): out = (T)ints * (sum_d tmp[y+d][x] * scale) * wscale
template <typename T>
__global__ void k_scale_join(const T* __restrict__ tmp, int tmp_w, const int32_t* __restrict__ ints,
                             int kh, T scale, T wscale, int out_h, int out_w, T* __restrict__ out) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= out_h * out_w) return;
  int y = p / out_w, x = p - y * out_w;
  T acc = T(0);
  for (int d = 0; d < kh; ++d) acc = add_rn(acc, tmp[(long)(y + d) * tmp_w + x]);
  out[p] = mul_rn(mul_rn((T)ints[p], mul_rn(acc, scale)), wscale);
}

// channel_abs_mean (tensor.py:103-105): numpy reduces axis 0 sequentially, then / C.
__global__ void k_channel_abs_mean_f64(const double* __restrict__ x, int C, long hw,
                                       double* __restrict__ A) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= hw) return;
  double s = fabs(x[i]);
  for (int c = 1; c < C; ++c) s = __dadd_rn(s, fabs(x[(long)c * hw + i]));
  A[i] = __ddiv_rn(s, (double)C);
}

// numpy's pairwise summation (numpy/_core/src/umath/loops_utils.h.src pairwise_sum):
// what np.abs(x).mean(axis=0) does when the reduced axis is the only one, i.e. a
// (C,1,1) tensor.  <8 terms: one running sum; <=128: eight strided accumulators
// combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a sequential tail; above that
// split at n/2 rounded down to a multiple of 8 and recurse.
__device__ double np_pairwise_abs_sum(const double* a, long n) {
  if (n < 8) {
    double r = 0.0;
    for (long i = 0; i < n; ++i) r = __dadd_rn(r, fabs(a[i]));
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = fabs(a[j]);
    long i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], fabs(a[i + j]));
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, fabs(a[i]));
    return res;
  }
  long n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(np_pairwise_abs_sum(a, n2), np_pairwise_abs_sum(a + n2, n - n2));
}

// channel_abs_mean of a (C,1,1) tensor: numpy reduces the lone contiguous axis
// pairwise (0.0 identity first), not sequentially.
__global__ void k_channel_abs_mean_1x1_f64(const double* __restrict__ x, int C, double* __restrict__ A) {
  if (threadIdx.x == 0 && blockIdx.x == 0) A[0] = __ddiv_rn(__dadd_rn(0.0, np_pairwise_abs_sum(x, C)), (double)C);
}

// apply_scaling (scaling.py:91-98): ints * K * alpha in float64, left to right.
__global__ void k_apply_scaling_f64(const int32_t* __restrict__ ints, const double* __restrict__ K,
                                    double alpha, long n, double* __restrict__ out) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = __dmul_rn(__dmul_rn((double)ints[i], K[i]), alpha);
}

inline unsigned blocks_for(long n, int bs = 256) { return (unsigned)((n + bs - 1) / bs); }

}  // namespace xnc

using namespace xnc;

extern "C" {

int xnc_pack_plane(const void* plane, int dtype, int h, int w, int tiles_y, int tiles_x,
                   int tile_h, int tile_w, int stride_y, int stride_x, uint64_t* out_words,
                   void* stream) {
  if (!plane || !out_words || h < 1 || w < 1 || tiles_y < 1 || tiles_x < 1 || tile_h * tile_w > 64 ||
      stride_y < 1 || stride_x < 1)
    return XNC_EINVAL;
  cudaStream_t s = as_stream(stream);
  long n = (long)tiles_y * tiles_x;
  u64* out = reinterpret_cast<u64*>(out_words);
  switch (dtype) {
    case XNC_DTYPE_F32:
      k_pack_plane<float><<<blocks_for(n), 256, 0, s>>>((const float*)plane, h, w, tiles_y, tiles_x,
                                                       tile_h, tile_w, stride_y, stride_x, out);
      break;
    case XNC_DTYPE_F64:
      k_pack_plane<double><<<blocks_for(n), 256, 0, s>>>((const double*)plane, h, w, tiles_y, tiles_x,
                                                        tile_h, tile_w, stride_y, stride_x, out);
      break;
    case XNC_DTYPE_I8:
      k_pack_plane<int8_t><<<blocks_for(n), 256, 0, s>>>((const int8_t*)plane, h, w, tiles_y, tiles_x,
                                                        tile_h, tile_w, stride_y, stride_x, out);
      break;
    default:
      return XNC_EINVAL;
  }
  return launch_status();
}

int xnc_unpack_plane(const uint64_t* words, int tiles_y, int tiles_x, int tile_h, int tile_w,
                     int stride_y, int stride_x, int8_t* plane_cov, int* mismatch, void* stream) {
  if (!words || !plane_cov || !mismatch || tiles_y < 1 || tiles_x < 1 || stride_y < 1 || stride_x < 1)
    return XNC_EINVAL;
  int cov_h = (tiles_y - 1) * stride_y + tile_h, cov_w = (tiles_x - 1) * stride_x + tile_w;
  long n = (long)cov_h * cov_w;
  k_unpack_plane<<<blocks_for(n), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const u64*>(words), tiles_y, tiles_x, tile_h, tile_w, stride_y, stride_x, cov_h,
      cov_w, plane_cov, mismatch);
  return launch_status();
}

int xnc_sign_plane(const double* x, long n, int8_t* out, void* stream) {
  if (!x || !out || n < 0) return XNC_EINVAL;
  if (n == 0) return XNC_OK;
  k_sign_f64<<<blocks_for(n), 256, 0, as_stream(stream)>>>(x, n, out);
  return launch_status();
}

int xnc_xnor_accumulate(const uint64_t* words, int channels, int tiles_y, int tiles_x,
                        const uint64_t* weight_words, uint64_t mask, int tile_w, int stride_y,
                        int stride_x, int k_area, int32_t* out, int out_h, int out_w,
                        void* stream) {
  if (!words || !weight_words || !out || channels < 1 || out_h < 1 || out_w < 1 ||
      tiles_y * stride_y < out_h || tiles_x * stride_x < out_w)
    return XNC_EINVAL;
  long n = (long)out_h * out_w;
  k_xnor_accumulate<<<blocks_for(n), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const u64*>(words), channels, tiles_y, tiles_x,
      reinterpret_cast<const u64*>(weight_words), (u64)mask, tile_w, stride_y, stride_x, k_area, out,
      out_h, out_w);
  return launch_status();
}

int xnc_filter_words(const double* w, int O, int C, int kh, int kw, int tile_w, uint64_t* words,
                     double* alpha, void* stream) {
  if (!w || !words || !alpha || O < 1 || C < 1 || kh < 1 || kw < 1 || kh * tile_w > 64 || kw > tile_w)
    return XNC_EINVAL;
  k_filter_words<<<blocks_for(O, 64), 64, 0, as_stream(stream)>>>(
      w, O, C, kh, kw, tile_w, reinterpret_cast<u64*>(words), alpha);
  return launch_status();
}

int xnc_box_mean(const void* a, int dtype, int h, int w, int kh, int kw, double scale, void* tmp,
                 void* out, void* stream) {
  int tmp_w = w - kw + 1, out_h = h - kh + 1;
  if (!a || !tmp || !out || tmp_w < 1 || out_h < 1 || kh < 1 || kw < 1) return XNC_EINVAL;
  cudaStream_t s = as_stream(stream);
  if (dtype == XNC_DTYPE_F64) {
    k_box_rows<double><<<blocks_for((long)h * tmp_w), 256, 0, s>>>((const double*)a, h, w, kw, (double*)tmp, tmp_w);
    k_box_cols<double><<<blocks_for((long)out_h * tmp_w), 256, 0, s>>>((const double*)tmp, tmp_w, kh, scale,
                                                                      out_h, (double*)out);
  } else if (dtype == XNC_DTYPE_F32) {
    k_box_rows<float><<<blocks_for((long)h * tmp_w), 256, 0, s>>>((const float*)a, h, w, kw, (float*)tmp, tmp_w);
    k_box_cols<float><<<blocks_for((long)out_h * tmp_w), 256, 0, s>>>((const float*)tmp, tmp_w, kh,
                                                                     (float)scale, out_h, (float*)out);
  } else {
    return XNC_EINVAL;
  }
  return launch_status();
}

int xnc_scale_rows(const void* padded, int dtype, int channels, int h, int w, int kw, void* tmp,
                   void* stream) {
  int tmp_w = w - kw + 1;
  if (!padded || !tmp || channels < 1 || tmp_w < 1) return XNC_EINVAL;
  cudaStream_t s = as_stream(stream);
  long n = (long)h * tmp_w;
  if (dtype == XNC_DTYPE_F64)
    k_scale_rows<double><<<blocks_for(n), 256, 0, s>>>((const double*)padded, channels, h, w, kw,
                                                       1.0 / channels, (double*)tmp, tmp_w);
  else if (dtype == XNC_DTYPE_F32)
    k_scale_rows<float><<<blocks_for(n), 256, 0, s>>>((const float*)padded, channels, h, w, kw,
                                                      (float)(1.0 / channels), (float*)tmp, tmp_w);
  else
    return XNC_EINVAL;
  return launch_status();
}

int xnc_scale_join(const void* tmp, int dtype, const int32_t* ints, int kh, double scale,
                   double weight_scale, int out_h, int out_w, void* out, void* stream) {
  if (!tmp || !ints || !out || out_h < 1 || out_w < 1 || kh < 1) return XNC_EINVAL;
  cudaStream_t s = as_stream(stream);
  long n = (long)out_h * out_w;
  if (dtype == XNC_DTYPE_F64)
    k_scale_join<double><<<blocks_for(n), 256, 0, s>>>((const double*)tmp, out_w, ints, kh, scale,
                                                       weight_scale, out_h, out_w, (double*)out);
  else if (dtype == XNC_DTYPE_F32)
    k_scale_join<float><<<blocks_for(n), 256, 0, s>>>((const float*)tmp, out_w, ints, kh, (float)scale,
                                                      (float)weight_scale, out_h, out_w, (float*)out);
  else
    return XNC_EINVAL;
  return launch_status();
}

int xnc_xnor_reconstruct(const uint64_t* weight_words, uint64_t mask, int tile_h, int tile_w,
                         int stride_y, int stride_x, int k_area, const void* padded, int dtype,
                         int channels, int ph, int pw, int kh, int kw, double scale,
                         double weight_scale, void* out, void* stream) {
  const int out_h = ph - kh + 1, out_w = pw - kw + 1;
  if (!weight_words || !padded || !out || channels < 1 || out_h < 1 || out_w < 1) return XNC_EINVAL;
  if (dtype != XNC_DTYPE_F32 && dtype != XNC_DTYPE_F64) return XNC_EINVAL;
  cudaStream_t s = as_stream(stream);
  const int tiles_y = cdiv(out_h, stride_y), tiles_x = cdiv(out_w, stride_x);
  const size_t esz = dtype == XNC_DTYPE_F64 ? 8 : 4;
  // stream-ordered scratch (the reference mallocs per band, _kernels_cy.pyx:285-289)
  const size_t words_b = (size_t)channels * tiles_y * tiles_x * 8, ints_b = (size_t)out_h * out_w * 4,
               tmp_b = (size_t)ph * out_w * esz;
  char* scratch = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&scratch, words_b + ints_b + tmp_b + 512, s);
  if (e != cudaSuccess) return XNC_ECUDA_BASE + (int)e;
  uint64_t* words = reinterpret_cast<uint64_t*>(scratch);
  int32_t* ints = reinterpret_cast<int32_t*>(scratch + ((words_b + 255) & ~(size_t)255));
  void* tmp = scratch + ((words_b + 255) & ~(size_t)255) + ((ints_b + 255) & ~(size_t)255);
  int rc = XNC_OK;
  const long plane = (long)ph * pw;
  for (int ch = 0; ch < channels && rc == XNC_OK; ++ch) {
    const char* p = static_cast<const char*>(padded) + ch * plane * esz;
    rc = xnc_pack_plane(p, dtype, ph, pw, tiles_y, tiles_x, tile_h, tile_w, stride_y, stride_x,
                        words + (long)ch * tiles_y * tiles_x, stream);
  }
  if (rc == XNC_OK)
    rc = xnc_xnor_accumulate(words, channels, tiles_y, tiles_x, weight_words, mask, tile_w, stride_y,
                             stride_x, k_area, ints, out_h, out_w, stream);
  if (rc == XNC_OK) rc = xnc_scale_rows(padded, dtype, channels, ph, pw, kw, tmp, stream);
  if (rc == XNC_OK)
    rc = xnc_scale_join(tmp, dtype, ints, kh, scale, weight_scale, out_h, out_w, out, stream);
  cudaFreeAsync(scratch, s);
  return rc;
}

int xnc_channel_abs_mean_f64(const double* x, int C, int H, int W, double* A, void* stream) {
  if (!x || !A || C < 1 || H < 1 || W < 1) return XNC_EINVAL;
  long hw = (long)H * W;
  if (hw == 1) {  // numpy's pairwise order for a lone reduced axis (see above)
    k_channel_abs_mean_1x1_f64<<<1, 32, 0, as_stream(stream)>>>(x, C, A);
    return launch_status();
  }
  k_channel_abs_mean_f64<<<blocks_for(hw), 256, 0, as_stream(stream)>>>(x, C, hw, A);
  return launch_status();
}

int xnc_apply_scaling_f64(const int32_t* ints, const double* K, double alpha, long n, double* out,
                          void* stream) {
  if (!ints || !K || !out || n < 0) return XNC_EINVAL;
  if (n == 0) return XNC_OK;
  k_apply_scaling_f64<<<blocks_for(n), 256, 0, as_stream(stream)>>>(ints, K, alpha, n, out);
  return launch_status();
}

}  // extern "C"
