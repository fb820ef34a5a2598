// K2: K map = zero-padded box filter of A (one per image, shared by all filters).
//
// Reference: xnor_reconstruct keeps kh row-window sums of the padded mean row
// (`_window_row`, _kernels_cy.pyx:231-239: left-to-right adds) and sums them
// top-to-bottom, then multiplies by f32(1/(kh*kw)) (:299-311, :259).  The
// reference recomputes this per (image, filter); here it is computed once per
// image.  Float op order is reproduced exactly, so K is bit-identical.
//
// Shared-memory halo tile: a block of 32 x 8 outputs stages the
// (8+kh-1) x (32+kw-1) window of A (zeros outside the image) in smem, forms the
// row sums in smem, then the column sums.
#include "xnc_common.cuh"

namespace xnc {

constexpr int kScTX = 32, kScTY = 8;

__global__ void __launch_bounds__(kScTX * kScTY) k_scale_map(const float* __restrict__ A, int H,
                                                            int W, int kh, int kw, int pad,
                                                            int oh, int ow, float box,
                                                            float* __restrict__ K) {
  __shared__ float m_s[kScTY + kMaxK - 1][kScTX + kMaxK];
  __shared__ float r_s[kScTY + kMaxK - 1][kScTX + 1];
  const int n = blockIdx.z;
  const int x0 = blockIdx.x * kScTX, y0 = blockIdx.y * kScTY;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int rows = kScTY + kh - 1, cols = kScTX + kw - 1;
  const float* a = A + (long)n * H * W;
  for (int r = ty; r < rows; r += kScTY)
    for (int c = tx; c < cols; c += kScTX) {
      int iy = y0 + r - pad, ix = x0 + c - pad;
      m_s[r][c] = (iy >= 0 && iy < H && ix >= 0 && ix < W) ? a[(long)iy * W + ix] : 0.0f;
    }
  __syncthreads();
  for (int r = ty; r < rows; r += kScTY) {
    float acc = 0.0f;
    for (int d = 0; d < kw; ++d) acc = __fadd_rn(acc, m_s[r][tx + d]);
    r_s[r][tx] = acc;
  }
  __syncthreads();
  const int y = y0 + ty, x = x0 + tx;
  if (y < oh && x < ow) {
    float acc = r_s[ty][tx];
    for (int d = 1; d < kh; ++d) acc = __fadd_rn(acc, r_s[ty + d][tx]);
    K[((long)n * oh + y) * ow + x] = __fmul_rn(acc, box);
  }
}

// Band form: one block per (image, band of BY full-width output rows).  The 32 x 8
// tiles above spend most of their time on block start-up and halo loads (C3: 3584
// blocks of 256 one-output threads, 0.014 ms for 6.4 MB); a band stages its
// (BY+kh-1) x (ow+kw-1) padded window once with coalesced row loads, and each
// thread forms several outputs.  Same op order, so the same bits.
#ifndef XNC_K2_BLOCKS_PER_SM
#define XNC_K2_BLOCKS_PER_SM 2
#endif
constexpr int kBandThreads = 256;
constexpr size_t kBandSmemMax = 48 * 1024;

__global__ void __launch_bounds__(kBandThreads) k_scale_map_band(const float* __restrict__ A, int H, int W,
                                                                  int kh, int kw, int pad, int oh, int ow,
                                                                  int BY, float box, float* __restrict__ K) {
  extern __shared__ float band_s[];
  pdl_launch_dependents();  // one short wave: the next kernel (the conv) may start its prologue
  pdl_wait();  // A is the previous kernel's output
  const int n = blockIdx.y, y0 = blockIdx.x * BY;
  const int by = min(BY, oh - y0);
  const int rows = by + kh - 1, cols = ow + kw - 1;
  float* m_s = band_s;                 // rows x cols padded A
  float* r_s = band_s + rows * cols;   // rows x ow row-window sums
  const float* a = A + (long)n * H * W;
  // eight loads in flight per thread before any smem store (one at a time, a
  // thread's dozen loads are a dozen DRAM round trips)
  constexpr int kU = 8;
  for (int i0 = threadIdx.x; i0 < rows * cols; i0 += kBandThreads * kU) {
    float v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = i0 + u * kBandThreads;
      const int r = i / cols, c = i - r * cols;
      const int iy = y0 + r - pad, ix = c - pad;
      v[u] = (i < rows * cols && iy >= 0 && iy < H && ix >= 0 && ix < W) ? __ldg(a + (long)iy * W + ix) : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (i0 + u * kBandThreads < rows * cols) m_s[i0 + u * kBandThreads] = v[u];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < rows * ow; i += kBandThreads) {
    const int r = i / ow, x = i - r * ow;
    const float* m = m_s + r * cols + x;
    float acc = 0.0f;
    for (int d = 0; d < kw; ++d) acc = __fadd_rn(acc, m[d]);
    r_s[i] = acc;
  }
  __syncthreads();
  float* k_out = K + ((long)n * oh + y0) * ow;
  for (int i = threadIdx.x; i < by * ow; i += kBandThreads) {
    float acc = r_s[i];
    for (int d = 1; d < kh; ++d) acc = __fadd_rn(acc, r_s[i + d * ow]);
    k_out[i] = __fmul_rn(acc, box);
  }
}

int launch_scale_map(const float* A, int N, int H, int W, int kh, int kw, int pad, float* K,
                     cudaStream_t s) {
  const int oh = H + 2 * pad - kh + 1, ow = W + 2 * pad - kw + 1;
  const float box = (float)(1.0 / (double)(kh * kw));  // <real_t> scale, _kernels_cy.pyx:259
  if (oh <= 0 || ow <= 0 || N <= 0) return launch_status();
  {
    // bands: about two blocks per SM over the batch, as few halo rows as that allows
    // (ncu, C3: 2 per SM 8.4 us, 4: 9.7, 8: 10.8, 16: 14.9; the 32 x 8 tiles 11.1)
    const int target = XNC_K2_BLOCKS_PER_SM * 148;
    int bands = N >= target ? 1 : (target + N - 1) / N;
    int BY = (oh + (bands < oh ? bands : oh) - 1) / (bands < oh ? bands : oh);
    auto smem_of = [&](int by) { return (size_t)(by + kh - 1) * ((ow + kw - 1) + ow) * sizeof(float); };
    while (BY > 1 && smem_of(BY) > kBandSmemMax) BY = (BY + 1) / 2;
    if (smem_of(BY) <= kBandSmemMax) {
      dim3 grid(cdiv(oh, BY), N);
      launch_pdl(k_scale_map_band, grid, dim3(kBandThreads), smem_of(BY), s, A, H, W, kh, kw, pad, oh, ow, BY, box, K);
      return launch_status();
    }
  }
  // very wide maps: 32 x 8 tiles
  dim3 grid(cdiv(ow, kScTX), cdiv(oh, kScTY), N);
  k_scale_map<<<grid, dim3(kScTX, kScTY), 0, s>>>(A, H, W, kh, kw, pad, oh, ow, box, K);
  return launch_status();
}

}  // namespace xnc
