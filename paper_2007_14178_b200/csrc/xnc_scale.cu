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

int launch_scale_map(const float* A, int N, int H, int W, int kh, int kw, int pad, float* K,
                     cudaStream_t s) {
  const int oh = H + 2 * pad - kh + 1, ow = W + 2 * pad - kw + 1;
  const float box = (float)(1.0 / (double)(kh * kw));  // <real_t> scale, _kernels_cy.pyx:259
  dim3 grid(cdiv(ow, kScTX), cdiv(oh, kScTY), N);
  k_scale_map<<<grid, dim3(kScTX, kScTY), 0, s>>>(A, H, W, kh, kw, pad, oh, ow, box, K);
  return launch_status();
}

}  // namespace xnc
