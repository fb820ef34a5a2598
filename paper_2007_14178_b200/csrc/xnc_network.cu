// Data-movement kernels around the binary layers of the XNOR-Net AlexNet forward
// (network.py): the max-pools (fused with the ReLU in front of them where the
// network has one) and conv1's pad + space-to-depth.  Pure data movement and
// max selection: the values are exactly those of the torch ops they replace.
#include <algorithm>

#include "xnc_common.cuh"

namespace xnc {

// Max-pool (kernel pk, stride ps, no padding) of every channel plane.  One thread
// per output element in NCHW order, so a warp's window loads are short strided
// spans of the same input rows (L1 serves the 3x3 / 2 overlap).  torch's rule (a
// later element replaces the max when greater, or NaN) in row-major window order,
// so the values are torch.max_pool2d's; relu != 0 applies torch's relu after the
// max (relu(max(w)) == max(relu(w)): the ReLU + pool of conv1 in one pass).
template <int PK>
__global__ void k_max_pool(const float* __restrict__ x, long planes, int C, int Hin, int Win, int Ho, int Wo,
                           int pk_rt, int ps, int relu, const float* __restrict__ bias, float* __restrict__ out) {
  const int pk = PK > 0 ? PK : pk_rt;
  const long total = planes * Ho * Wo;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const long pl = i / (Ho * Wo);
    const int r = (int)(i - pl * (Ho * Wo));
    const int oy = r / Wo, ox = r - oy * Wo;
    const float* b = x + pl * Hin * Win + (oy * ps) * Win + ox * ps;
    float m = __ldg(b);
#pragma unroll
    for (int dy = 0; dy < (PK > 0 ? PK : 8); ++dy) {
      if (PK == 0 && dy >= pk) break;
#pragma unroll
      for (int dx = 0; dx < (PK > 0 ? PK : 8); ++dx) {
        if (PK == 0 && dx >= pk) break;
        const float v = __ldg(b + dy * Win + dx);
        if (v > m || v != v) m = v;
      }
    }
    if (bias != nullptr) m = __fadd_rn(m, __ldg(bias + (int)(pl % C)));  // max(v + b) == max(v) + b
    if (relu && m < 0.0f) m = 0.0f;  // clamp_min(0): NaN and -0.0 pass through
    out[i] = m;
  }
}

// The same pool on channels-last (NHWC) maps, output NHWC: one thread per output
// element with the channel fastest, so window loads and stores are coalesced.
__global__ void k_max_pool_nhwc(const float* __restrict__ x, int C, int Hin, int Win, int Ho, int Wo, int pk,
                                int ps, int relu, int total, const float* __restrict__ bias,
                                float* __restrict__ out) {
  // 32-bit index math (host-checked): 64-bit div/mod made this pass 3x slower
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int c = i % C;
    int t = i / C;
    const int ox = t % Wo;
    t /= Wo;
    const int oy = t % Ho;
    const int n = t / Ho;
    const float* b = x + ((long)(n * Hin + oy * ps) * Win + ox * ps) * C + c;
    float m = __ldg(b);
    for (int dy = 0; dy < pk; ++dy)
      for (int dx = 0; dx < pk; ++dx) {
        const float v = __ldg(b + ((long)dy * Win + dx) * C);
        if (v > m || v != v) m = v;
      }
    if (bias != nullptr) m = __fadd_rn(m, __ldg(bias + c));
    if (relu && m < 0.0f) m = 0.0f;
    out[i] = m;
  }
}

// 4 channels per thread (C % 4 == 0, 16-byte aligned maps): float4 window loads and
// stores, a quarter of the index math per output.
template <int PK>
__global__ void k_max_pool_nhwc4(const float4* __restrict__ x, int C4, int Hin, int Win, int Ho, int Wo, int pk_rt,
                                 int ps, int relu, int total, const float4* __restrict__ bias,
                                 float4* __restrict__ out) {
  // PK > 0: the window loops unroll, so all PK*PK loads are in flight at once (a
  // runtime-bounded loop issued them one round trip at a time: 2 TB/s)
  const int pk = PK > 0 ? PK : pk_rt;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int c = i % C4;
    int t = i / C4;
    const int ox = t % Wo;
    t /= Wo;
    const int oy = t % Ho;
    const int n = t / Ho;
    const float4* b = x + ((long)(n * Hin + oy * ps) * Win + ox * ps) * C4 + c;
    float4 m = __ldg(b);
#pragma unroll
    for (int dy = 0; dy < (PK > 0 ? PK : 8); ++dy) {
      if (PK == 0 && dy >= pk) break;
#pragma unroll
      for (int dx = 0; dx < (PK > 0 ? PK : 8); ++dx) {
        if (PK == 0 && dx >= pk) break;
        const float4 v = __ldg(b + ((long)dy * Win + dx) * C4);
        if (v.x > m.x || v.x != v.x) m.x = v.x;
        if (v.y > m.y || v.y != v.y) m.y = v.y;
        if (v.z > m.z || v.z != v.z) m.z = v.z;
        if (v.w > m.w || v.w != v.w) m.w = v.w;
      }
    }
    if (bias != nullptr) {  // per-channel bias after the max: max(v + b) == max(v) + b exactly
      const float4 b4 = __ldg(bias + c);
      m.x = __fadd_rn(m.x, b4.x); m.y = __fadd_rn(m.y, b4.y); m.z = __fadd_rn(m.z, b4.z); m.w = __fadd_rn(m.w, b4.w);
    }
    if (relu) {
      if (m.x < 0.0f) m.x = 0.0f;
      if (m.y < 0.0f) m.y = 0.0f;
      if (m.z < 0.0f) m.z = 0.0f;
      if (m.w < 0.0f) m.w = 0.0f;
    }
    out[i] = m;
  }
}

int launch_max_pool_nhwc(const float* x, int N, int C, int Hin, int Win, int pk, int ps, int relu,
                         const float* bias, float* out, cudaStream_t s) {
  if (pk < 1 || pk > 8 || ps < 1 || Hin < pk || Win < pk) return XNC_EINVAL;
  const int Ho = (Hin - pk) / ps + 1, Wo = (Win - pk) / ps + 1;
  const long total = (long)N * Ho * Wo * C;
  if (total >= 0x7fffffffL || (long)N * Hin * Win * C >= 0x7fffffffL) return XNC_ENOTSUP;
  if ((C & 3) == 0 &&
      ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(bias)) & 15) == 0) {
    const unsigned blocks = (unsigned)std::min<long>(cdivl(total / 4, 256), 148L * 16);
    auto kern = pk == 3 ? k_max_pool_nhwc4<3> : pk == 2 ? k_max_pool_nhwc4<2> : k_max_pool_nhwc4<0>;
    kern<<<blocks, 256, 0, s>>>(reinterpret_cast<const float4*>(x), C / 4, Hin, Win, Ho, Wo, pk, ps, relu,
                                (int)(total / 4), reinterpret_cast<const float4*>(bias), reinterpret_cast<float4*>(out));
    return launch_status();
  }
  const unsigned blocks = (unsigned)std::min<long>(cdivl(total, 256), 148L * 16);
  k_max_pool_nhwc<<<blocks, 256, 0, s>>>(x, C, Hin, Win, Ho, Wo, pk, ps, relu, (int)total, bias, out);
  return launch_status();
}

int launch_max_pool(const float* x, int N, int C, int Hin, int Win, int pk, int ps, int relu, const float* bias,
                    float* out, cudaStream_t s) {
  if (pk < 1 || pk > 8 || ps < 1 || Hin < pk || Win < pk) return XNC_EINVAL;
  const int Ho = (Hin - pk) / ps + 1, Wo = (Win - pk) / ps + 1;
  const long planes = (long)N * C, total = planes * Ho * Wo;
  const unsigned blocks = (unsigned)std::min<long>(cdivl(total, 256), 148L * 16);
  if (pk == 3)
    k_max_pool<3><<<blocks, 256, 0, s>>>(x, planes, C, Hin, Win, Ho, Wo, pk, ps, relu, bias, out);
  else if (pk == 2)
    k_max_pool<2><<<blocks, 256, 0, s>>>(x, planes, C, Hin, Win, Ho, Wo, pk, ps, relu, bias, out);
  else
    k_max_pool<0><<<blocks, 256, 0, s>>>(x, planes, C, Hin, Win, Ho, Wo, pk, ps, relu, bias, out);
  return launch_status();
}

// Zero pad by p on every side, then space-to-depth by r (torch's F.pad followed by
// F.pixel_unshuffle(., r)): out[n][(c*r + i)*r + j][y][x] = x_pad[n][c][y*r + i][x*r + j],
// out spatial (H + 2p) / r x (W + 2p) / r, stored NCHW or, nhwc != 0, channels-last
// (what cuDNN's fastest conv kernels read).  One pass instead of two copies.  A
// thread takes r consecutive elements of one padded input row and writes one
// element to each of the r output channels j (NCHW: for a fixed j consecutive
// threads write consecutive floats; NHWC: the thread's r outputs are adjacent).
// 32-bit index math (host-checked sizes).
__global__ void k_pad_s2d(const float* __restrict__ x, int C, int H, int W, int p, int r, int Hp, int Ho,
                          int Wo, int total, int nhwc, float* __restrict__ out) {
  const int Co = C * r * r;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int xo = i % Wo;
    int t = i / Wo;
    const int Y = t % Hp;
    t /= Hp;
    const int c = t % C, n = t / C;
    const int yi = Y - p, ii = Y % r, yo = Y / r;
    const bool row_in = yi >= 0 && yi < H;
    const float* src = x + ((long)(n * C + c) * H + (row_in ? yi : 0)) * W;
    const int co0 = (c * r + ii) * r;
    float* dst;
    long jstride;
    if (nhwc) {
      dst = out + (((long)n * Ho + yo) * Wo + xo) * Co + co0;
      jstride = 1;
    } else {
      dst = out + ((long)n * Co + co0) * Ho * Wo + (long)yo * Wo + xo;
      jstride = (long)Ho * Wo;
    }
    for (int j = 0; j < r; ++j) {
      const int xi = xo * r + j - p;
      dst[j * jstride] = (row_in && xi >= 0 && xi < W) ? __ldg(src + xi) : 0.0f;
    }
  }
}

// Channels-last output: one thread per output element in memory order (channel
// fastest), so the stores are fully coalesced; a warp's reads are r-float runs of a
// few input rows that neighbouring pixels share through L1.
__global__ void k_pad_s2d_nhwc(const float* __restrict__ x, int C, int H, int W, int p, int r, int Ho, int Wo,
                               int total, float* __restrict__ out) {
  const int Co = C * r * r;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int co = i % Co;
    int t = i / Co;
    const int xo = t % Wo;
    t /= Wo;
    const int yo = t % Ho, n = t / Ho;
    const int c = co / (r * r), ij = co - c * r * r, ii = ij / r, jj = ij - ii * r;
    const int yi = yo * r + ii - p, xi = xo * r + jj - p;
    out[i] = (yi >= 0 && yi < H && xi >= 0 && xi < W) ? __ldg(x + ((long)(n * C + c) * H + yi) * W + xi) : 0.0f;
  }
}

// r = 4, channels-last: one thread per (n, yo, xo, c) writes its 16 outputs
// (ii, jj) as four 16-byte stores (contiguous across threads with c fastest) from
// four input row segments.
__global__ void k_pad_s2d4_nhwc(const float* __restrict__ x, int C, int H, int W, int p, int Ho, int Wo, int total,
                                float4* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int c = i % C;
    int t = i / C;
    const int xo = t % Wo;
    t /= Wo;
    const int yo = t % Ho, n = t / Ho;
    const float* plane = x + (long)(n * C + c) * H * W;
    float4* o = out + (long)i * 4;  // 16 floats: (ii, jj) of channel c at pixel (yo, xo)
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) {
      const int yi = yo * 4 + ii - p;
      float v[4];
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int xi = xo * 4 + jj - p;
        v[jj] = (yi >= 0 && yi < H && xi >= 0 && xi < W) ? __ldg(plane + (long)yi * W + xi) : 0.0f;
      }
      o[ii] = make_float4(v[0], v[1], v[2], v[3]);
    }
  }
}

int launch_pad_s2d(const float* x, int N, int C, int H, int W, int p, int r, int nhwc, float* out,
                   cudaStream_t s) {
  if (r < 1 || p < 0 || (H + 2 * p) % r || (W + 2 * p) % r) return XNC_EINVAL;
  const int Hp = H + 2 * p, Ho = Hp / r, Wo = (W + 2 * p) / r;
  const long total = (long)N * C * Hp * Wo, out_total = (long)N * C * r * r * Ho * Wo;
  if (total >= 0x7fffffffL || out_total >= 0x7fffffffL) return XNC_ENOTSUP;
  if (nhwc && r == 4 && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
    const long tot = (long)N * C * Ho * Wo;
    const unsigned blocks = (unsigned)std::min<long>(cdivl(tot, 256), 148L * 16);
    k_pad_s2d4_nhwc<<<blocks, 256, 0, s>>>(x, C, H, W, p, Ho, Wo, (int)tot, reinterpret_cast<float4*>(out));
  } else if (nhwc) {
    const unsigned blocks = (unsigned)std::min<long>(cdivl(out_total, 256), 148L * 16);
    k_pad_s2d_nhwc<<<blocks, 256, 0, s>>>(x, C, H, W, p, r, Ho, Wo, (int)out_total, out);
  } else {
    const unsigned blocks = (unsigned)std::min<long>(cdivl(total, 256), 148L * 16);
    k_pad_s2d<<<blocks, 256, 0, s>>>(x, C, H, W, p, r, Hp, Ho, Wo, (int)total, 0, out);
  }
  return launch_status();
}

// The affine of the conv epilogue (y * scale[o] + shift[o], one rounding per op,
// __fmul_rn then __fadd_rn) as a pass over a finished y [N][O][plane]: the popc /
// b1mma kernels' form of the fused tcgen05 out_affine.  One block row per (n, o)
// plane, so the filter index is a block constant.
__global__ void k_plane_affine(float* __restrict__ y, long p0, int O, long plane, const float* __restrict__ scale,
                               const float* __restrict__ shift) {
  const long np = p0 + blockIdx.y;
  const int o = (int)(np % O);
  const float sc = __ldg(scale + o), sh = __ldg(shift + o);
  float* row = y + np * plane;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < plane; i += (long)gridDim.x * blockDim.x)
    row[i] = __fadd_rn(__fmul_rn(row[i], sc), sh);
}

int launch_plane_affine(float* y, int N, int O, long plane, const float* scale, const float* shift,
                        cudaStream_t s) {
  const long planes = (long)N * O;
  if (planes == 0 || plane == 0) return XNC_OK;
  const unsigned gx = (unsigned)std::min<long>(cdivl(plane, 256), 64);
  // planes beyond the 65535 grid rows run as successive launches
  for (long p0 = 0; p0 < planes; p0 += 65535) {
    const unsigned gy = (unsigned)std::min<long>(planes - p0, 65535);
    k_plane_affine<<<dim3(gx, gy), 256, 0, s>>>(y, p0, O, plane, scale, shift);
  }
  return launch_status();
}

}  // namespace xnc
