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
#include <algorithm>
#include <type_traits>

#include "xnc_common.cuh"

namespace xnc {

// Kernel K1.  Block = 256 threads x VEC consecutive pixels (linear pixel index
// q = n*HW + p, contiguous for the whole block because HW % VEC == 0).
// Phase 1: each thread walks the C channels of its pixels (16-byte coalesced
// loads, x read once), builds one 32-channel word per pixel per j and the A
// sum, and parks the words in shared memory as [j][pixel] (16-byte stores).
// Phase 2: the block writes the bits [q][Cw] from shared memory with
// consecutive lanes on consecutive words (coalesced warp stores).  Every conv
// kernel (popc, b1 mma.sync and the tcgen05 pair kernel, which expands the
// bits to its byte operand in shared memory) reads this one format.
#ifndef XNC_PACK_THREADS
#define XNC_PACK_THREADS 128  // sweep (tools/pack_sweep.py, explicit 8-deep loads): 128 = 6.6 TB/s at C3, 256 = 6.5, 512 = 5.7
#endif
#ifndef XNC_PACK_UNROLL
#define XNC_PACK_UNROLL 8
#endif
constexpr int kPackThreads = XNC_PACK_THREADS;  // preferred block size (smaller if smem is short)
constexpr int kPackUnroll = XNC_PACK_UNROLL;  // channel loads in flight per thread
#ifndef XNC_ABS_BATCH
#define XNC_ABS_BATCH 8  // k_absmean: channel loads issued per batch (16/32/64 measured slower)
#endif

template <int VEC, int THREADS, bool AFF>
__global__ void __launch_bounds__(THREADS) k_pack_input(const float* __restrict__ x, int C, int HW,
                                                             int Cw, float inv, long groups_per_img,
                                                             long total_groups,
                                                             uint32_t* __restrict__ bits,
                                                             float* __restrict__ A,
                                                             const float* __restrict__ in_scale,
                                                             const float* __restrict__ in_shift) {
  extern __shared__ uint4 pack_smem[];
  pdl_wait();  // x may be the previous kernel's output
  uint32_t* wtile = reinterpret_cast<uint32_t*>(pack_smem);
  constexpr int PIX = THREADS * VEC;          // pixels per block
  constexpr int JS = PIX + 4;                 // word-plane stride (bank skew, keeps 16 B alignment)
  const long gid0 = (long)blockIdx.x * THREADS;
  const long gid = gid0 + threadIdx.x;
  const long q0 = gid0 * VEC;                 // first linear pixel of the block
  const long q_end = total_groups * VEC;
  if (gid < total_groups) {
    const long n = gid / groups_per_img;
    const int p0 = (int)(gid - n * groups_per_img) * VEC;
    const float* xp = x + (long)n * C * HW + p0;
    float s[VEC];
#pragma unroll
    for (int i = 0; i < VEC; ++i) s[i] = 0.0f;
    for (int j = 0; j < Cw; ++j) {
      uint32_t word[VEC];
#pragma unroll
      for (int i = 0; i < VEC; ++i) word[i] = 0u;
      const int cend = min(32, C - 32 * j);
      // kPackUnroll channel loads are issued before any is consumed (written out
      // explicitly: left to the compiler, the streaming loads were issued one at a
      // time, each right before its use, and K1 ran at ~80% of the HBM read rate)
      for (int c0 = 0; c0 < cend; c0 += kPackUnroll) {
        float v[kPackUnroll][VEC];
#pragma unroll
        for (int u = 0; u < kPackUnroll; ++u) {
          const float* src = xp + (long)(32 * j + c0 + u) * HW;
          if (c0 + u < cend) {
            if constexpr (VEC == 4) {
              const float4 t = __ldcs(reinterpret_cast<const float4*>(src));  // streamed once
              v[u][0] = t.x; v[u][1] = t.y; v[u][2] = t.z; v[u][3] = t.w;
            } else {
#pragma unroll
              for (int i = 0; i < VEC; ++i) v[u][i] = __ldcs(src + i);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < kPackUnroll; ++u) {
          if (c0 + u < cend) {
            const int cc = c0 + u;
            if constexpr (AFF) {  // per-channel affine (folded BN) before sign and |.|
              const float sc = __ldg(in_scale + 32 * j + cc), sh = __ldg(in_shift + 32 * j + cc);
#pragma unroll
              for (int i = 0; i < VEC; ++i) v[u][i] = __fadd_rn(__fmul_rn(v[u][i], sc), sh);
            }
#pragma unroll
            for (int i = 0; i < VEC; ++i) {
              s[i] = __fadd_rn(s[i], fabsf(v[u][i]));
              word[i] |= (v[u][i] >= 0.0f ? 1u : 0u) << cc;
            }
          }
        }
      }
      if constexpr (VEC == 4) {
        *reinterpret_cast<uint4*>(wtile + j * JS + threadIdx.x * 4) = make_uint4(word[0], word[1], word[2], word[3]);
      } else {
        wtile[j * JS + threadIdx.x] = word[0];
      }
    }
    if (A != nullptr) {
      float* ap = A + (long)n * HW + p0;
      if constexpr (VEC == 4) {
        *reinterpret_cast<float4*>(ap) = make_float4(__fmul_rn(s[0], inv), __fmul_rn(s[1], inv),
                                                     __fmul_rn(s[2], inv), __fmul_rn(s[3], inv));
      } else {
        ap[0] = __fmul_rn(s[0], inv);
      }
    }
  }
  __syncthreads();
  const int npix = (int)min((long)PIX, q_end - q0);
  if (bits != nullptr) {
    uint32_t* bp = bits + q0 * Cw;
    for (int idx = threadIdx.x; idx < npix * Cw; idx += THREADS) {
      const int px = idx / Cw, j = idx - px * Cw;
      bp[idx] = wtile[j * JS + px];
    }
  }
}

// Small-image path (few pixels, many channels: 13x13 conv3-5 inputs, the 6x6
// fc6 input, the 1x1 fc7 input): the per-pixel kernel above would run one
// thread per pixel over thousands of channels on a fraction of the SMs.  Here
// the words are built by one thread per (pixel, word) and A by one thread per
// pixel (the channel sum must stay sequential for bit-exactness); x is read
// twice, from L2 for these sizes.
__device__ __forceinline__ float affine_in(float v, const float* sc, const float* sh, int c) {
  return sc != nullptr ? __fadd_rn(__fmul_rn(v, __ldg(sc + c)), __ldg(sh + c)) : v;
}

__global__ void k_pack_words(const float* __restrict__ x, int C, int HW, int Cw, long npix,
                             uint32_t* __restrict__ bits, const float* __restrict__ in_scale,
                             const float* __restrict__ in_shift) {
  const long tid = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= npix * Cw) return;
  long q;
  int j;
  if (HW >= 32) {  // pixels fastest: coalesced NCHW reads across the warp
    j = (int)(tid / npix);
    q = tid - (long)j * npix;
  } else {         // words fastest: each thread reads 32 nearby channels
    q = tid / Cw;
    j = (int)(tid - q * Cw);
  }
  const long n = q / HW, p = q - n * HW;
  const float* xp = x + (n * C + 32L * j) * HW + p;
  const int cend = min(32, C - 32 * j);
  float v[32];  // all 32 loads in flight before the compares
#pragma unroll
  for (int cc = 0; cc < 32; ++cc) v[cc] = cc < cend ? __ldg(xp + (long)cc * HW) : 0.0f;
  uint32_t word = 0u;
#pragma unroll
  for (int cc = 0; cc < 32; ++cc)
    if (cc < cend) word |= (affine_in(v[cc], in_scale, in_shift, 32 * j + cc) >= 0.0f ? 1u : 0u) << cc;
  bits[q * Cw + j] = word;
}

__global__ void k_absmean(const float* __restrict__ x, int C, int HW, long npix, float inv,
                          float* __restrict__ A, const float* __restrict__ in_scale,
                          const float* __restrict__ in_shift) {
  const long q = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= npix) return;
  const long n = q / HW, p = q - n * HW;
  const float* xp = x + n * C * (long)HW + p;
  float s = 0.0f;
  // The sum is one sequential f32 chain per pixel (bit-exactness), so the loads
  // are issued in batches of 8 ahead of the adds.
  if (HW == 1 && (C & 31) == 0 && ((reinterpret_cast<uintptr_t>(xp) & 15) == 0) && in_scale == nullptr) {
    for (int c = 0; c < C; c += 32) {  // channels contiguous: 16-byte loads, same sequential order
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldg(reinterpret_cast<const float4*>(xp + c) + u);
#pragma unroll
      for (int u = 0; u < 8; ++u)
        s = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(s, fabsf(v[u].x)), fabsf(v[u].y)), fabsf(v[u].z)), fabsf(v[u].w));
    }
  } else {
    // batches of kB channel loads ahead of the sequential adds
    constexpr int kB = XNC_ABS_BATCH;
    int c = 0;
    for (; c + kB <= C; c += kB) {
      float v[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) v[u] = __ldg(xp + (long)(c + u) * HW);
#pragma unroll
      for (int u = 0; u < kB; ++u) s = __fadd_rn(s, fabsf(affine_in(v[u], in_scale, in_shift, c + u)));
    }
    for (; c < C; ++c) s = __fadd_rn(s, fabsf(affine_in(__ldg(xp + (long)c * HW), in_scale, in_shift, c)));
  }
  A[q] = __fmul_rn(s, inv);
}

// K1 for few-pixel maps with up to 768 channels (the 13x13 / 6x6 inputs of conv3-5
// and fc6): a block stages 32 consecutive pixels x all C channels in shared memory
// (four warps issue the coalesced 128-byte loads, the folded BN applied on the
// way in), then warp 0 runs each pixel's sequential |.| chain from shared memory
// while warps 1-3 build the sign words.  x is read once; the per-word and
// per-pixel kernels read it twice and the per-pixel chain waited out a memory
// round trip per 8 channels (conv4's input: 76 -> ~20 us).
constexpr int kSmallMaxC = 768;
template <bool AFF>
__global__ void __launch_bounds__(128) k_pack_small(const float* __restrict__ x, int C, int HW, int Cw, long npix,
                                                    float inv, uint32_t* __restrict__ bits, float* __restrict__ A,
                                                    const float* __restrict__ in_scale,
                                                    const float* __restrict__ in_shift) {
  extern __shared__ float tile[];  // [C][32]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long q = (long)blockIdx.x * 32 + lane;
  const bool in = q < npix;
  const long n = in ? q / HW : 0, p = in ? q - n * HW : 0;
  const float* xp = x + n * C * (long)HW + p;
  // 16 channel loads in flight per thread before any store (a load -> store loop
  // waited out one memory latency per channel)
  constexpr int kU = 16;
  for (int c0 = warp; c0 < C; c0 += 4 * kU) {
    float v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int c = c0 + 4 * u;
      v[u] = (in && c < C) ? __ldg(xp + (long)c * HW) : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int c = c0 + 4 * u;
      if (c < C) {
        float t = v[u];
        if (AFF) t = __fadd_rn(__fmul_rn(t, __ldg(in_scale + c)), __ldg(in_shift + c));
        tile[c * 32 + lane] = t;
      }
    }
  }
  __syncthreads();
  if (!in) return;
  if (warp == 0) {
    // sequential chain per pixel; the next 16 channels' LDS issued before this 16's adds
    float s = 0.0f;
    float cur[16], nxt[16];
    const int nb = C >> 4;
#pragma unroll
    for (int u = 0; u < 16; ++u) cur[u] = nb > 0 ? tile[u * 32 + lane] : 0.0f;
    for (int k = 0; k < nb; ++k) {
      if (k + 1 < nb) {
#pragma unroll
        for (int u = 0; u < 16; ++u) nxt[u] = tile[((k + 1) * 16 + u) * 32 + lane];
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) s = __fadd_rn(s, fabsf(cur[u]));
#pragma unroll
      for (int u = 0; u < 16; ++u) cur[u] = nxt[u];
    }
    for (int c = nb << 4; c < C; ++c) s = __fadd_rn(s, fabsf(tile[c * 32 + lane]));
    if (A) A[q] = __fmul_rn(s, inv);
  } else {
    for (int j = warp - 1; j < Cw; j += 3) {
      const int cend = min(32, C - 32 * j);
      uint32_t word = 0u;
#pragma unroll 8
      for (int u = 0; u < cend; ++u) word |= (tile[(32 * j + u) * 32 + lane] >= 0.0f ? 1u : 0u) << u;
      bits[q * Cw + j] = word;
    }
  }
}

// max-pool step in xnc_max_pool's order and rule: a later value wins when it
// is larger or NaN (so a window's result is its last NaN, else its maximum)
__device__ __forceinline__ float pool_pick(float m, float v) { return (v > m || v != v) ? v : m; }

// K1 of a max-pooled map without materialising it (XNOR-Net's pool -> BN -> sign in
// front of conv3 and fc6): x is the PRE-pool map [N][C][Hin][Win]; the value staged
// for (channel c, pooled pixel (oy, ox)) is the max over its pk x pk window at
// stride ps with xnc_max_pool's rule (row-major window order, NaN propagates), then
// the optional affine -- exactly K1 of xnc_max_pool's output.  Otherwise the block
// is k_pack_small: 32 pooled pixels x all C channels in shared memory, warp 0 runs
// the sequential |.| chains, warps 1-3 the sign words.  Saves the pooled map's
// write and re-read and one launch.
#ifndef XNC_POOL_KU
#define XNC_POOL_KU 6  // 2 / 4 / 6 / 8: conv3's input 81 / 73 / 64 / 73 us at batch 256 (tools/pool_probe.py)
#endif
// NW warps per block (4; 8 when the grid is under two blocks per SM -- fc6's input at
// batch 256 is 288 blocks: each warp's channel loop is half as long)
template <bool AFF, int PK, int NW>
__global__ void __launch_bounds__(NW * 32) k_pack_small_pool(const float* __restrict__ x, int C, int Hin, int Win,
                                                         int Ho, int Wo, int ps, int Cw, long npix, float inv,
                                                         uint32_t* __restrict__ bits, float* __restrict__ A,
                                                         const float* __restrict__ in_scale,
                                                         const float* __restrict__ in_shift) {
  extern __shared__ float tile[];  // [C][32]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long q = (long)blockIdx.x * 32 + lane;
  const bool in = q < npix;
  const int HWo = Ho * Wo;
  const long n = in ? q / HWo : 0;
  const int p = in ? (int)(q - n * HWo) : 0;
  const int oy = p / Wo, ox = p - (p / Wo) * Wo;
  const float* xp = x + n * C * (long)Hin * Win + (long)(oy * ps) * Win + ox * ps;
  const long plane = (long)Hin * Win;
  constexpr int kU = XNC_POOL_KU;  // channels per thread per batch: kU * PK * PK loads in flight
  for (int c0 = warp; c0 < C; c0 += NW * kU) {
    float v[kU][PK * PK], sc[kU], sh[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int c = c0 + NW * u;
      const float* b = xp + (long)c * plane;
#pragma unroll
      for (int dy = 0; dy < PK; ++dy)
#pragma unroll
        for (int dx = 0; dx < PK; ++dx) v[u][dy * PK + dx] = (in && c < C) ? __ldg(b + dy * Win + dx) : 0.0f;
      // the affine's constants in the same batch of loads (loaded after the window
      // values were used, each was another memory round trip: ncu's top stall)
      sc[u] = (AFF && c < C) ? __ldg(in_scale + c) : 1.0f;
      sh[u] = (AFF && c < C) ? __ldg(in_shift + c) : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int c = c0 + NW * u;
      if (c < C) {
        float m = v[u][0];
#pragma unroll
        for (int k = 1; k < PK * PK; ++k) m = pool_pick(m, v[u][k]);
        if (AFF) m = __fadd_rn(__fmul_rn(m, sc[u]), sh[u]);
        tile[c * 32 + lane] = m;
      }
    }
  }
  __syncthreads();
  if (!in) return;
  if (warp == 0) {
    float s = 0.0f;
    float cur[16], nxt[16];
    const int nb = C >> 4;
#pragma unroll
    for (int u = 0; u < 16; ++u) cur[u] = nb > 0 ? tile[u * 32 + lane] : 0.0f;
    for (int k = 0; k < nb; ++k) {
      if (k + 1 < nb) {
#pragma unroll
        for (int u = 0; u < 16; ++u) nxt[u] = tile[((k + 1) * 16 + u) * 32 + lane];
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) s = __fadd_rn(s, fabsf(cur[u]));
#pragma unroll
      for (int u = 0; u < 16; ++u) cur[u] = nxt[u];
    }
    for (int c = nb << 4; c < C; ++c) s = __fadd_rn(s, fabsf(tile[c * 32 + lane]));
    if (A) A[q] = __fmul_rn(s, inv);
  } else {
    for (int j = warp - 1; j < Cw; j += NW - 1) {
      const int cend = min(32, C - 32 * j);
      uint32_t word = 0u;
#pragma unroll 8
      for (int u = 0; u < cend; ++u) word |= (tile[(32 * j + u) * 32 + lane] >= 0.0f ? 1u : 0u) << u;
      bits[q * Cw + j] = word;
    }
  }
}

// xnc_pack_input_pool: the fused form when the pooled map takes the small-map path
// (>= 32 pooled pixels per image, C <= kSmallMaxC) and the window is 3 x 3;
// XNC_ENOTSUP otherwise (the caller pools, then packs).
int launch_pack_input_pool(const float* x, int N, int C, int Hin, int Win, int pk, int ps, uint32_t* bits,
                           float* A, cudaStream_t s, const float* in_scale, const float* in_shift) {
  if (pk != 3 || ps < 1 || Hin < pk || Win < pk) return XNC_ENOTSUP;
  const int Ho = (Hin - pk) / ps + 1, Wo = (Win - pk) / ps + 1;
  const long npix = (long)N * Ho * Wo;
  if (Ho * Wo < 32 || C < 32 || C > kSmallMaxC) return XNC_ENOTSUP;
  const int Cw = cdiv(C, 32);
  const size_t sm = (size_t)C * 32 * sizeof(float);
  const bool wide = cdivl(npix, 32) < 2L * device_sm_count();
  auto kern = wide ? (in_scale ? k_pack_small_pool<true, 3, 8> : k_pack_small_pool<false, 3, 8>)
                   : (in_scale ? k_pack_small_pool<true, 3, 4> : k_pack_small_pool<false, 3, 4>);
  if (int rc = smem_opt_in(kern, sm)) return rc;  // per device (xnc_runtime.cu)
  kern<<<(unsigned)cdivl(npix, 32), wide ? 256 : 128, sm, s>>>(x, C, Hin, Win, Ho, Wo, ps, Cw, npix, (float)(1.0 / (double)C),
                                                  bits, A, in_scale, in_shift);
  return launch_status();
}

// K1 of xnc_max_pool_nhwc's output fused with the pool (the network's front end:
// conv1's channels-last map -> max 3 x 3 / ps -> + bias -> ReLU -> conv2's folded BN
// -> sign / A).  Laid out like the pool kernel (a thread per 4 channels of one pooled
// pixel, nine float4 window loads, coalesced along the channels, many warps in flight:
// that pass runs at HBM speed); a block takes npx = 384 / (C/4) pooled pixels x C/4
// threads (16 at conv2's 96 channels), at most 42 registers so that four blocks share
// an SM (one block of 384 threads per 46-register SM slot ran 93-108 us, four 83 us at
// batch 256, tools/pool_probe.py).  The pool's rule in window order, its bias and ReLU,
// then the affine as K1 applies it; the sign nibbles are OR-reduced over 8-thread groups
// (one 32-channel word each: C % 32 == 0, so groups never straddle pixels or warps) and
// the values staged [C][npx + 1] for the per-pixel sequential |.| chains.  Saves the
// pooled map's write and re-read (72 MB at batch 256) and one launch.
constexpr int kPoolThreads = 384;
// NPX > 0: the pixel count (and C = 4 * 384 / NPX) fixed at compile time -- conv2's 96
// channels (16 pixels; 83 vs 87 us with the runtime form)
template <bool AFF, int NPX>
__global__ void __launch_bounds__(kPoolThreads, 4) k_pool_pack_nhwc(const float4* __restrict__ x, int C_rt, int Hin,
                                                                   int Win, int Ho, int Wo, int ps, int relu,
                                                                   const float* __restrict__ bias, long npix,
                                                                   int npx_rt, float inv, uint32_t* __restrict__ bits,
                                                                   float* __restrict__ A,
                                                                   const float* __restrict__ in_scale,
                                                                   const float* __restrict__ in_shift) {
  extern __shared__ float tile[];  // [C][npx + 1]
  const int npx = NPX > 0 ? NPX : npx_rt;
  const int C = NPX > 0 ? 4 * kPoolThreads / NPX : C_rt;
  const int ld = npx + 1;
  const int C4 = C >> 2, Cw = C >> 5;
  const int t = threadIdx.x, lane = t & 31;
  const int px = t / C4, c4 = t - px * C4;
  const long q = (long)blockIdx.x * npx + px;  // blockDim = (C/4) * npx: px < npx
  const bool in = q < npix;
  uint32_t nib = 0u;
  if (in) {
    const int HWo = Ho * Wo;
    const int n = (int)(q / HWo), p = (int)(q - (long)n * HWo);
    const int oy = p / Wo, ox = p - (p / Wo) * Wo;
    const float4* b = x + ((size_t)(n * Hin + oy * ps) * Win + ox * ps) * C4 + c4;
    float4 w[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) w[k] = __ldg(b + ((size_t)(k / 3) * Win + (k % 3)) * C4);
    float4 m = w[0];
#pragma unroll
    for (int k = 1; k < 9; ++k) {
      m.x = pool_pick(m.x, w[k].x); m.y = pool_pick(m.y, w[k].y);
      m.z = pool_pick(m.z, w[k].z); m.w = pool_pick(m.w, w[k].w);
    }
    float v[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = 4 * c4 + u;
      if (bias != nullptr) v[u] = __fadd_rn(v[u], __ldg(bias + c));
      if (relu && v[u] < 0.0f) v[u] = 0.0f;
      if (AFF) v[u] = __fadd_rn(__fmul_rn(v[u], __ldg(in_scale + c)), __ldg(in_shift + c));
      tile[c * ld + px] = v[u];
      nib |= (v[u] >= 0.0f ? 1u : 0u) << u;
    }
  }
  // 32-channel word = 8 consecutive threads (c4 = 8j .. 8j + 7 of one pixel)
  uint32_t wv = nib << (4 * (lane & 7));
  wv |= __shfl_xor_sync(0xffffffffu, wv, 1);
  wv |= __shfl_xor_sync(0xffffffffu, wv, 2);
  wv |= __shfl_xor_sync(0xffffffffu, wv, 4);
  if (in && (c4 & 7) == 0) bits[q * Cw + (c4 >> 3)] = wv;
  __syncthreads();
  if (t < npx && A != nullptr) {
    const long qa = (long)blockIdx.x * npx + t;
    if (qa < npix) {
      float s = 0.0f;
      int c = 0;
      for (; c + 8 <= C; c += 8) {
        float tv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) tv[u] = tile[(c + u) * ld + t];
#pragma unroll
        for (int u = 0; u < 8; ++u) s = __fadd_rn(s, fabsf(tv[u]));
      }
      for (; c < C; ++c) s = __fadd_rn(s, fabsf(tile[c * ld + t]));
      A[qa] = __fmul_rn(s, inv);
    }
  }
}

int launch_pack_input_pool_nhwc(const float* x, int N, int C, int Hin, int Win, int pk, int ps, int relu,
                                const float* bias, uint32_t* bits, float* A, cudaStream_t s, const float* in_scale,
                                const float* in_shift) {
  if (pk != 3 || ps < 1 || Hin < pk || Win < pk) return XNC_ENOTSUP;
  if ((C & 31) != 0 || C / 4 > kPoolThreads || (reinterpret_cast<uintptr_t>(x) & 15) != 0) return XNC_ENOTSUP;
  const int npx = kPoolThreads / (C / 4);
  const int Ho = (Hin - pk) / ps + 1, Wo = (Win - pk) / ps + 1;
  const long npix = (long)N * Ho * Wo;
  if ((long)N * Hin * Win * C >= 0x7fffffffL * 4L) return XNC_ENOTSUP;
  const size_t sm = (size_t)C * (npx + 1) * sizeof(float);
  auto kern = C == 96 ? (in_scale ? k_pool_pack_nhwc<true, 16> : k_pool_pack_nhwc<false, 16>)
                      : (in_scale ? k_pool_pack_nhwc<true, 0> : k_pool_pack_nhwc<false, 0>);
  if (int rc = smem_opt_in(kern, sm)) return rc;
  kern<<<(unsigned)cdivl(npix, npx), (C / 4) * npx, sm, s>>>(reinterpret_cast<const float4*>(x), C, Hin, Win, Ho, Wo,
                                                             ps, relu, bias, npix, npx, (float)(1.0 / (double)C), bits,
                                                             A, in_scale, in_shift);
  return launch_status();
}

// A for 1x1 images with long channel vectors (the fc7 input, 4096 channels): the
// sum is one sequential chain per pixel, so one thread per pixel left all but a
// couple of SMs idle and waited out a memory latency per few channels.  Here a
// warp per pixel streams 1024-channel chunks into shared memory (the next chunk's
// loads in flight while lane 0 runs the chain over the current one, in channel
// order; the folded BN, if any, is applied by the loading lanes, the same two
// roundings).
constexpr int kAbsChunk = 1024;
constexpr int kAbsWideMax = 4096;  // channels staged whole per warp (16 KB)
__global__ void __launch_bounds__(128) k_absmean_wide(const float* __restrict__ x, int C, long npix, float inv,
                                                      float* __restrict__ A, const float* __restrict__ in_scale,
                                                      const float* __restrict__ in_shift) {
  // The pixel's whole channel vector is staged first (all lanes' loads, chunk after
  // chunk, no chain in between), then lane 0 runs the one sequential chain with its
  // shared-memory reads a batch ahead.  Interleaving per 1024-channel chunk made
  // the warp wait out a load latency per chunk on top of the chain (ncu: 70 %
  // long-scoreboard stalls, 50 us for fc7's 256 x 4096 input).
  extern __shared__ __align__(16) float absw_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long q = (long)blockIdx.x * 4 + warp;
  if (q >= npix) return;
  const float* xp = x + q * C;
  float* b = absw_smem + (size_t)warp * C;
  for (int c0 = 0; c0 < C; c0 += kAbsChunk) {
    const int n = min(kAbsChunk, C - c0);
    // the chunk's 32 loads per lane are all issued before any is used: with the
    // optional affine's loads interleaved the compiler issued them one at a time and
    // the warp waited out 32 load latencies per chunk (ncu: 70 % long-scoreboard
    // stalls on the first use; 57 us for fc7's 256 x 4096 input)
    float v[kAbsChunk / 32];
#pragma unroll
    for (int u = 0; u < kAbsChunk / 32; ++u) {
      const int c = u * 32 + lane;
      v[u] = c < n ? __ldg(xp + c0 + c) : 0.0f;
    }
    if (in_scale != nullptr) {
#pragma unroll
      for (int u = 0; u < kAbsChunk / 32; ++u) {
        const int c = c0 + u * 32 + lane;
        if (u * 32 + lane < n) v[u] = __fadd_rn(__fmul_rn(v[u], __ldg(in_scale + c)), __ldg(in_shift + c));
      }
    }
#pragma unroll
    for (int u = 0; u < kAbsChunk / 32; ++u)
      if (u * 32 + lane < n) b[c0 + u * 32 + lane] = fabsf(v[u]);
  }
  __syncwarp();
  if (lane == 0) {
    float s = 0.0f;
    const float4* b4 = reinterpret_cast<const float4*>(b);
    const int nb = C >> 5;  // whole 32-channel batches
    float4 cur[8], nxt[8];
    if (nb > 0) {
#pragma unroll
      for (int u = 0; u < 8; ++u) cur[u] = b4[u];
    }
    for (int k = 0; k < nb; ++k) {
      if (k + 1 < nb) {
#pragma unroll
        for (int u = 0; u < 8; ++u) nxt[u] = b4[(k + 1) * 8 + u];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        s = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(s, cur[u].x), cur[u].y), cur[u].z), cur[u].w);
#pragma unroll
      for (int u = 0; u < 8; ++u) cur[u] = nxt[u];
    }
    for (int i = nb << 5; i < C; ++i) s = __fadd_rn(s, b[i]);
    A[q] = __fmul_rn(s, inv);
  }
}

// K1 of 1 x 1 images with long channel vectors (fc7's 4096-channel input) in ONE
// pass: per pixel a loader warp streams the vector in 1024-channel chunks into
// shared memory and emits the sign words with ballots (bit = lane), while lane 0 of
// a chain warp runs the sequential |.| sum over each chunk as soon as it is staged
// (bar.arrive / bar.sync handshake per chunk).  Replaces k_pack_words +
// k_absmean_wide (x read once instead of twice; the chain overlaps the loads).
__global__ void __launch_bounds__(64) k_pack_wide(const float* __restrict__ x, int C, float inv,
                                                  uint32_t* __restrict__ bits, float* __restrict__ A,
                                                  const float* __restrict__ in_scale,
                                                  const float* __restrict__ in_shift) {
  extern __shared__ __align__(16) float wide_s[];  // [C] |x'|
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long q = blockIdx.x;
  const int Cw = C >> 5;
  const int nchunk = (C + kAbsChunk - 1) / kAbsChunk;  // <= 4 (host-checked C <= kAbsWideMax)
  if (warp == 0) {
    const float* xp = x + q * C;
    for (int k = 0; k < nchunk; ++k) {
      const int c0 = k * kAbsChunk, n = min(kAbsChunk, C - c0);  // n % 32 == 0
      float v[kAbsChunk / 32];
#pragma unroll
      for (int u = 0; u < kAbsChunk / 32; ++u) v[u] = u * 32 < n ? __ldg(xp + c0 + u * 32 + lane) : 0.0f;
      if (in_scale != nullptr) {
#pragma unroll
        for (int u = 0; u < kAbsChunk / 32; ++u) {
          const int c = c0 + u * 32 + lane;
          if (u * 32 < n) v[u] = __fadd_rn(__fmul_rn(v[u], __ldg(in_scale + c)), __ldg(in_shift + c));
        }
      }
#pragma unroll
      for (int u = 0; u < kAbsChunk / 32; ++u) {
        if (u * 32 < n) {
          wide_s[c0 + u * 32 + lane] = fabsf(v[u]);
          const uint32_t word = __ballot_sync(0xffffffffu, v[u] >= 0.0f);  // bit lane = channel c0+32u+lane
          if (lane == (u & 31)) bits[q * Cw + (c0 >> 5) + u] = word;
        }
      }
      __threadfence_block();
      asm volatile("bar.arrive %0, 64;" ::"r"(1 + k) : "memory");  // chunk k staged
    }
  } else {
    float s = 0.0f;
    for (int k = 0; k < nchunk; ++k) {
      asm volatile("bar.sync %0, 64;" ::"r"(1 + k) : "memory");
      if (lane == 0) {
        const int c0 = k * kAbsChunk, n = min(kAbsChunk, C - c0);
        const float4* b4 = reinterpret_cast<const float4*>(wide_s + c0);
        const int nb = n >> 5;
        float4 cur[8], nxt[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) cur[u] = b4[u];
        for (int b = 0; b < nb; ++b) {
          if (b + 1 < nb) {
#pragma unroll
            for (int u = 0; u < 8; ++u) nxt[u] = b4[(b + 1) * 8 + u];
          }
#pragma unroll
          for (int u = 0; u < 8; ++u)
            s = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(s, cur[u].x), cur[u].y), cur[u].z), cur[u].w);
#pragma unroll
          for (int u = 0; u < 8; ++u) cur[u] = nxt[u];
        }
      }
    }
    if (lane == 0 && A != nullptr) A[q] = __fmul_rn(s, inv);
  }
}

// The two-kernel form of K1 (sign words, then the sequential |.| means): no shared
// word tile, so it serves any channel count; the preferred form for few pixels with
// long channel loops.
static int launch_pack_2d(const float* x, int N, int C, int H, int W, uint32_t* bits, float* A,
                          cudaStream_t s, const float* in_scale, const float* in_shift) {
  const long npix = (long)N * H * W;
  const int Cw = cdiv(C, 32);
  const long words = npix * Cw;
  if (H * W == 1 && C >= 1024 && C <= kAbsWideMax && (C & 31) == 0 && npix < 0x7fffffffL) {
    const size_t sm = (size_t)C * sizeof(float);
    if (int rc = smem_opt_in(k_pack_wide, sm)) return rc;  // per device (xnc_runtime.cu)
    k_pack_wide<<<(unsigned)npix, 64, sm, s>>>(x, C, (float)(1.0 / (double)C), bits, A, in_scale, in_shift);
    return launch_status();
  }
  k_pack_words<<<(unsigned)cdivl(words, 256), 256, 0, s>>>(x, C, H * W, Cw, npix, bits, in_scale, in_shift);
  if (A && H * W == 1 && C >= 1024 && C <= kAbsWideMax && (C & 3) == 0) {
    const size_t sm = (size_t)4 * C * sizeof(float);
    if (int rc = smem_opt_in(k_absmean_wide, sm)) return rc;  // per device (xnc_runtime.cu)
    k_absmean_wide<<<(unsigned)cdivl(npix, 4), 128, sm, s>>>(x, C, npix, (float)(1.0 / (double)C), A, in_scale,
                                                             in_shift);
  }
  else if (A)
    k_absmean<<<(unsigned)cdivl(npix, 128), 128, 0, s>>>(x, C, H * W, npix, (float)(1.0 / (double)C), A,
                                                         in_scale, in_shift);
  return launch_status();
}

int launch_pack_input(const float* x, int N, int C, int H, int W, uint32_t* bits, float* A,
                      cudaStream_t s, const float* in_scale, const float* in_shift) {
  {
    const long npix = (long)N * H * W;
    const long vec_groups = (H * W) % 4 == 0 ? npix / 4 : npix;
    // few pixels with long channel loops (13x13 / 6x6 / 1x1 layers): the 2-D path
    if (vec_groups < 2L * 148 * 256 && C >= 256) {
      const int Cw = cdiv(C, 32);
      if (H * W >= 32 && C <= kSmallMaxC) {  // one pass: 32 pixels x C channels per block
        const size_t sm = (size_t)C * 32 * sizeof(float);
        auto kern = in_scale ? k_pack_small<true> : k_pack_small<false>;
        if (int rc = smem_opt_in(kern, sm)) return rc;  // per device (xnc_runtime.cu)
        kern<<<(unsigned)cdivl(npix, 32), 128, sm, s>>>(x, C, H * W, Cw, npix, (float)(1.0 / (double)C), bits, A,
                                                        in_scale, in_shift);
        return launch_status();
      }
      return launch_pack_2d(x, N, C, H, W, bits, A, s, in_scale, in_shift);
    }
  }
  const int HW = H * W;
  const int Cw = cdiv(C, 32);
  const float inv = (float)(1.0 / (double)C);  // <real_t>(1.0 / channels), _kernels_cy.pyx:258
  const bool vec4 = (HW % 4 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0) &&
                    (A == nullptr || (reinterpret_cast<uintptr_t>(A) & 15) == 0);
  const int vec = vec4 ? 4 : 1;
  const long gpi = HW / vec, total = gpi * N;
  // largest block (up to kPackThreads) whose word tile still lets two blocks share an SM
  int threads = kPackThreads;
  while (threads > 128 && (size_t)Cw * (threads * vec + 4) * 4 > 100 * 1024) threads /= 2;
  const size_t smem = (size_t)Cw * (threads * vec + 4) * 4;
  // the word tile does not fit (C > ~3.1k channels at VEC = 4, ~12k at VEC = 1): the
  // two-kernel form (words, then the |.| means) handles any C
  if (smem > 200 * 1024) return launch_pack_2d(x, N, C, H, W, bits, A, s, in_scale, in_shift);
  const unsigned blocks = (unsigned)cdivl(total, threads);
  const bool aff = in_scale != nullptr;
  int opt_rc = XNC_OK;
  auto go = [&](auto kern, int t) {
    opt_rc = smem_opt_in(kern, smem);  // per device (xnc_runtime.cu)
    if (opt_rc == XNC_OK)
      launch_pdl(kern, dim3(blocks), dim3(t), smem, s, x, C, HW, Cw, inv, gpi, total, bits, A, in_scale, in_shift);
  };
  auto pick = [&](auto aff_tag) {
    constexpr bool AF = decltype(aff_tag)::value;
    if (vec4) {
      if (threads == 512) go(k_pack_input<4, 512, AF>, 512);
      else if (threads == 256) go(k_pack_input<4, 256, AF>, 256);
      else go(k_pack_input<4, 128, AF>, 128);
    } else {
      if (threads == 512) go(k_pack_input<1, 512, AF>, 512);
      else if (threads == 256) go(k_pack_input<1, 256, AF>, 256);
      else go(k_pack_input<1, 128, AF>, 128);
    }
  };
  if (aff) pick(std::true_type{});
  else pick(std::false_type{});
  if (opt_rc) return opt_rc;
  return launch_status();
}

// K1 for a channels-last input [N][H][W][C]: one thread per pixel walks its C
// contiguous channels in order (16-byte loads when C % 4 == 0), building the words
// and the sequential |.| sum exactly as k_pack_input does for NCHW.
template <bool AFF>
__global__ void __launch_bounds__(128) k_pack_input_nhwc(const float* __restrict__ x, int C, int Cw, long npix,
                                                         float inv, uint32_t* __restrict__ bits,
                                                         float* __restrict__ A,
                                                         const float* __restrict__ in_scale,
                                                         const float* __restrict__ in_shift) {
  const long q = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= npix) return;
  const float* xp = x + q * C;
  const bool v4 = (C & 3) == 0 && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  float s = 0.0f;
  for (int j = 0; j < Cw; ++j) {
    const int c0 = 32 * j, cend = min(32, C - c0);
    float v[32];
    if (v4 && cend == 32) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(xp + c0) + u);
        v[4 * u] = t.x; v[4 * u + 1] = t.y; v[4 * u + 2] = t.z; v[4 * u + 3] = t.w;
      }
    } else {
#pragma unroll
      for (int u = 0; u < 32; ++u) v[u] = u < cend ? __ldg(xp + c0 + u) : 0.0f;
    }
    uint32_t word = 0u;
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      if (u < cend) {
        float t = v[u];
        if (AFF) t = __fadd_rn(__fmul_rn(t, __ldg(in_scale + c0 + u)), __ldg(in_shift + c0 + u));
        s = __fadd_rn(s, fabsf(t));
        word |= (t >= 0.0f ? 1u : 0u) << u;
      }
    }
    bits[q * Cw + j] = word;
  }
  if (A) A[q] = __fmul_rn(s, inv);
}

int launch_pack_input_nhwc(const float* x, int N, int C, int H, int W, uint32_t* bits, float* A, cudaStream_t s,
                           const float* in_scale, const float* in_shift) {
  const long npix = (long)N * H * W;
  const int Cw = cdiv(C, 32);
  const float inv = (float)(1.0 / (double)C);
  const unsigned blocks = (unsigned)cdivl(npix, 128);
  if (in_scale)
    k_pack_input_nhwc<true><<<blocks, 128, 0, s>>>(x, C, Cw, npix, inv, bits, A, in_scale, in_shift);
  else
    k_pack_input_nhwc<false><<<blocks, 128, 0, s>>>(x, C, Cw, npix, inv, bits, A, in_scale, in_shift);
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
