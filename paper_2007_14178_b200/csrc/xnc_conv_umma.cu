// K3 on the 5th-generation tensor cores: tcgen05.mma.kind::i8, accumulators in TMEM.
//
// Exact-integer reformulation of the XNOR sum.  With d = 1 for a negative input
// sign (0 for +1, for zero padding and for tail channels) and s_w = +-1 the
// filter sign (0 for tail channels):
//     sum_taps s_x * s_w = sum_taps (1 - 2d) * s_w = S_w[o] - 2 * sum_taps d * s_w
// where S_w[o] is the sum of the filter's signs.  sum d*s_w is a u8 x s8 GEMM
// with an s32 accumulator (M = output pixels, N = filters, K = kh*kw*C), so the
// result is bit-identical to the reference decode `k_area - 2*popc(diff)`
// summed over channels (_kernels_cy.pyx:100-104); the alpha*K epilogue
// (_kernels_cy.pyx:349) is applied from TMEM.  Zero-filled taps are d = 0 = the
// +1 padding of zero_pad-then-binarize (reference.py:87): TMA's out-of-bounds
// zero fill IS the reference padding rule.
//
// Implicit GEMM without an im2col buffer.  Per image the output is walked on an
// "extended" grid of H' rows x IC = W + 2*pad columns (the padded input row
// length; the last kw-1 columns of every row are discarded).  Output pixel e and
// tap (ky, kx) then read padded input pixel e + ky*IC + kx: every tap of a
// 128-row MMA tile is the SAME shared-memory tile shifted by whole 128-byte rows,
// i.e. one K-major SWIZZLE_128B descriptor per tap and no data movement
// (tools/microbench/umma_probe.cu: row-shifted descriptors with base_offset = 0
// verified against a CPU GEMM on a B200, 0 mismatches for shifts 0-9).
//
// Persistent, warp-specialised pipeline (one CTA per SM, 640 threads):
//   warp 0      B producer: cp.async.bulk of one (tap, K block) filter chunk,
//               NB x 128 B, pre-swizzled in HBM by k_pack_weights_umma
//   warp 1      MMA issuer (one thread): per tile and filter block,
//               MH M=128 row blocks x 4 K=32 steps per chunk, accumulate in TMEM
//   warp 2      A producer: one TMA tile load per 128-channel K block of the
//               d-bytes written by K1 (xnc_pack_input_umma): R padded rows x IC
//               columns x 128 B, zero fill outside the image
//   warps 4-19  epilogue: TMEM -> registers -> S_w - 2*acc -> (f32 * K) * alpha
//               -> y, four warps per TMEM lane quadrant
// Work unit = (tile of 128*MH extended pixels of one image, filter block of NB).
// TMEM holds two accumulators (MH x NB columns each): the epilogue of one unit
// overlaps the MMAs of the next.  A K-block plane is released as soon as
// the tile's last filter block has consumed it, so the next tile's TMA load
// overlaps the remaining MMAs.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

#include "xnc_common.cuh"

namespace xnc {

constexpr int kU2Threads = 640;
constexpr int kU2Stages = 6;     // B pipeline depth
constexpr int kU2MaxKB = 4;      // K blocks (128 channels each) kept resident: C <= 512
constexpr int kU2EpiWarp0 = 4;   // first epilogue warp
constexpr int kU2EpiWarps = 16;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// K-major, SWIZZLE_128B UMMA shared-memory descriptor (sm_100 version 1): rows
// 128 B apart, 8-row groups 1024 B apart (SBO).  The swizzle is a function of the
// absolute smem address, so row-shifted starts need no base offset.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  }
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ void tma_prefetch_4d(const CUtensorMap* map, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}

__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_addr(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16_async(uint32_t addr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15},"
      " [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
        "=r"(v[15])
      : "r"(addr));
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t addr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15},"
      " [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
        "=r"(v[15])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

struct UmmaGeom {
  int C, H, W, O, kh, kw, pad, oh, ow, IC, KBn, NB, R, plane_bytes, n_mt, n_nb, tiles, taps, MH;
  uint32_t box_bytes, tmem_cols;
  int debug;  // profiling only (env XNC_UMMA_DEBUG): bit 0 = skip epilogue stores, bit 1 = load B once,
             // bit 2 = load the input rows once, bit 3 = no B barrier protocol after the
             // first stages, bit 4 = no tcgen05 fence after B waits
};

// MH = M=128 row blocks per tile (tile = 128*MH extended pixels); the two TMEM
// accumulators hold MH x NB columns each (MH * NB <= 256).
template <int MH>
__global__ void __launch_bounds__(kU2Threads, 1) k_conv_umma(
    const __grid_constant__ CUtensorMap a_map, const uint8_t* __restrict__ wq,
    const int32_t* __restrict__ sw, const float* __restrict__ Kmap, const float* __restrict__ alpha,
    const UmmaGeom g, float* __restrict__ y, int32_t* __restrict__ acc_out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  uint8_t* a_s = smem;                                   // KBn planes of R*IC rows x 128 B
  uint8_t* b_s = a_s + (size_t)g.KBn * g.plane_bytes;    // stages x NB rows x 128 B
  const uint32_t b_bytes = (uint32_t)g.NB * 128u;
  __shared__ __align__(8) uint64_t b_full[kU2Stages], b_empty[kU2Stages];
  __shared__ __align__(8) uint64_t a_full[kU2MaxKB], a_empty[kU2MaxKB];
  __shared__ __align__(8) uint64_t t_full[2], t_empty[2];
  __shared__ uint32_t tmem_base_s;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kU2Stages; ++s) { mbar_init(&b_full[s], 1); mbar_init(&b_empty[s], 1); }
    for (int k = 0; k < kU2MaxKB; ++k) { mbar_init(&a_full[k], 1); mbar_init(&a_empty[k], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&t_full[b], 1); mbar_init(&t_empty[b], kU2EpiWarps); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2 && lane == 0)
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a_map)) : "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_addr(&tmem_base_s)), "r"(g.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_s;

  if (warp == 0) {
    // ================= B producer
    if (lane == 0) {
      uint32_t step = 0;
      for (int t = blockIdx.x; t < g.tiles; t += gridDim.x)
        for (int nb = 0; nb < g.n_nb; ++nb)
          for (int kb = 0; kb < g.KBn; ++kb)
            for (int tap = 0; tap < g.taps; ++tap, ++step) {
              const uint32_t st = step % kU2Stages;
              if (step >= kU2Stages) mbar_wait(&b_empty[st], ((step / kU2Stages) - 1) & 1);
              if ((g.debug & 8) && step >= kU2Stages) continue;  // profiling: no B protocol at all
              if ((g.debug & 2) && step >= kU2Stages) {
                mbar_arrive(&b_full[st]);  // profiling: reuse resident chunks, no traffic
                continue;
              }
              mbar_expect_tx(&b_full[st], b_bytes);
              const size_t chunk = ((size_t)nb * g.taps + tap) * g.KBn + kb;
              bulk_load(b_s + st * b_bytes, wq + chunk * b_bytes, b_bytes, &b_full[st]);
            }
    }
  } else if (warp == 2) {
    // ================= A producer (TMA)
    if (lane == 0) {
      uint32_t it = 0;
      for (int t = blockIdx.x; t < g.tiles; t += gridDim.x, ++it) {
        const int n = t / g.n_mt, m0 = (t - n * g.n_mt) * (128 * MH);
        const int r0 = m0 / g.IC;
        for (int kb = 0; kb < g.KBn; ++kb) {
          if (it >= 1) mbar_wait(&a_empty[kb], (it - 1) & 1);
          if ((g.debug & 4) && it >= 1) {  // profiling: keep the first tile's rows, no traffic
            mbar_arrive(&a_full[kb]);
            continue;
          }
          mbar_expect_tx(&a_full[kb], g.box_bytes);
          tma_load_4d(a_s + (size_t)kb * g.plane_bytes, &a_map, kb * 128, -g.pad, r0 - g.pad, n, &a_full[kb]);
        }
        // warm L2 with the next tile's rows: its loads are issued while this
        // tile's last MMAs run, and must land before the tensor core drains
        const int tn = t + gridDim.x;
        if (tn < g.tiles) {
          const int nn = tn / g.n_mt, rn = ((tn - nn * g.n_mt) * (128 * MH)) / g.IC;
          for (int kb = 0; kb < g.KBn; ++kb) tma_prefetch_4d(&a_map, kb * 128, -g.pad, rn - g.pad, nn);
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer
    // Descriptors are built once and advanced by adding (byte offset >> 4) to
    // the start-address field (addresses < 256 KB never carry out of it), so
    // each MMA costs one 64-bit add: the issue loop must stay well ahead of
    // the tensor core (a 128x128x32 i8 MMA retires in ~67 cycles).
    if (lane == 0) {
      const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(g.NB >> 3) << 17) |
                             ((uint32_t)(128 >> 4) << 24);
      const uint64_t a_desc0 = umma_desc_sw128(smem_addr(a_s));
      const uint64_t b_desc0 = umma_desc_sw128(smem_addr(b_s));
      const uint32_t plane16 = (uint32_t)g.plane_bytes >> 4, b16 = b_bytes >> 4;
      uint32_t step = 0, item = 0, it = 0;
      for (int t = blockIdx.x; t < g.tiles; t += gridDim.x, ++it) {
        const int n = t / g.n_mt, m0 = (t - n * g.n_mt) * (128 * MH);
        const uint32_t tile16 = (uint32_t)(m0 - (m0 / g.IC) * g.IC) * 8u;  // off0 rows x 128 B / 16
        for (int nb = 0; nb < g.n_nb; ++nb, ++item) {
          const uint32_t buf = item & 1;
          if (item >= 2) {
            mbar_wait(&t_empty[buf], ((item >> 1) - 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
          }
          const uint32_t d0 = tmem + buf * (MH * g.NB);
          uint32_t acc = 0;
          for (int kb = 0; kb < g.KBn; ++kb) {
            if (nb == 0) {
              mbar_wait(&a_full[kb], it & 1);
              asm volatile("tcgen05.fence::after_thread_sync;");
            }
            const uint64_t a_kb = a_desc0 + kb * plane16 + tile16;
            for (int ky = 0; ky < g.kh; ++ky) {
              for (int kx = 0; kx < g.kw; ++kx, ++step) {
                const uint32_t st = step % kU2Stages;
                const bool b_sync = !(g.debug & 8) || step < kU2Stages;
                if (b_sync) {
                  mbar_wait(&b_full[st], (step / kU2Stages) & 1);
                  if (!(g.debug & 16)) asm volatile("tcgen05.fence::after_thread_sync;");
                }
                const uint64_t a_tap = a_kb + (uint32_t)(ky * g.IC + kx) * 8u;
                const uint64_t b_st = b_desc0 + st * b16;
#pragma unroll
                for (int s = 0; s < 4; ++s) {
#pragma unroll
                  for (int h = 0; h < MH; ++h)
                    umma_i8(d0 + h * g.NB, a_tap + h * 1024 + 2 * s, b_st + 2 * s, idesc, acc | (uint32_t)s);
                }
                acc = 1;
                if (b_sync) umma_commit(&b_empty[st]);
              }
            }
            if (nb == g.n_nb - 1) umma_commit(&a_empty[kb]);
          }
          umma_commit(&t_full[buf]);
        }
      }
    }
  } else if (warp >= kU2EpiWarp0 && warp < kU2EpiWarp0 + kU2EpiWarps) {
    // ================= epilogue
    // 16 warps: warp w reads TMEM lane quadrant (w & 3) and the 16-column chunks
    // cg, cg+4, ... (cg = (w-4) >> 2) of every accumulator row block.  Each
    // thread owns one extended pixel per row block; for a chunk it issues the
    // TMEM loads of all row blocks before one wait, then writes 16 filters x MH
    // pixels (for a fixed filter the 32 lanes store 32 consecutive pixels).
    const int e_w = warp - kU2EpiWarp0;
    const int quad = warp & 3;              // TMEM lane quadrant this warp may access
    const int cg = e_w >> 2;
    const int n_chunks = g.NB / 16;
    const size_t plane_out = (size_t)g.oh * g.ow;
    uint32_t item = 0;
    const bool vec_ok = ((reinterpret_cast<uintptr_t>(sw) & 15) == 0) &&
                        ((reinterpret_cast<uintptr_t>(alpha) & 15) == 0);
    for (int t = blockIdx.x; t < g.tiles; t += gridDim.x) {
      const int n = t / g.n_mt, m0 = (t - n * g.n_mt) * (128 * MH);
      size_t pix[MH];
      bool ok[MH];
      float kv[MH];
#pragma unroll
      for (int h = 0; h < MH; ++h) {
        const int e = m0 + h * 128 + quad * 32 + lane;
        const int rr = e / g.IC, cc = e - (e / g.IC) * g.IC;
        ok[h] = rr < g.oh && cc < g.ow;
        pix[h] = (size_t)n * g.O * plane_out + (size_t)rr * g.ow + cc;
        kv[h] = (ok[h] && y) ? __ldg(Kmap + (size_t)n * plane_out + (size_t)rr * g.ow + cc) : 0.0f;
      }
      for (int nb = 0; nb < g.n_nb; ++nb, ++item) {
        const uint32_t buf = item & 1;
        mbar_wait(&t_full[buf], (item >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        for (int ch = cg; ch < n_chunks; ch += 4) {
          const int c = ch * 16;
          const int obase = nb * g.NB + c;
          uint32_t v[MH][16];
#pragma unroll
          for (int h = 0; h < MH; ++h)
            tmem_ld16_async(tmem + ((uint32_t)(quad * 32) << 16) + buf * (MH * g.NB) + h * g.NB + c, v[h]);
          // per-filter constants for these 16 columns (uniform across lanes)
          int swv[16];
          float av[16];
          if (vec_ok && obase + 16 <= g.O) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int4 si = __ldg(reinterpret_cast<const int4*>(sw + obase) + q);
              const float4 ai = __ldg(reinterpret_cast<const float4*>(alpha + obase) + q);
              swv[4 * q] = si.x; swv[4 * q + 1] = si.y; swv[4 * q + 2] = si.z; swv[4 * q + 3] = si.w;
              av[4 * q] = ai.x; av[4 * q + 1] = ai.y; av[4 * q + 2] = ai.z; av[4 * q + 3] = ai.w;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const bool in = obase + j < g.O;
              swv[j] = in ? __ldg(sw + obase + j) : 0;
              av[j] = in ? __ldg(alpha + obase + j) : 0.0f;
            }
          }
          tmem_wait_ld();
          if (g.debug & 1) continue;
#pragma unroll
          for (int h = 0; h < MH; ++h) {
            if (!ok[h]) continue;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int o = obase + j;
              if (o < g.O) {
                const int accv = swv[j] - 2 * (int)v[h][j];
                const size_t idx = pix[h] + (size_t)o * plane_out;
                if (y) __stcs(y + idx, __fmul_rn(__fmul_rn((float)accv, kv[h]), av[j]));
                if (acc_out) acc_out[idx] = accv;
              }
            }
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) mbar_arrive(&t_empty[buf]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    __syncwarp();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(g.tmem_cols));
  }
}

// ---------------------------------------------------------------- weights
// wq[nb][tap][kb][row = filter within block][128 B], s8 signs (+1/-1, 0 for tail
// channels and filters >= O); each (tap, kb) chunk pre-swizzled for a 1024-aligned
// smem destination (16-byte chunk q of row r stored at q ^ (r & 7)).
template <typename T>
__global__ void k_pack_weights_umma(const T* __restrict__ w, int O, int C, int kh, int kw, int NB,
                                    int KBn, uint8_t* __restrict__ wq) {
  const long total = (long)cdiv(O, NB) * kh * kw * KBn * NB * 8;
  long it = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (it >= total) return;
  const int q = (int)(it & 7);
  long rest = it >> 3;
  const int row = (int)(rest % NB); rest /= NB;
  const int kb = (int)(rest % KBn); rest /= KBn;
  const int tap = (int)(rest % (kh * kw));
  const int nb = (int)(rest / (kh * kw));
  const int o = nb * NB + row;
  uint32_t vals[4] = {0u, 0u, 0u, 0u};
  if (o < O) {
    for (int b = 0; b < 16; ++b) {
      const int c = kb * 128 + q * 16 + b;
      if (c < C) {
        const T v = w[((long)o * C + c) * kh * kw + tap];
        const uint32_t sgn = v >= T(0) ? 0x01u : 0xFFu;
        vals[b >> 2] |= sgn << ((b & 3) * 8);
      }
    }
  }
  uint8_t* chunk = wq + ((((long)nb * kh * kw + tap) * KBn + kb) * NB + row) * 128;
  *reinterpret_cast<uint4*>(chunk + ((q ^ (row & 7)) << 4)) = make_uint4(vals[0], vals[1], vals[2], vals[3]);
}

template <typename T>
__global__ void k_weight_sign_sums(const T* __restrict__ w, int O, int C, int kk, int32_t* __restrict__ sw) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= O) return;
  int s = 0;
  for (long i = 0; i < (long)C * kk; ++i) s += w[(long)o * C * kk + i] >= T(0) ? 1 : -1;
  sw[o] = s;
}

// Tile shape.  NB (filters per block) must not depend on the image shape, since
// the weights are packed before any input is seen; MH (M=128 row blocks per tile)
// is picked per shape.  2 accumulators x MH x NB columns must fit 512 TMEM cols.
// XNC_UMMA_TILE="MH,NB" overrides both (tuning knob, read once per process).
struct UmmaTilePref {
  int mh = 2, nb = 128;
  UmmaTilePref() {
    if (const char* e = getenv("XNC_UMMA_TILE")) {
      int a = 0, b = 0;
      if (sscanf(e, "%d,%d", &a, &b) == 2 && (a == 1 || a == 2 || a == 4) && b >= 32 && b % 32 == 0 &&
          2 * a * b <= 512) {
        mh = a;
        nb = b;
      }
    }
  }
};
static const UmmaTilePref& tile_pref() {
  static UmmaTilePref p;
  return p;
}
static int umma_nb(int O) { return O >= tile_pref().nb ? tile_pref().nb : round_up(O, 32); }

size_t umma_weight_bytes(int O, int C, int kh, int kw) {
  const int NB = umma_nb(O);
  return (size_t)cdiv(O, NB) * NB * kh * kw * cdiv(C, 128) * 128;
}

int launch_pack_weights_umma(const void* w, int dtype, int O, int C, int kh, int kw, uint8_t* wq,
                             int32_t* sw, cudaStream_t s) {
  const int NB = umma_nb(O), KBn = cdiv(C, 128);
  const long total = (long)cdiv(O, NB) * kh * kw * KBn * NB * 8;
  const unsigned blocks = (unsigned)cdivl(total, 256);
  if (dtype == XNC_DTYPE_F64) {
    k_pack_weights_umma<double><<<blocks, 256, 0, s>>>((const double*)w, O, C, kh, kw, NB, KBn, wq);
    k_weight_sign_sums<double><<<cdiv(O, 128), 128, 0, s>>>((const double*)w, O, C, kh * kw, sw);
  } else {
    k_pack_weights_umma<float><<<blocks, 256, 0, s>>>((const float*)w, O, C, kh, kw, NB, KBn, wq);
    k_weight_sign_sums<float><<<cdiv(O, 128), 128, 0, s>>>((const float*)w, O, C, kh * kw, sw);
  }
  return launch_status();
}

static bool umma_plan_mh(int N, int C, int H, int W, int O, int kh, int kw, int pad, int MH, UmmaGeom& g,
                         size_t& smem) {
  g.C = C; g.H = H; g.W = W; g.O = O; g.kh = kh; g.kw = kw; g.pad = pad; g.MH = MH;
  g.oh = H + 2 * pad - kh + 1; g.ow = W + 2 * pad - kw + 1;
  g.IC = W + 2 * pad;
  g.KBn = cdiv(C, 128);
  g.NB = umma_nb(O);
  g.taps = kh * kw;
  const int MT = 128 * MH;
  // padded input rows a tile touches: pixel indices off0 .. off0+MT-1 + (kh-1)*IC + kw-1
  g.R = (g.IC - 1 + MT - 1 + kw - 1) / g.IC + kh;
  g.box_bytes = (uint32_t)g.R * g.IC * 128u;
  g.plane_bytes = round_up(g.R * g.IC * 128, 1024);
  g.n_mt = cdiv(g.oh * g.IC, MT);
  g.n_nb = cdiv(O, g.NB);
  g.tiles = N * g.n_mt;
  const int cols = 2 * MH * g.NB;  // two accumulators x MH row blocks
  g.tmem_cols = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
  smem = (size_t)g.KBn * g.plane_bytes + (size_t)kU2Stages * g.NB * 128 + 1024;
  return cols <= 512 && g.KBn <= kU2MaxKB && g.IC <= 256 && g.R <= 256 && smem <= 225 * 1024 &&
         (long)N * g.n_mt < 0x7fffffffL;
}

// Preferred MH first, then smaller tiles if the input rows do not fit shared memory.
static bool umma_plan(int N, int C, int H, int W, int O, int kh, int kw, int pad, UmmaGeom& g,
                      size_t& smem) {
  for (int mh = tile_pref().mh; mh >= 1; mh /= 2)
    if (umma_plan_mh(N, C, H, W, O, kh, kw, pad, mh, g, smem)) return true;
  return false;
}

bool umma_supported(int N, int C, int H, int W, int O, int kh, int kw, int pad) {
  UmmaGeom g;
  size_t smem;
  return umma_plan(N, C, H, W, O, kh, kw, pad, g, smem);
}

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// Profiling counters (XNC_UMMA_DEBUG bit 7): none in this kernel yet.
__device__ unsigned long long g_umma_prof[1024][16];

int umma_profile_read(unsigned long long* host, int n_ctas) {
  if (n_ctas > 1024) n_ctas = 1024;
  cudaError_t e = cudaMemcpyFromSymbol(host, g_umma_prof, sizeof(unsigned long long) * 16 * n_ctas);
  return e == cudaSuccess ? 0 : XNC_ECUDA_BASE + (int)e;
}

int launch_conv_umma(const uint8_t* dbytes, const uint8_t* wq, const int32_t* sw, const float* K,
                     const float* alpha, int N, int C, int H, int W, int O, int kh, int kw, int pad,
                     float* y, int32_t* acc, cudaStream_t s) {
  UmmaGeom g;
  size_t smem;
  if (!umma_plan(N, C, H, W, O, kh, kw, pad, g, smem)) return XNC_ENOTSUP;
  auto encode = tensor_map_encoder();
  if (!encode) return XNC_ENOTSUP;
  // d-bytes [N][H][W][Cpad] u8; TMA box = 128 channels x IC columns x R rows x 1 image
  const int Cpad = g.KBn * 128;
  CUtensorMap map;
  cuuint64_t dims[4] = {(cuuint64_t)Cpad, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
  cuuint64_t strides[3] = {(cuuint64_t)Cpad, (cuuint64_t)W * Cpad, (cuuint64_t)H * W * Cpad};
  cuuint32_t box[4] = {128u, (cuuint32_t)g.IC, (cuuint32_t)g.R, 1u};
  cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
  CUresult cr = encode(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<uint8_t*>(dbytes), dims, strides,
                       box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return XNC_ENOTSUP;
  {
    static const int dbg = getenv("XNC_UMMA_DEBUG") ? atoi(getenv("XNC_UMMA_DEBUG")) : 0;
    g.debug = dbg;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = g.tiles < sms ? g.tiles : sms;
  static size_t attr_smem[3] = {0, 0, 0};  // one-time (per size increase) shared-memory opt-in
  auto kern = g.MH == 4 ? k_conv_umma<4> : g.MH == 2 ? k_conv_umma<2> : k_conv_umma<1>;
  size_t& attr = attr_smem[g.MH == 4 ? 2 : g.MH == 2 ? 1 : 0];
  if (smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return XNC_ECUDA_BASE + (int)e;
    attr = smem;
  }
  kern<<<grid, kU2Threads, smem, s>>>(map, wq, sw, K, alpha, g, y, acc);
  return launch_status();
}

}  // namespace xnc
