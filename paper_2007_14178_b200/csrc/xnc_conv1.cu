// XNOR-Net AlexNet conv1 (11x11, stride 4, pad 2, 3 -> 96 channels, 224 -> 55) on
// the tcgen05 tensor cores in TF32 -- the network's full-precision first layer
// (network.py), outside the binary hot path.  It replaces three passes (pad +
// space-to-depth, cuDNN's TF32 implicit GEMM, and their 160 MB intermediate) with
// one kernel that reads the raw NCHW images once.
//
// Formulation: the 11x11/4 conv is a 3x3/1 conv over the 4x4 space-to-depth grid
// of the 2-padded image (57 x 57 cells of 48 values: raw channel c, phase dy, dx;
// the kernel zero-padded to 12 x 12), the same products and sums as
// network.py's cuDNN path.  As in the binary conv (xnc_conv_umma.cu), output pixels
// are walked on the "extended" grid -- all 57 x 57 cells of every image, linear
// over the batch -- so tap (ky, kx) of extended pixel e reads cell e + ky*57 + kx:
// one shared-memory plane per tile, each tap a row-shifted descriptor.  Outputs
// with Y or X >= 55 are discarded (6.9 % of the MMA work).
//
// CTA pairs (cta_group::2): one MMA is M = 256 extended pixels (128 per CTA) x
// N = 96 filters (48 rows of B in each CTA) x K = 8.  Per tile, 3 raw channels x 9
// taps x 2 K-steps = 54 MMAs, f32 accumulators in TMEM (double-buffered).  Tiles
// stay inside one image (13 pair tiles of 256 cells per 57 x 57 image).
//   warp 0      B (once: this CTA's 48 filter rows of all 27 (c, tap) blocks, TMA,
//               SWIZZLE_64B), then the MMA issuer on the leader CTA
//   warp 1      TMA of the raw rows a CTA tile reads (24 rows x 224 per channel,
//               zero-filled outside the image) through a 4-slot staging ring; TMEM owner
// The A operand is one tile's three per-channel sub-planes, each with its own
// full / empty barriers: the MMAs of channel c start as soon as its sub-plane is
// built, and the next tile's channel c is built while channels c+1.. are multiplied
// (a whole-tile double buffer does not fit beside the 83 KB of resident B and the
// staging ring; with a 2-slot ring the TMA latency was exposed once per tile).
//   warps 2-3, 8-11  A producers: staging -> TF32 (round to nearest) -> the tile's
//               three 64-byte-row SWIZZLE_64B sub-planes (c = 0, 1, 2), 244 rows each
//   warps 4-7   epilogue: TMEM -> registers -> y, one pixel per thread, its 96
//               channels contiguous (NHWC: 24 x 16-byte stores)
// (Producers loading x with 8-byte LDGs themselves were LSU-queue bound: ncu 57 %
// long-scoreboard + 10 % lg_throttle stalls, tensor pipe 30 % active, 209 us at C4.)
// The caller applies bias + ReLU + max-pool (xnc_max_pool, channels-last).
#include <algorithm>
#include <cstdlib>

#include "xnc_common.cuh"
#include "xnc_tcgen05.cuh"

namespace xnc {

constexpr int kC1N = 96;                    // filters (MMA N)
constexpr int kC1Half = 48;                 // B rows per CTA of the pair
constexpr int kC1In = 224;                  // input rows / cols
constexpr int kC1SG = 57;                   // space-to-depth grid: (224 + 2 * 2) / 4
constexpr int kC1Out = 55;                  // output rows / cols
constexpr int kC1Ext = kC1SG * kC1SG;       // extended pixels per image
constexpr int kC1P = 128 + 2 * kC1SG + 2;   // plane rows a CTA tile reads (244)
constexpr int kC1Rows = 248;                // rounded up to whole 8-row (512 B) swizzle atoms
constexpr int kC1Sub = kC1Rows * 64;        // one raw channel's sub-plane
constexpr int kC1Plane = 3 * kC1Sub;        // one tile's A operand (47,616 B)
constexpr int kC1Blocks = 27;               // (c, tap) weight blocks
constexpr int kC1BBlock = kC1Half * 64;     // one block, this CTA's rows (3,072 B)
constexpr int kC1BBytes = kC1Blocks * kC1BBlock;
constexpr int kC1Tiles = (kC1Ext + 255) / 256;  // pair tiles per image (13)
constexpr int kC1StRows = 24;               // raw rows a CTA tile spans: 6 cell rows x 4
constexpr int kC1Stage = kC1StRows * kC1In * 4;  // one channel's rows (21,504 B)
constexpr int kC1Slots = 3;                       // staging ring
constexpr int kC1OutPitch = 52;                   // epilogue staging row: 48 floats + 4 (bank skew)
constexpr int kC1Out1 = 32 * kC1OutPitch * 4;     // one epilogue warp's staging (6,656 B)
constexpr int kC1Smem = kC1Plane + kC1BBytes + kC1Slots * kC1Stage + 4 * kC1Out1 + 1024;
constexpr int kC1ProdWarps = 6;
constexpr int kC1Threads = 12 * 32;
constexpr int kC1TmemCols = 256;            // two 96-column accumulators

__device__ __forceinline__ float to_tf32(float v) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return __uint_as_float(r);
}

// One (c, tap): two K=8 MMAs (the 64-byte row's two halves), one elected lane.
__device__ __forceinline__ void umma_tf32_tap(uint32_t d, uint32_t a_lo, uint32_t b_lo, uint32_t hi,
                                              uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t.reg .b32 al, bl;\n\t.reg .b64 a, b;\n\t"
      "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "mov.b64 a, {%1, %5};\n\tmov.b64 b, {%2, %5};\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, b, %3, p;\n\t"
      "add.u32 al, %1, 2;\n\tadd.u32 bl, %2, 2;\n\tmov.b64 a, {al, %5};\n\tmov.b64 b, {bl, %5};\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a, b, %3, 1;\n\t}" ::"r"(d),
      "r"(a_lo), "r"(b_lo), "r"(idesc), "r"(acc), "r"(hi));
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kC1Threads, 1)
    k_conv1_tf32_pair(const __grid_constant__ CUtensorMap x_map, int N, const __grid_constant__ CUtensorMap b_map,
                      float* __restrict__ y, int tiles, int dbg) {
  // dbg (profiling only, env XNC_CONV1_DEBUG): bit 0 = epilogue skips its stores,
  // bit 1 = producers build only the first tile's planes, bit 2 = no MMAs issued
  extern __shared__ __align__(1024) uint8_t c1_smem_raw[];
  uint8_t* smem = c1_smem_raw + ((1024u - (smem_addr(c1_smem_raw) & 1023u)) & 1023u);
  uint8_t* a_s = smem;                                   // one tile's 3 sub-planes
  uint8_t* b_s = smem + kC1Plane;                        // 27 blocks x 48 rows x 64 B
  float* st_s = reinterpret_cast<float*>(b_s + kC1BBytes);  // raw rows ring [slot][24][224]
  float* out_s = st_s + kC1Slots * (kC1Stage / 4);          // epilogue staging [warp][32 px][52]
  __shared__ __align__(8) uint64_t b_full, a_full[3], a_empty[3], s_full[kC1Slots], s_empty[kC1Slots],
      t_full[2], t_empty[2];
  __shared__ uint32_t tmem_base_s;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;
  if (tid == 0) {
    mbar_init(&b_full, 1);
    for (int b = 0; b < kC1Slots; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&s_empty[b], kC1ProdWarps);
    }
    for (int c = 0; c < 3; ++c) {
      mbar_init(&a_full[c], 2 * kC1ProdWarps);
      mbar_init(&a_empty[c], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&t_full[b], 1);
      mbar_init(&t_empty[b], 2 * 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();  // barrier inits complete before any role starts (and before the TMEM alloc)
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_addr(&tmem_base_s)), "r"(kC1TmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_s;

  if (warp == 0) {
    // ---- B: this CTA's 48 rows of every (c, tap) block, once; completes on the leader
    if (lane == 0) {
      const uint32_t full = map_to_rank(smem_addr(&b_full), 0);
      if (leader) mbar_expect_tx(&b_full, 2u * kC1BBytes);
      for (int b = 0; b < kC1Blocks; ++b)
        tma_load_2d_pair(b_s + b * kC1BBlock, &b_map, 0, b * kC1N + (int)rank * kC1Half, full);
    }
    __syncwarp();
    if (leader) {
      // ---- MMA issuer: D f32 (bits 4-5 = 1), A and B TF32 (2), K-major, N = 96, M = 256
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kC1N >> 3) << 17) |
                             ((uint32_t)(256 >> 4) << 24);
      const uint64_t a_desc0 = umma_desc_sw64(smem_addr(a_s));
      const uint64_t b_desc0 = umma_desc_sw64(smem_addr(b_s));
      const uint32_t a_lo0 = (uint32_t)a_desc0, hi = (uint32_t)(a_desc0 >> 32), b_lo0 = (uint32_t)b_desc0;
      mbar_wait(&b_full, 0);
      asm volatile("tcgen05.fence::after_thread_sync;");
      uint32_t item = 0;
      for (int t = cluster; t < tiles; t += n_clusters, ++item) {
        const uint32_t buf = item & 1;
        if (item >= 2) {
          mbar_wait(&t_empty[buf], ((item >> 1) - 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
        }
        const uint32_t d = tmem + buf * kC1N;
        const uint32_t a_plane = a_lo0;
        uint32_t acc = 0;
#pragma unroll 1
        for (int c = 0; c < 3; ++c) {
          mbar_wait(&a_full[c], item & 1);  // sub-plane c of this tile built (both CTAs)
          asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
          for (int tap = 0; tap < 9; ++tap) {
            const int ky = tap / 3, kx = tap - 3 * (tap / 3);
            const uint32_t a_lo = a_plane + (uint32_t)(c * (kC1Sub >> 4) + (ky * kC1SG + kx) * 4);
            const uint32_t b_lo = b_lo0 + (uint32_t)((c * 9 + tap) * (kC1BBlock >> 4));
            if (!(dbg & 4)) umma_tf32_tap(d, a_lo, b_lo, hi, idesc, acc);
            acc = 1;
          }
          umma_commit_pair_elect(&a_empty[c]);  // sub-plane c free once these MMAs finish
        }
        umma_commit_pair_elect(&t_full[buf]);
      }
    }
  } else if (warp == 1) {
    // ---- raw-row TMA, one channel per slot: rows 4*Y0 - 2 .. 4*Y0 + 21 of channel c
    if (lane == 0) {
      uint32_t use = 0;
      for (int t = cluster; t < tiles; t += n_clusters) {
        const int img = t / kC1Tiles, e0 = (t - img * kC1Tiles) * 256 + (int)rank * 128;
        const int Y0 = e0 / kC1SG;
        for (int c = 0; c < 3; ++c, ++use) {
          const uint32_t sl = use % kC1Slots;
          if (use >= kC1Slots) mbar_wait(&s_empty[sl], ((use / kC1Slots) - 1) & 1);
          mbar_expect_tx(&s_full[sl], (uint32_t)kC1Stage);
          asm volatile(
              "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_addr(st_s) + sl * kC1Stage),
              "l"(reinterpret_cast<uint64_t>(&x_map)), "r"(0), "r"(4 * Y0 - 2), "r"(c), "r"(img),
              "r"(smem_addr(&s_full[sl]))
              : "memory");
        }
      }
    }
  } else if (warp < 4 || warp >= 8) {
    // ---- A producers: row p of sub-plane c from the staged rows of channel c; a
    // warp's lanes take consecutive rows (cells)
    const int pw = warp < 4 ? warp - 2 : warp - 6;
    const int pt = pw * 32 + lane, n_pt = kC1ProdWarps * 32;
    const uint32_t full0 = map_to_rank(smem_addr(&a_full[0]), 0);
    uint32_t item = 0, use = 0;
    for (int t = cluster; t < tiles; t += n_clusters, ++item) {
      const int img = t / kC1Tiles, e0 = (t - img * kC1Tiles) * 256 + (int)rank * 128;
      const int Y0 = e0 / kC1SG;
      uint8_t* plane = a_s;
      for (int c = 0; c < 3; ++c, ++use) {
        const uint32_t sl = use % kC1Slots;
        if (lane == 0) {
          mbar_wait(&s_full[sl], (use / kC1Slots) & 1);                // channel c's rows landed
          if (item >= 1) mbar_wait(&a_empty[c], (item - 1) & 1);        // previous tile's c MMAs done
        }
        __syncwarp();
        const float* st = st_s + (size_t)sl * (kC1Stage / 4);
        for (int p = pt; p < ((dbg & 2) && item > 0 ? 0 : kC1P); p += n_pt) {
          const int e = e0 + p;
          const int Y = e / kC1SG, X = e - (e / kC1SG) * kC1SG;
          const bool live = e < kC1Ext;
          const float* src = st + (4 * (Y - Y0)) * kC1In + 4 * X;
          uint8_t* row = plane + c * kC1Sub + p * 64;
#pragma unroll
          for (int dy = 0; dy < 4; ++dy) {
            const float2 lo = (live && X >= 1) ? *reinterpret_cast<const float2*>(src + dy * kC1In - 2)
                                               : make_float2(0.f, 0.f);
            const float2 hi = (live && X < kC1SG - 1) ? *reinterpret_cast<const float2*>(src + dy * kC1In)
                                                      : make_float2(0.f, 0.f);
            const float4 q4 = make_float4(to_tf32(lo.x), to_tf32(lo.y), to_tf32(hi.x), to_tf32(hi.y));
            *reinterpret_cast<float4*>(row + ((dy ^ ((p >> 1) & 3)) << 4)) = q4;  // SWIZZLE_64B
          }
        }
        fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core
        __syncwarp();
        if (lane == 0) {
          // this warp is done reading the slot, and its rows of sub-plane c are ready
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&s_empty[sl])) : "memory");
          mbar_arrive_cluster(full0 + c * 8);
        }
      }
    }
  } else {
    // ---- epilogue: warp 4 + q reads TMEM lanes 32q .. 32q+31 (pixels), 96 columns,
    // in two halves of 48 channels.  Each half is staged in shared memory [pixel][48]
    // and written back pixel-major: a warp store covers 512 B of consecutive
    // 192-byte channel runs (whole sectors).  Per-lane stores of a pixel's own
    // channels hit 32 rows 384 B apart per instruction and took half the kernel
    // (profiles/conv1_debug_r2k.log: 0.217 ms, 0.111 ms with the stores off).
    const int q = warp & 3;
    const uint32_t t_empty0 = map_to_rank(smem_addr(&t_empty[0]), 0);
    float* ost = out_s + (size_t)q * (kC1Out1 / 4);
    uint32_t item = 0;
    for (int t = cluster; t < tiles; t += n_clusters, ++item) {
      const uint32_t buf = item & 1;
      const int img = t / kC1Tiles;
      const int r0 = (t - img * kC1Tiles) * 256 + (int)rank * 128 + q * 32;  // the warp's first cell
      mbar_wait(&t_full[buf], (item >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16) + buf * kC1N;
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        uint32_t v[3][16];
#pragma unroll
        for (int j = 0; j < 3; ++j) tmem_ld16_async(tb + (half * 3 + j) * 16, v[j]);
        tmem_wait_ld_regs(v[0]);
        reg_dep16(v[1]);
        reg_dep16(v[2]);
        __syncwarp();  // the previous half's copy-out reads are done
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
          for (int u = 0; u < 4; ++u)
            *reinterpret_cast<float4*>(ost + lane * kC1OutPitch + j * 16 + 4 * u) =
                make_float4(__uint_as_float(v[j][4 * u]), __uint_as_float(v[j][4 * u + 1]),
                            __uint_as_float(v[j][4 * u + 2]), __uint_as_float(v[j][4 * u + 3]));
        __syncwarp();
        if (!(dbg & 1)) {
          // 32 pixels x 12 float4 = 384 chunks; chunk g -> pixel g / 12, float4 g % 12
#pragma unroll 4
          for (int g = lane; g < 32 * 12; g += 32) {
            const int i = g / 12, f4 = g - (g / 12) * 12;
            const int r = r0 + i;
            const int Y = r / kC1SG, X = r - (r / kC1SG) * kC1SG;
            if (r < kC1Ext && Y < kC1Out && X < kC1Out) {
              float* dst = y + (((size_t)img * kC1Out + Y) * kC1Out + X) * kC1N + half * 48 + f4 * 4;
              *reinterpret_cast<float4*>(dst) = *reinterpret_cast<const float4*>(ost + i * kC1OutPitch + f4 * 4);
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(t_empty0 + buf * 8);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kC1TmemCols));
  }
}

// wq[(c*9 + ky*3 + kx)][o][dy*4 + dx] = tf32(w[o][c][4ky+dy][4kx+dx]), 0 outside 11 x 11
__global__ void k_conv1_pack_weights(const float* __restrict__ w, float* __restrict__ wq) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= kC1Blocks * kC1N * 16) return;
  const int k = i & 15, o = (i >> 4) % kC1N, blk = i / (16 * kC1N);
  const int c = blk / 9, tap = blk - 9 * c, ky = tap / 3, kx = tap - 3 * ky;
  const int r = 4 * ky + (k >> 2), s = 4 * kx + (k & 3);
  wq[i] = (r < 11 && s < 11) ? to_tf32(w[((o * 3 + c) * 11 + r) * 11 + s]) : 0.0f;
}

}  // namespace xnc

using namespace xnc;

extern "C" {

size_t xnc_conv1_weight_bytes(void) { return (size_t)kC1Blocks * kC1N * 16 * sizeof(float); }

int xnc_conv1_pack_weights(const float* w, float* wq, void* stream) {
  if (!w || !wq) return XNC_EINVAL;
  const int total = kC1Blocks * kC1N * 16;
  k_conv1_pack_weights<<<(total + 255) / 256, 256, 0, as_stream(stream)>>>(w, wq);
  return launch_status();
}

int xnc_conv1_forward(const float* x, int N, const float* wq, float* y, void* stream) {
  if (!x || !wq || !y || N < 1) return XNC_EINVAL;
  if ((reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(y) & 15) ||
      (reinterpret_cast<uintptr_t>(wq) & 15))
    return XNC_EINVAL;
  auto encode = tensor_map_encoder();
  if (!encode) return XNC_ENOTSUP;
  CUtensorMap b_map;
  cuuint64_t dims[2] = {16u, (cuuint64_t)kC1Blocks * kC1N};
  cuuint64_t strides[1] = {16u * sizeof(float)};
  cuuint32_t box[2] = {16u, (cuuint32_t)kC1Half};
  cuuint32_t estr[2] = {1u, 1u};
  if (encode(&b_map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(wq), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return XNC_ENOTSUP;
  CUtensorMap x_map;
  {
    cuuint64_t xd[4] = {(cuuint64_t)kC1In, (cuuint64_t)kC1In, 3u, (cuuint64_t)N};
    cuuint64_t xs[3] = {(cuuint64_t)kC1In * 4, (cuuint64_t)kC1In * kC1In * 4, (cuuint64_t)3 * kC1In * kC1In * 4};
    cuuint32_t xb[4] = {(cuuint32_t)kC1In, (cuuint32_t)kC1StRows, 1u, 1u};
    cuuint32_t xe[4] = {1u, 1u, 1u, 1u};
    if (encode(&x_map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(x), xd, xs, xb, xe,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return XNC_ENOTSUP;
  }
  const long tiles_l = (long)N * kC1Tiles;
  if (tiles_l > 0x7fffffffL) return XNC_EINVAL;
  const int tiles = (int)tiles_l;
  const int pairs = std::min(tiles, device_sm_count() / 2);
  if (int rc = smem_opt_in(k_conv1_tf32_pair, (size_t)kC1Smem)) return rc;
  static const int dbg = getenv("XNC_CONV1_DEBUG") ? atoi(getenv("XNC_CONV1_DEBUG")) : 0;
  k_conv1_tf32_pair<<<2 * pairs, kC1Threads, kC1Smem, as_stream(stream)>>>(x_map, N, b_map, y, tiles, dbg);
  return launch_status();
}

}  // extern "C"
