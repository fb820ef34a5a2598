// tcgen05.mma.cta_group::2.kind::mxf4 (E2M1 x E2M1, UE8M0 block-32 scales, f32
// accumulator) with every scale = 1.0: (1) exactness of integer-valued dot
// products of {0, 1} x {-1, +1} operands against the host, including K = 9216
// accumulated over 36 chunks (fc6's K), and (2) SM cycles per MMA for M = 256
// (pair) x N in {256, 128} x K = 64, next to the same loop on kind::i8 (K = 32).
// A 128-byte K row holds 256 E2M1 values (kind::mxf4) or 128 bytes (kind::i8), so
// equal cycles per MMA mean twice the MAC rate.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mxf4_probe mxf4_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void wait_bar(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(smem_u32(b)), "r"(par) : "memory");
}

constexpr uint32_t kSfCol = 256 + 128;  // scale-factor columns (after two 128/256-column accumulators)

// KIND 0: mxf4 block-scaled, KIND 1: i8 (u8 x s8).  a/b: per CTA 128 rows x 128 B, logical
// (unswizzled) order.  reps: chunks (4 MMAs each) accumulated.  out: [2][128][NP] f32 / s32.
template <int NP, int KIND>
__global__ void __cluster_dims__(2, 1, 1) k_probe(const uint8_t* a, const uint8_t* b, int reps, int rate, float* out,
                                                  long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* a_s = smem;                 // 128 rows x 128 B
  uint8_t* b_s = smem + 128 * 128;     // 128 rows x 128 B (NP/2 used)
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t done_bar;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 128 * 128; i += blockDim.x) {
    const int r = i >> 7, c = i & 127;
    const int phys = r * 128 + ((((c >> 4) ^ (r & 7)) << 4) | (c & 15));
    a_s[phys] = a[rank * 128 * 128 + i];
    b_s[phys] = b[rank * 128 * 128 + i];
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&done_bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  // scale factors: 0x7F (2^0) in every byte of 32 columns x 128 lanes
  {
    const uint32_t t = tmem + ((uint32_t)(warp * 32) << 16) + kSfCol;
    const uint32_t v = 0x7F7F7F7Fu;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
                 "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(t), "r"(v) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t idesc;
  if (KIND == 0)
    idesc = (1u << 7) | (1u << 10) | ((uint32_t)(NP >> 3) << 17) | (1u << 23) | ((uint32_t)(256 >> 4) << 24);
  else
    idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(NP >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
  if (rank == 0 && warp == 0) {
    const uint64_t a0 = desc_sw128(smem_u32(a_s)), b0 = desc_sw128(smem_u32(b_s));
    const uint32_t sf = tmem + kSfCol;
    const long long t0 = clock64();
    for (int g = 0; g < reps; ++g) {
      const uint32_t d = tmem + (rate ? (uint32_t)(g & 1) * (uint32_t)NP : 0u);
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const uint32_t acc = (rate ? g >= 2 : g > 0) || s > 0;
        if (KIND == 0)
          asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%5], p;\n\t}"
                       ::"r"(d), "l"(a0 + 2 * s), "l"(b0 + 2 * s), "r"(idesc), "r"(acc), "r"(sf));
        else
          asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                       ::"r"(d), "l"(a0 + 2 * s), "l"(b0 + 2 * s), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
                 ::"r"(smem_u32(&done_bar)), "h"((uint16_t)3) : "memory");
    wait_bar(&done_bar, 0);
    if (lane == 0) cyc[blockIdx.x / 2] = clock64() - t0;
  } else if (tid == 0) {
    wait_bar(&done_bar, 0);
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (!rate) {
    // warp w reads lanes 32w..32w+31 of the accumulator: columns 0..NP-1
    for (int c0 = 0; c0 < NP; c0 += 16) {
      uint32_t r[16];
      const uint32_t t = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                     "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                   : "r"(t));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int j = 0; j < 16; ++j) {
        const float v = KIND == 0 ? __uint_as_float(r[j]) : (float)(int32_t)r[j];
        out[((size_t)rank * 128 + warp * 32 + lane) * NP + c0 + j] = v;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

static float e2m1(uint32_t nib) {
  static const float mag[8] = {0.f, 0.5f, 1.f, 1.5f, 2.f, 3.f, 4.f, 6.f};
  return (nib & 8) ? -mag[nib & 7] : mag[nib & 7];
}

// host operands: A = d in {0, 1} (+ a few 0.5 / 2 to expose nibble order), B = +-1 (0 for some)
template <int NP, int KIND>
bool check(int reps, uint32_t seed, bool all_ones) {
  const size_t n = 2 * 128 * 128;
  uint8_t *ha = (uint8_t*)malloc(n), *hb = (uint8_t*)malloc(n);
  uint32_t s = seed;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return s >> 8; };
  for (size_t i = 0; i < n; ++i) {
    if (KIND == 0) {
      uint8_t x = 0, y = 0;
      for (int h = 0; h < 2; ++h) {
        const uint32_t ra = rnd(), rb = rnd();
        const uint32_t na = all_ones ? 0x2 : ((ra & 1) ? 0x2 : 0x0);
        const uint32_t nb = all_ones ? 0x2 : ((rb & 15) == 0 ? 0x0 : ((rb & 2) ? 0x2 : 0xA));
        x |= na << (4 * h);
        y |= nb << (4 * h);
      }
      ha[i] = x;
      hb[i] = y;
    } else {
      ha[i] = all_ones ? 1 : (rnd() & 1);
      const uint32_t rb = rnd();
      hb[i] = all_ones ? 1 : (uint8_t)(int8_t)((rb & 15) == 0 ? 0 : ((rb & 2) ? 1 : -1));
    }
  }
  uint8_t *da, *db;
  float* dout;
  long long* dcyc;
  CK(cudaMalloc(&da, n)); CK(cudaMalloc(&db, n));
  CK(cudaMalloc(&dout, sizeof(float) * 256 * NP)); CK(cudaMalloc(&dcyc, 8 * 128));
  CK(cudaMemcpy(da, ha, n, cudaMemcpyHostToDevice)); CK(cudaMemcpy(db, hb, n, cudaMemcpyHostToDevice));
  const size_t smem = 2 * 128 * 128 + 1024;
  CK(cudaFuncSetAttribute(k_probe<NP, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_probe<NP, KIND><<<2, 128, smem>>>(da, db, reps, 0, dout, dcyc);
  CK(cudaDeviceSynchronize());
  float* hout = (float*)malloc(sizeof(float) * 256 * NP);
  CK(cudaMemcpy(hout, dout, sizeof(float) * 256 * NP, cudaMemcpyDeviceToHost));
  long bad = 0;
  double maxabs = 0;
  for (int m = 0; m < 256; ++m)
    for (int nn = 0; nn < NP; ++nn) {
      // row m of A lives in CTA m/128 row m%128; filter nn in CTA nn/(NP/2) row nn%(NP/2)
      const uint8_t* ar = ha + (size_t)(m / 128) * 128 * 128 + (size_t)(m % 128) * 128;
      const uint8_t* br = hb + (size_t)(nn / (NP / 2)) * 128 * 128 + (size_t)(nn % (NP / 2)) * 128;
      double ref = 0;
      for (int c = 0; c < 128; ++c) {
        if (KIND == 0)
          ref += e2m1(ar[c] & 15) * e2m1(br[c] & 15) + e2m1(ar[c] >> 4) * e2m1(br[c] >> 4);
        else
          ref += (double)ar[c] * (double)(int8_t)br[c];
      }
      ref *= reps;
      const float got = hout[(size_t)m * NP + nn];
      if (got != (float)ref) {
        if (bad < 5) printf("  mismatch m=%d n=%d got %.1f want %.1f\n", m, nn, got, ref);
        ++bad;
      }
      if (fabs(ref) > maxabs) maxabs = fabs(ref);
    }
  printf("{\"bench\": \"mxf4_probe\", \"check\": \"%s\", \"NP\": %d, \"reps\": %d, \"all_ones\": %d, \"max_abs\": %.0f, "
         "\"mismatches\": %ld}\n", KIND == 0 ? "mxf4" : "i8", NP, reps, (int)all_ones, maxabs, bad);
  free(ha); free(hb); free(hout);
  CK(cudaFree(da)); CK(cudaFree(db)); CK(cudaFree(dout)); CK(cudaFree(dcyc));
  return bad == 0;
}

template <int NP, int KIND>
void rate(int sms) {
  const size_t n = 2 * 128 * 128;
  uint8_t *da, *db;
  float* dout;
  long long* dcyc;
  CK(cudaMalloc(&da, n)); CK(cudaMalloc(&db, n));
  CK(cudaMemset(da, KIND == 0 ? 0x22 : 1, n)); CK(cudaMemset(db, KIND == 0 ? 0xA2 : 0xFF, n));
  CK(cudaMalloc(&dout, 4)); CK(cudaMalloc(&dcyc, 8 * 128));
  const size_t smem = 2 * 128 * 128 + 1024;
  CK(cudaFuncSetAttribute(k_probe<NP, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int reps = 20000;
  k_probe<NP, KIND><<<sms, 128, smem>>>(da, db, reps, 1, dout, dcyc);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_probe<NP, KIND><<<sms, 128, smem>>>(da, db, reps, 1, dout, dcyc);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long cyc[128];
  CK(cudaMemcpy(cyc, dcyc, 8 * (sms / 2), cudaMemcpyDeviceToHost));
  double c = 0;
  for (int i = 0; i < sms / 2; ++i) c += (double)cyc[i] / (sms / 2);
  const double mmas = (double)reps * 4;
  const double k = KIND == 0 ? 64 : 32;
  const double macs_per_sm_clk = 128.0 * NP * k / (c / mmas);
  printf("{\"bench\": \"mxf4_probe\", \"rate\": \"%s\", \"NP\": %d, \"ms\": %.3f, \"sm_cycles_per_mma\": %.2f, "
         "\"mac_per_clk_per_sm\": %.0f, \"sm_clock_ghz\": %.3f, \"tmacs\": %.1f}\n",
         KIND == 0 ? "mxf4" : "i8", NP, ms, c / mmas, macs_per_sm_clk, c / (ms * 1e-3) / 1e9,
         (double)sms / 2 * 256.0 * NP * k * mmas / (ms * 1e-3) / 1e12);
  CK(cudaFree(da)); CK(cudaFree(db)); CK(cudaFree(dout)); CK(cudaFree(dcyc));
}

int main() {
  int dev; cudaGetDevice(&dev);
  cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  bool ok = true;
  ok &= check<256, 1>(1, 1, false);
  ok &= check<256, 0>(1, 1, false);
  ok &= check<128, 0>(1, 2, false);
  ok &= check<256, 0>(36, 3, false);
  ok &= check<256, 0>(36, 4, true);  // 9216 in every accumulator
  ok &= check<256, 0>(64, 5, true);  // 16384
  rate<256, 1>(p.multiProcessorCount);
  rate<256, 0>(p.multiProcessorCount);
  rate<128, 1>(p.multiProcessorCount);
  rate<128, 0>(p.multiProcessorCount);
  printf("{\"bench\": \"mxf4_probe\", \"all_exact\": %s}\n", ok ? "true" : "false");
  return ok ? 0 : 2;
}
