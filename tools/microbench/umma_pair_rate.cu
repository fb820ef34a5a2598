// tcgen05.mma.cta_group::2.kind::i8 rate on CTA pairs (cluster of 2): SM cycles
// per (128x128x32 per SM) of MMA work, for M=256 and N in {128, 256}, with and
// without the per-group pipeline protocol (try_wait + fence before, multicast
// commit after every 4 MMAs).  Resident random operands, no memory traffic.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o umma_pair_rate umma_pair_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// MODE 0: back-to-back MMAs; MODE 1: per group of 4: try_wait(done barrier) + fence, commit multicast;
// MODE 2: as 1 but the wait sits between the group's 2nd and 3rd MMA; MODE 3: as 1 with a
// commit only (no wait); MODE 4: as 1 with a wait only (no commit).  out[64 + pair] = cycles
// spent inside the waits.  MODE 5: as 0 but every MMA accumulates into the same
// accumulator; MODE 6: as 0 alternating the accumulator on every MMA; MODE 7: as 1 with one accumulator.
template <int NP, int MODE>
__global__ void __cluster_dims__(2, 1, 1) k_pair(int n_groups, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t done_bar, cbar, ready;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int tid = threadIdx.x;
  for (int i = tid; i < (512 + 6 * 128) * 32; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u + blockIdx.x * 97u;
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
    reinterpret_cast<uint32_t*>(smem)[i] = i < 512 * 32 ? (h & 0x01010101u) : (0x01010101u | ((h & 0x01010101u) * 0xFEu));
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&done_bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&cbar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&ready)));
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&ready)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(NP >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
  if (rank == 0 && tid == 0) {
    const uint64_t a0 = desc_sw128(smem_u32(smem)), b0 = desc_sw128(smem_u32(smem + 512 * 128));
    const long long t0 = clock64();
    long long tw = 0;
    auto wait_ready = [&]() {
      const long long a = clock64();
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(&ready)), "r"(0) : "memory");
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      tw += clock64() - a;
    };
    for (int g = 0; g < n_groups; ++g) {
      if (MODE == 1 || MODE == 4 || MODE == 7) wait_ready();
      const int tap = g % 9;
      const uint64_t a = a0 + (uint32_t)((tap / 3) * 58 + tap % 3) * 8u;
      const uint64_t b = b0 + (uint32_t)(g % 6) * (64 * 128 / 16);
      const uint32_t d = tmem + ((MODE == 5 || MODE == 7) ? 0u : (g & 1) * NP);
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        if (MODE == 2 && s == 2) wait_ready();
        const uint32_t dd = MODE == 6 ? tmem + (s & 1) * NP : d;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(dd), "l"(a + 2 * s), "l"(b + 2 * s), "r"(idesc), "r"((uint32_t)(g >= 2 || s > 0)));
      }
      if (MODE == 1 || MODE == 2 || MODE == 3 || MODE == 7)
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                     ::"r"(smem_u32(&cbar)), "h"((uint16_t)3) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(smem_u32(&done_bar)), "h"((uint16_t)3) : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&done_bar)), "r"(0) : "memory");
    out[blockIdx.x / 2] = clock64() - t0;
    out[128 + blockIdx.x / 2] = tw;
  } else if (rank == 1 && tid == 0) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&done_bar)), "r"(0) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (tid < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int NP, int MODE>
int run(int sms, long long* d_out) {
  const size_t smem = (512 + 6 * 128) * 128 + 1024;
  CK(cudaFuncSetAttribute(k_pair<NP, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int n_groups = 40000 * 256 / NP;
  k_pair<NP, MODE><<<sms, 128, smem>>>(n_groups, d_out);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_pair<NP, MODE><<<sms, 128, smem>>>(n_groups, d_out);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long cyc[256];
  CK(cudaMemcpy(cyc, d_out, sizeof(long long) * 256, cudaMemcpyDeviceToHost));
  double c = 0, w = 0;
  for (int i = 0; i < sms / 2; ++i) { c += (double)cyc[i] / (sms / 2); w += (double)cyc[128 + i] / (sms / 2); }
  // per SM: each MMA = 128 rows x NP x 32 -> NP/128 units of 128x128x32
  const double units = (double)n_groups * 4 * NP / 128;
  printf("{\"bench\": \"umma_pair_rate\", \"NP\": %d, \"protocol\": %d, \"ms\": %.3f, \"sm_cycles_per_128x128x32\": %.2f, "
         "\"wait_cycles_per_group\": %.1f, \"sm_clock_ghz\": %.3f}\n", NP, MODE, ms, c / units, w / n_groups,
         c / (ms * 1e-3) / 1e9);
  return 0;
}

int main() {
  int dev; cudaGetDevice(&dev);
  cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  long long* d_out; CK(cudaMalloc(&d_out, 4096));
  run<256, 0>(p.multiProcessorCount, d_out); run<256, 1>(p.multiProcessorCount, d_out);
  run<256, 2>(p.multiProcessorCount, d_out); run<256, 3>(p.multiProcessorCount, d_out);
  run<256, 4>(p.multiProcessorCount, d_out); run<256, 5>(p.multiProcessorCount, d_out);
  run<256, 6>(p.multiProcessorCount, d_out); run<256, 7>(p.multiProcessorCount, d_out);
  run<128, 0>(p.multiProcessorCount, d_out); run<128, 1>(p.multiProcessorCount, d_out);
  run<128, 2>(p.multiProcessorCount, d_out); run<128, 3>(p.multiProcessorCount, d_out);
  run<128, 4>(p.multiProcessorCount, d_out);
  return 0;
}
