// Probe of the tcgen05 kind::i8 building blocks the implicit-GEMM conv relies on:
//  * K-major SWIZZLE_128B smem descriptors, including a start address shifted by
//    whole 128-byte rows (the im2col tap shift) and the base_offset field;
//  * the i8 instruction descriptor (A u8, B s8, D s32, M=128, N=256);
//  * tcgen05.ld 32x32b.x32 lane/column mapping.
// Runs one CTA per (shift, base_offset policy) and checks D against a CPU GEMM.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int ROWS_A = 256 + 16;  // rows stored in smem (A), 128 B each
constexpr int M = 128, N = 256, KB = 128;  // one 128-byte K block = 4 MMAs of K=32

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr, int base_off) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                      // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;            // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                      // version = 1 (sm_100)
  d |= (uint64_t)(base_off & 7) << 49;
  d |= (uint64_t)2 << 61;                      // SWIZZLE_128B
  return d;
}

__global__ void k_probe(const uint8_t* __restrict__ A, const int8_t* __restrict__ B, int shift,
                        int base_policy, int32_t* __restrict__ D) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* a_s = smem;                       // ROWS_A x 128 (1024-aligned)
  uint8_t* b_s = smem + ROWS_A * 128;        // N x 128
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x;
  // swizzled store: 16-byte chunk q of row r goes to chunk q ^ (r & 7) (absolute-address based)
  for (int i = tid; i < ROWS_A * 8; i += blockDim.x) {
    int r = i / 8, q = i % 8;
    uint4 v = *reinterpret_cast<const uint4*>(A + r * 128 + q * 16);
    uint32_t addr = smem_u32(a_s + r * 128);
    int sw = (addr >> 7) & 7;
    *reinterpret_cast<uint4*>(a_s + r * 128 + ((q ^ sw) << 4)) = v;
  }
  for (int i = tid; i < N * 8; i += blockDim.x) {
    int r = i / 8, q = i % 8;
    uint4 v = *reinterpret_cast<const uint4*>(B + r * 128 + q * 16);
    uint32_t addr = smem_u32(b_s + r * 128);
    int sw = (addr >> 7) & 7;
    *reinterpret_cast<uint4*>(b_s + r * 128 + ((q ^ sw) << 4)) = v;
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" :: "r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // generic-proxy smem writes -> visible to the tensor core (async proxy)
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  if (tid == 0) {
    uint32_t a0 = smem_u32(a_s) + shift * 128;
    uint32_t b0 = smem_u32(b_s);
    for (int s = 0; s < KB / 32; ++s) {
      uint32_t aa = a0 + s * 32;
      int boff = base_policy == 0 ? 0 : (int)((aa >> 7) & 7);
      uint64_t ad = desc_sw128(aa, boff);
      uint64_t bd = desc_sw128(b0 + s * 32, 0);
      uint32_t acc = s > 0;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                   :: "r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&mbar)));
  }
  // wait for the MMAs
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int warp = tid / 32, lane = tid % 32;
  if (warp < 4) {
    for (int c0 = 0; c0 < N; c0 += 32) {
      uint32_t v[32];
      uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                   "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                     "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                     "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                     "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                   : "r"(addr));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int j = 0; j < 32; ++j) D[(warp * 32 + lane) * N + c0 + j] = (int32_t)v[j];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" :: "r"(tmem));
}


// Throughput: every CTA issues `iters` x 4 MMAs (M=128, N=256, K=32) from resident smem.
// random != 0: A bytes random 0/1 (the d-byte operand), B bytes random +-1 (the
// filter signs) instead of constant 0x01 -- tensor-core power is data dependent.
__global__ void k_rate(int iters, int n_mma, int shift, int32_t* out, int random) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x;
  for (int i = tid; i < (128 + 16 + 256) * 128 / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u + blockIdx.x * 97u;
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
    uint32_t v = 0x01010101u;
    if (random) {
      if (i < (128 + 16) * 128 / 4) v = h & 0x01010101u;                       // A: 0/1
      else v = 0x01010101u | ((h & 0x01010101u) * 0xFEu);                    // B: 0x01 or 0xFF
    }
    reinterpret_cast<uint32_t*>(smem)[i] = v;
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(n_mma >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (tid == 0) {
    uint32_t a0 = smem_u32(smem) + shift * 128, b0 = smem_u32(smem) + (128 + 16) * 128;
    for (int it = 0; it < iters; ++it)
      for (int s = 0; s < 4; ++s) {
        uint64_t ad = desc_sw128(a0 + s * 32, 0), bd = desc_sw128(b0 + s * 32, 0);
        uint32_t acc = (it | s) != 0;
        uint32_t d = tmem + (it & 1) * n_mma;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                     :: "r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&mbar)));
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tmem));
  if (tid == 0 && iters < 0) out[0] = 1;
}

int main() {
  std::vector<uint8_t> A(ROWS_A * 128);
  std::vector<int8_t> B(N * 128);
  srand(1);
  for (auto& a : A) a = rand() & 1;
  for (auto& b : B) { int r = rand() % 3; b = (int8_t)(r - 1); }
  uint8_t* dA; int8_t* dB; int32_t* dD;
  CK(cudaMalloc(&dA, A.size())); CK(cudaMalloc(&dB, B.size())); CK(cudaMalloc(&dD, M * N * 4));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  size_t smem = ROWS_A * 128 + N * 128 + 1024;
  CK(cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  std::vector<int32_t> D(M * N);
  for (int policy = 0; policy < 2; ++policy)
    for (int shift = 0; shift < 10; ++shift) {
      CK(cudaMemset(dD, 0x7f, M * N * 4));
      k_probe<<<1, 128, smem>>>(dA, dB, shift, policy, dD);
      CK(cudaGetLastError());
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost));
      long bad = 0;
      for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
          int ref = 0;
          for (int k = 0; k < KB; ++k) ref += (int)A[(m + shift) * 128 + k] * (int)B[n * 128 + k];
          if (ref != D[m * N + n]) ++bad;
        }
      printf("{\"probe\": \"umma_i8_sw128\", \"base_offset_policy\": %d, \"row_shift\": %d, \"mismatches\": %ld}\n",
             policy, shift, bad);
    }
  // ---- tcgen05 i8 throughput (UTCIMMA), 1 CTA per SM
  {
    int dev; cudaGetDevice(&dev); cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
    int clk_khz; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    size_t sm2 = (128 + 16 + 256) * 128 + 1024;
    CK(cudaFuncSetAttribute(k_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2));
    for (int random : {0, 1})
    for (int shift : {0, 1, 3, 8})
    for (int n_mma : {256, 128}) {
      int iters = 20000 * 256 / n_mma;
      for (int w = 0; w < 2; ++w) k_rate<<<p.multiProcessorCount, 128, sm2>>>(iters, n_mma, shift, dD, random);
      CK(cudaDeviceSynchronize());
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      float best = 1e30f;
      for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        k_rate<<<p.multiProcessorCount, 128, sm2>>>(iters, n_mma, shift, dD, random);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      double macs = (double)p.multiProcessorCount * iters * 4 * 128.0 * n_mma * 32;
      printf("{\"bench\": \"tcgen05_i8_m128n%dk32\", \"random_data\": %d, \"a_row_shift\": %d, \"ms\": %.4f, \"rate\": %.4e, \"unit\": \"MAC/s\", "
             "\"per_sm_per_clk_at_max\": %.1f, \"sms\": %d}\n", n_mma, random, shift, best, macs / (best * 1e-3),
             macs / (best * 1e-3) / p.multiProcessorCount / (clk_khz * 1e3), p.multiProcessorCount);
    }
  }
  return 0;
}
