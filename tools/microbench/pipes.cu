// Pipe-throughput microbenchmarks for the XNOR-conv roofline (sm_100a).
// Measures lanes/clk/SM for POPC, LOP3, IADD3, the xor+popc+add mix, and
// legacy mma.sync int8 / b1 rates.  Each kernel runs many independent
// chains so the measured number is throughput, not latency.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;

__global__ void k_popc(uint32_t* out, uint32_t seed) {
  uint32_t v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = seed * (threadIdx.x + i * 7919u);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) asm volatile("popc.b32 %0, %0;" : "+r"(v[i]));
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += v[i];
  if (s == 0xdeadbeef) out[0] = s;
}

__global__ void k_lop3(uint32_t* out, uint32_t seed) {
  uint32_t v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = seed * (threadIdx.x + i * 7919u);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) asm volatile("xor.b32 %0, %0, %1;" : "+r"(v[i]) : "r"(seed));
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += v[i];
  if (s == 0xdeadbeef) out[0] = s;
}

// xor + popc + add per word pair, 16 independent accumulators; weights vary
// per iteration through a register rotate so nothing is loop-invariant.
__global__ void k_mix(uint32_t* out, uint32_t seed) {
  uint32_t a[4], w[4], acc[16];
#pragma unroll
  for (int i = 0; i < 4; ++i) { a[i] = seed * (threadIdx.x + i); w[i] = seed ^ (i * 0x9e3779b9u); }
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = 0;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int f = 0; f < 4; ++f) {
        uint32_t x, c;
        asm volatile("xor.b32 %0, %1, %2;" : "=r"(x) : "r"(a[p]), "r"(w[f]));
        asm volatile("popc.b32 %0, %1;" : "=r"(c) : "r"(x));
        acc[p * 4 + f] += c;
      }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 0xdeadbeef) out[0] = s;
}

__global__ void k_imma_s8(uint32_t* out, uint32_t seed) {
  uint32_t a0 = seed, a1 = seed * 3, a2 = seed * 5, a3 = seed * 7, b0 = seed * 11, b1 = seed * 13;
  int d[8][4] = {};
  for (int it = 0; it < ITERS / 8; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(d[i][0]), "+r"(d[i][1]), "+r"(d[i][2]), "+r"(d[i][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1] + d[i][2] + d[i][3];
  if (s == 0x12345) out[0] = s;
}

__global__ void k_b1_xor(uint32_t* out, uint32_t seed) {
  uint32_t a0 = seed, a1 = seed * 3, a2 = seed * 5, a3 = seed * 7, b0 = seed * 11, b1 = seed * 13;
  int d[8][4] = {};
  for (int it = 0; it < ITERS / 8; ++it) {
    a0 += it; b0 ^= it;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.xor.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(d[i][0]), "+r"(d[i][1]), "+r"(d[i][2]), "+r"(d[i][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1] + d[i][2] + d[i][3];
  if (s == 0x12345) out[0] = s;
}

__global__ void k_b1_and(uint32_t* out, uint32_t seed) {
  uint32_t a0 = seed, a1 = seed * 3, a2 = seed * 5, a3 = seed * 7, b0 = seed * 11, b1 = seed * 13;
  int d[8][4] = {};
  for (int it = 0; it < ITERS / 8; ++it) {
    a0 += it; b0 ^= it;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(d[i][0]), "+r"(d[i][1]), "+r"(d[i][2]), "+r"(d[i][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1] + d[i][2] + d[i][3];
  if (s == 0x12345) out[0] = s;
}

__global__ void k_hmma(uint32_t* out, uint32_t seed) {
  uint32_t a0 = seed, a1 = seed * 3, a2 = seed * 5, a3 = seed * 7, b0 = seed * 11, b1 = seed * 13;
  float d[8][4] = {};
  for (int it = 0; it < ITERS / 8; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(d[i][0]), "+f"(d[i][1]), "+f"(d[i][2]), "+f"(d[i][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1] + d[i][2] + d[i][3];
  if (s == 1234.5f) out[0] = 1;
}

typedef void (*kfn)(uint32_t*, uint32_t);

static int run(const char* name, kfn k, double ops_per_thread, const char* unit, int blocks_per_sm, int threads) {
  int dev; cudaGetDevice(&dev);
  cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int clk_khz; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  uint32_t* out; CK(cudaMalloc(&out, 4));
  int grid = p.multiProcessorCount * blocks_per_sm;
  for (int w = 0; w < 3; ++w) k<<<grid, threads>>>(out, 0x1234567u + w);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k<<<grid, threads>>>(out, 0x7654321u + r);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  double total = ops_per_thread * grid * (double)threads;
  double per_s = total / (best * 1e-3);
  // per SM per clock at the nominal max clock (the run may be below it)
  double per_sm_clk = per_s / p.multiProcessorCount / (clk_khz * 1e3);
  printf("{\"bench\": \"%s\", \"ms\": %.4f, \"rate\": %.4e, \"unit\": \"%s/s\", \"per_sm_per_clk_at_max\": %.2f, \"sms\": %d, \"max_clk_mhz\": %.0f}\n",
         name, best, per_s, unit, per_sm_clk, p.multiProcessorCount, clk_khz / 1e3);
  cudaFree(out);
  return 0;
}

int main() {
  run("popc", k_popc, 16.0 * ITERS, "lane-op", 4, 256);
  run("lop3_xor", k_lop3, 16.0 * ITERS, "lane-op", 4, 256);
  run("xor_popc_add_pairs", k_mix, 16.0 * ITERS, "word-pair", 4, 256);
  // per warp-level mma: m16n8k32 = 4096 MAC; per thread = 4096/32 = 128 MAC
  run("mma_sync_s8_m16n8k32", k_imma_s8, (ITERS / 8) * 8 * 128.0, "MAC", 4, 256);
  run("mma_sync_b1_xor_m16n8k256", k_b1_xor, (ITERS / 8) * 8 * 1024.0, "bitMAC", 4, 256);
  run("mma_sync_b1_and_m16n8k256", k_b1_and, (ITERS / 8) * 8 * 1024.0, "bitMAC", 4, 256);
  run("mma_sync_bf16_m16n8k16", k_hmma, (ITERS / 8) * 8 * 64.0, "MAC", 4, 256);
  return 0;
}
