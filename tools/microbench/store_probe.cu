// Output-store rate of the tcgen05 conv's epilogue pattern, without the conv: the
// C3 output (256 images x 256 filters x 56*56 pixels, f32 NCHW, 822 MB) written by
// one persistent CTA per SM in (128-pixel tile, 16-filter chunk) pieces.
//   fill      float4 grid-stride stores (the HBM write ceiling)
//   stg<W>    W epilogue warps; a warp owns 32 pixels and stores 16 filters per chunk,
//             one coalesced st.global.cs.f32 per filter (the kernel's current epilogue)
//   bulk<W>   the four quadrant warps of a chunk stage 16 filters x 128 pixels in shared
//             memory (one STS per output), then 16 lanes issue one cp.async.bulk each
//             (a filter's 128 pixels are 512 contiguous bytes of its plane); two staging
//             buffers per chunk group, reused after cp.async.bulk.wait_group.read
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o store_probe store_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int kImg = 256, kFilt = 256, kPix = 56 * 56, kTile = 128;
constexpr int kTilesPerImg = (kPix + kTile - 1) / kTile;

__global__ void k_fill(float4* y, long n4, float v) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x)
    __stcs(y + i, make_float4(v, v + 1, v + 2, v + 3));
}

__device__ __forceinline__ void st_cs(float* p, float v, bool pred) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.cs.f32 [%0], %1;\n\t}" ::"l"(p), "f"(v),
               "r"((int)pred) : "memory");
}

template <int W>
__global__ void __launch_bounds__(W * 32, 1) k_stg(float* y, float v) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int quad = warp & 3, cg = warp >> 2;
  constexpr int cstep = W / 4;
  const int units = kImg * kTilesPerImg;
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    const int n = u / kTilesPerImg, t = u - n * kTilesPerImg;
    const int p = t * kTile + quad * 32 + lane;
    const bool in = p < kPix;
    float* base = y + ((size_t)n * kFilt) * kPix + p;
    for (int c = cg; c < kFilt / 16; c += cstep) {
#pragma unroll
      for (int j = 0; j < 16; ++j) st_cs(base + (size_t)(c * 16 + j) * kPix, v * (float)(j + 1) + (float)p, in);
    }
  }
}

template <int W>
__global__ void __launch_bounds__(W * 32, 1) k_bulk(float* y, float v) {
  // per chunk group: 2 buffers x 16 filters x 128 pixels
  extern __shared__ __align__(128) float stage[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int quad = warp & 3, cg = warp >> 2;
  constexpr int cstep = W / 4;
  const int units = kImg * kTilesPerImg;
  float* my = stage + (size_t)cg * 2 * 16 * kTile;
  uint32_t it = 0;
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    const int n = u / kTilesPerImg, t = u - n * kTilesPerImg;
    const int p0 = t * kTile;
    const int np = min(kTile, kPix - p0);
    const int p = p0 + quad * 32 + lane;
    for (int c = cg; c < kFilt / 16; c += cstep, ++it) {
      float* buf = my + (it & 1) * 16 * kTile;
      // the copies that read this buffer two chunks ago must be done reading
      if (quad == 0 && lane < 16) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      asm volatile("bar.sync %0, 128;" ::"r"(1 + cg) : "memory");
#pragma unroll
      for (int j = 0; j < 16; ++j) buf[j * kTile + quad * 32 + lane] = v * (float)(j + 1) + (float)p;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync %0, 128;" ::"r"(1 + cg) : "memory");
      if (quad == 0 && lane < 16) {
        float* dst = y + ((size_t)n * kFilt + c * 16 + lane) * kPix + p0;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                     "r"((uint32_t)__cvta_generic_to_shared(buf + lane * kTile)), "r"((uint32_t)(np * 4)) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
  }
  if (quad == 0 && lane < 16) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <class F>
float time_it(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  f();
  cudaDeviceSynchronize();
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  int dev; cudaGetDevice(&dev);
  cudaDeviceProp prop; cudaGetDeviceProperties(&prop, dev);
  const int sms = prop.multiProcessorCount;
  const size_t n = (size_t)kImg * kFilt * kPix;
  float* y;
  CK(cudaMalloc(&y, n * 4));
  const double gb = n * 4 / 1e9;
  auto rep = [&](const char* name, float ms) {
    printf("{\"bench\": \"store_probe\", \"kernel\": \"%s\", \"ms\": %.4f, \"GBs\": %.0f}\n", name, ms, gb / (ms * 1e-3));
  };
  rep("fill_float4", time_it([&] { k_fill<<<sms * 8, 256>>>(reinterpret_cast<float4*>(y), (long)(n / 4), 1.f); }));
  rep("stg_w8", time_it([&] { k_stg<8><<<sms, 256>>>(y, 1.f); }));
  rep("stg_w16", time_it([&] { k_stg<16><<<sms, 512>>>(y, 1.f); }));
  rep("stg_w32", time_it([&] { k_stg<32><<<sms, 1024>>>(y, 1.f); }));
  {
    const size_t sm8 = 2 * 2 * 16 * kTile * 4, sm16 = 4 * 2 * 16 * kTile * 4;
    CK(cudaFuncSetAttribute(k_bulk<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm8));
    CK(cudaFuncSetAttribute(k_bulk<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm16));
    rep("bulk_w8", time_it([&] { k_bulk<8><<<sms, 256, sm8>>>(y, 1.f); }));
    rep("bulk_w16", time_it([&] { k_bulk<16><<<sms, 512, sm16>>>(y, 1.f); }));
  }
  CK(cudaGetLastError());
  // check a few bulk outputs
  float h[4];
  CK(cudaMemcpy(h, y + (size_t)3 * kPix + 100, 16, cudaMemcpyDeviceToHost));
  printf("{\"bench\": \"store_probe\", \"sample\": [%.1f, %.1f], \"want\": [%.1f, %.1f]}\n", h[0], h[1], 4.f + 100, 4.f + 101);
  return 0;
}
