// HBM read ceiling on this B200: streaming float4 reads of an 822 MB buffer
// (the C3 input, filled with U(-1,1)-like values), (0) contiguous grid-stride, (1) K1's pattern: a thread owns 4
// consecutive pixels and walks 256 channel planes 12.5 KB apart, 8 loads in
// flight.  Prints GB/s per pattern (CUDA events, best of 5).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o hbm_read hbm_read.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_contig(const float4* __restrict__ x, long n4, float* out) {
  float s = 0.f;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
    float4 v = __ldcs(x + i);
    s += v.x + v.y + v.z + v.w;
  }
  if (s == 12345.f) out[0] = s;
}

template <int UNROLL>
__global__ void k_planes(const float* __restrict__ x, int C, int HW, long groups_per_img, long total, float* out) {
  const long gid = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= total) return;
  const long n = gid / groups_per_img;
  const int p0 = (int)(gid - n * groups_per_img) * 4;
  const float* xp = x + n * C * (long)HW + p0;
  float s = 0.f;
#pragma unroll UNROLL
  for (int c = 0; c < C; ++c) {
    float4 v = __ldcs(reinterpret_cast<const float4*>(xp + (long)c * HW));
    s += v.x + v.y + v.z + v.w;
  }
  if (s == 12345.f) out[0] = s;
}

__global__ void k_fill(float* x, long n) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    unsigned h = (unsigned)i * 2654435761u;
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
    x[i] = (float)(h & 0xFFFFFF) / 8388608.0f - 1.0f;
  }
}

int main() {
  const int N = 256, C = 256, HW = 56 * 56;
  const long n = (long)N * C * HW;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* x;
  float* out;
  cudaMalloc(&x, n * 4);
  cudaMalloc(&out, 4);
  k_fill<<<sms * 8, 256>>>(x, n);  // U(-1,1)-like values: HBM power depends on the data
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);

  auto run = [&](const char* name, auto launch) {
    float best = 1e9f;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r > 0 && ms < best) best = ms;
    }
    printf("{\"bench\": \"hbm_read\", \"pattern\": \"%s\", \"ms\": %.4f, \"GBps\": %.1f}\n", name, best, n * 4.0 / best / 1e6);
  };
  run("contig_grid_stride_148x8x256", [&] { k_contig<<<sms * 8, 256>>>(reinterpret_cast<const float4*>(x), n / 4, out); });
  run("contig_grid_stride_148x4x512", [&] { k_contig<<<sms * 4, 512>>>(reinterpret_cast<const float4*>(x), n / 4, out); });
  const long total = (long)N * HW / 4;
  run("k1_planes_256thr_u8", [&] { k_planes<8><<<(unsigned)((total + 255) / 256), 256>>>(x, C, HW, HW / 4, total, out); });
  run("k1_planes_512thr_u8", [&] { k_planes<8><<<(unsigned)((total + 511) / 512), 512>>>(x, C, HW, HW / 4, total, out); });
  run("k1_planes_128thr_u16", [&] { k_planes<16><<<(unsigned)((total + 127) / 128), 128>>>(x, C, HW, HW / 4, total, out); });
  return 0;
}
