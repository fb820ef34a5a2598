// Does a SWIZZLE_128B TMA tile load into a shared-memory destination that is
// only 128-byte aligned (not 1024) place the data by the absolute-address
// swizzle (16-byte chunk q of the row at address a stored at chunk q ^ ((a >> 7) & 7))?
// The 2-CTA conv kernel needs this to give both CTAs of a pair the same A
// descriptor.  Prints one JSON line per destination offset.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tma_align tma_align.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int C = 128, W = 58, H = 8, ROWS = 4;

__global__ void k_load(const __grid_constant__ CUtensorMap map, int dst_off, uint8_t* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024 - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023)) & 1023);
  uint8_t* dst = base + dst_off;
  __shared__ __align__(8) uint64_t bar;
  const uint32_t bar_a = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
  for (int i = threadIdx.x; i < (ROWS * W * C + 2048) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0xEEEEEEEEu;
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_a));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_a), "r"(ROWS * W * C));
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
            static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
        "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(0), "r"(2), "r"(0), "r"(bar_a)
        : "memory");
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"(bar_a), "r"(0) : "memory");
  }
  __syncthreads();
  for (int i = threadIdx.x; i < ROWS * W * C; i += blockDim.x) out[i] = dst[i];
  if (threadIdx.x == 0) out[ROWS * W * C] = (uint8_t)((static_cast<uint32_t>(__cvta_generic_to_shared(dst)) >> 7) & 7);
}

int main() {
  std::vector<uint8_t> h((size_t)H * W * C);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (uint8_t)(i * 7 + (i >> 7) * 13 + 1);
  uint8_t *d_in, *d_out;
  cudaMalloc(&d_in, h.size());
  cudaMalloc(&d_out, ROWS * W * C + 16);
  cudaMemcpy(d_in, h.data(), h.size(), cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap map;
  cuuint64_t dims[4] = {C, W, H, 1};
  cuuint64_t strides[3] = {C, (cuuint64_t)W * C, (cuuint64_t)H * W * C};
  cuuint32_t box[4] = {C, W, ROWS, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, d_in, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("{\"error\": \"encode %d\"}\n", (int)r); return 1; }
  cudaFuncSetAttribute(k_load, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  std::vector<uint8_t> o(ROWS * W * C + 16);
  for (int off : {0, 128, 384, 640, 896, 1024 + 256}) {
    cudaMemset(d_out, 0, o.size());
    k_load<<<1, 256, 64 * 1024>>>(map, off, d_out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("{\"dst_off\": %d, \"error\": \"%s\"}\n", off, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(o.data(), d_out, o.size(), cudaMemcpyDeviceToHost);
    const int phase0 = o[ROWS * W * C];  // (address >> 7) & 7 of the destination
    long bad_abs = 0, bad_rel = 0;
    for (int row = 0; row < ROWS * W; ++row)
      for (int qq = 0; qq < 8; ++qq)
        for (int b = 0; b < 16; ++b) {
          const uint8_t want = h[(size_t)(2 * W + row) * C + qq * 16 + b];  // rows start at image row 2
          const int q_abs = qq ^ ((phase0 + row) & 7), q_rel = qq ^ (row & 7);
          if (o[(size_t)row * C + q_abs * 16 + b] != want) ++bad_abs;
          if (o[(size_t)row * C + q_rel * 16 + b] != want) ++bad_rel;
        }
    printf("{\"probe\": \"tma_sw128_dst_alignment\", \"dst_off\": %d, \"addr_phase\": %d, \"mismatch_abs_swizzle\": %ld, "
           "\"mismatch_rel_swizzle\": %ld}\n", off, phase0, bad_abs, bad_rel);
  }
  return 0;
}
