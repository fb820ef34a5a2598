// Shared helpers for the sm_100a XNOR-conv kernels (libxnorb200.so).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/xnorb200.h"

namespace xnc {

constexpr int kMaxK = 8;  // reference: kernel must fit an 8x8 (64-bit) tile, pack.py:45-53

__host__ __device__ inline int cdiv(int a, int b) { return (a + b - 1) / b; }
__host__ __device__ inline long cdivl(long a, long b) { return (a + b - 1) / b; }
__host__ __device__ inline int round_up(int a, int b) { return cdiv(a, b) * b; }

// Word j of the +1 padding pixel: every valid channel bit set, tail bits 0
// (padding binarizes to sign(0) = +1, reference.py:87; tail channels must be
// 0 in both operands so they never count as disagreements).
__host__ __device__ inline uint32_t pad_word(int j, int C) {
  int rem = C - 32 * j;
  return rem >= 32 ? 0xFFFFFFFFu : ((1u << rem) - 1u);
}

inline int launch_status() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? XNC_OK : XNC_ECUDA_BASE + (int)e;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Per-device launch state (xnc_runtime.cu), thread-safe.  The dynamic shared-memory
// opt-in is a per-device, per-function setting: a process-wide "done" flag would skip
// it on a second GPU and its >48 KB launches would fail.
// Raises func's opt-in on the current device to at least `bytes`; 0 or XNC_ECUDA_BASE+e.
int smem_opt_in(const void* func, size_t bytes);
template <class F>
inline int smem_opt_in(F* func, size_t bytes) { return smem_opt_in(reinterpret_cast<const void*>(func), bytes); }
// SM count of the current device (cached per device).
int device_sm_count();

// Programmatic dependent launch: a kernel started with launch_pdl may be scheduled
// while the previous kernel of its stream drains; every thread that reads what an
// earlier kernel wrote, or writes what it may still read, calls pdl_wait() first (a
// no-op for an ordinary launch).  Since each such kernel waits before it completes,
// the order holds transitively along the stream.  env XNC_PDL=0: ordinary launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
int pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

}  // namespace xnc

// Kernel launchers implemented in the per-kernel translation units.
namespace xnc {
int launch_pack_input(const float* x, int N, int C, int H, int W, uint32_t* bits, float* A,
                      cudaStream_t s, const float* in_scale = nullptr, const float* in_shift = nullptr);
int launch_pack_weights(const float* w, int O, int C, int kh, int kw, uint32_t* wbits,
                        float* alpha, double* alpha64, cudaStream_t s);
int launch_pack_weights_f64(const double* w, int O, int C, int kh, int kw, uint32_t* wbits,
                            float* alpha, double* alpha64, cudaStream_t s);
int launch_scale_map(const float* A, int N, int H, int W, int kh, int kw, int pad, float* K,
                     cudaStream_t s);
int launch_conv_popc(const uint32_t* bits, const uint32_t* wbits, const float* K,
                     const float* alpha, int N, int C, int H, int W, int O, int kh, int kw,
                     int pad, float* y, int32_t* acc, cudaStream_t s);
int launch_conv_b1mma(const uint32_t* bits, const uint32_t* wbits, const float* K,
                      const float* alpha, int N, int C, int H, int W, int O, int kh, int kw,
                      int pad, float* y, int32_t* acc, cudaStream_t s);
size_t umma_weight_bytes(int O, int C, int kh, int kw);
bool umma_supported(int N, int C, int H, int W, int O, int kh, int kw, int pad);
int launch_pack_weights_umma(const void* w, int dtype, int O, int C, int kh, int kw, uint8_t* wq,
                             int32_t* sw, cudaStream_t s);
int umma_profile_read(unsigned long long* host, int n_ctas);
int launch_conv_umma(const uint32_t* bits, const uint8_t* wq, const int32_t* sw, const float* K,
                     const float* alpha, int N, int C, int H, int W, int O, int kh, int kw, int pad,
                     float* y, int32_t* acc, cudaStream_t s, const float* out_scale = nullptr,
                     const float* out_shift = nullptr, int32_t* split_ws = nullptr,
                     uint32_t* next_bits = nullptr, float* next_A = nullptr, int y_pm = 0);
bool umma_emit_supported(int N, int C, int H, int W, int O, int kh, int kw, int pad);
size_t umma_split_ws_bytes(int N, int C, int H, int W, int O, int kh, int kw, int pad);
int launch_max_pool(const float* x, int N, int C, int Hin, int Win, int pk, int ps, int relu, const float* bias,
                    float* out, cudaStream_t s);
int launch_pad_s2d(const float* x, int N, int C, int H, int W, int p, int r, int nhwc, float* out,
                   cudaStream_t s);
int launch_max_pool_nhwc(const float* x, int N, int C, int Hin, int Win, int pk, int ps, int relu,
                         const float* bias, float* out, cudaStream_t s);
int launch_plane_affine(float* y, int N, int O, long plane, const float* scale, const float* shift,
                        cudaStream_t s);
int launch_pack_input_pool(const float* x, int N, int C, int Hin, int Win, int pk, int ps, uint32_t* bits,
                           float* A, cudaStream_t s, const float* in_scale, const float* in_shift);
int launch_pack_input_nhwc(const float* x, int N, int C, int H, int W, uint32_t* bits, float* A, cudaStream_t s,
                           const float* in_scale, const float* in_shift);
int launch_pack_input_pool_nhwc(const float* x, int N, int C, int Hin, int Win, int pk, int ps, int relu,
                                const float* bias, uint32_t* bits, float* A, cudaStream_t s, const float* in_scale,
                                const float* in_shift);
}  // namespace xnc
