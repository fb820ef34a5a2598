// K3 on the 5th-generation tensor cores: tcgen05.mma.kind::i8, accumulators in TMEM.
//
// Exact-integer reformulation of the XNOR sum.  With d = 1 for a negative input
// sign (d = 0 for +1, for padding and -- through zero weights -- for tail
// channels) and s_w = +-1 the filter sign (0 for tail channels):
//     sum_taps s_x * s_w = sum_taps (1 - 2d) * s_w = S_w[o] - 2 * sum_taps d * s_w
// where S_w[o] = sum of the filter's signs.  sum d*s_w is a u8 x s8 GEMM with an
// s32 accumulator: M = output pixels, N = filters, K = kh*kw*C (one byte per
// sign), so the result is bit-identical to the reference decode
// `k_area - 2*popc(diff)` summed over channels (_kernels_cy.pyx:100-104), and
// the alpha*K epilogue (_kernels_cy.pyx:349) is applied from TMEM.
// Zero-filled taps are d = 0 = the +1 padding of zero_pad-then-binarize
// (reference.py:87) -- no special case.
//
// Implicit GEMM without an im2col buffer.  Per image the output is walked on an
// "extended" grid of H' rows x IC = W' + kw - 1 columns (the padded input row
// length; the last kw-1 columns of every row are discarded).  Then output pixel
// e and tap (ky, kx) read padded input pixel e + ky*IC + kx, i.e. every tap of a
// 128-row MMA tile is the SAME smem tile shifted by a whole number of 128-byte
// rows: one K-major SWIZZLE_128B descriptor per tap, no data movement
// (tools/microbench/umma_probe.cu verified row-shifted descriptors with
// base_offset = 0 against a CPU GEMM on a B200: 0 mismatches for shifts 0-9).
//
// CTA = one image, 256 extended output pixels (two M=128 MMA tiles sharing
// each B tile), NB <= 256 filters.  Shared memory:
//   A: the padded input rows the 256 pixels touch, as u8 d-values, one
//      1024-aligned plane per 128-channel K block (expanded in smem from the
//      packed sign bits of K1 -- 1 bit/element from L2, 8x less than bytes);
//   B: S stages of one (tap, K block) weight chunk, NB x 128 B, streamed with
//      cp.async.bulk (the chunks are pre-swizzled in HBM by k_pack_weights_umma);
// TMEM: 2 x NB s32 columns.  Warp roles: warp 0 = B producer, warp 1 = MMA
// issuer (one thread), warps 4-7 = epilogue (TMEM lane quadrants 0-3); every
// warp helps expand A in the prologue.
#include "xnc_common.cuh"

namespace xnc {

constexpr int kUmmaThreads = 256;
constexpr int kUmmaMT = 256;     // extended output pixels per CTA (2 x M=128)
constexpr int kUmmaStages = 3;   // B pipeline depth

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// K-major, SWIZZLE_128B UMMA shared-memory descriptor (sm_100 version 1).
// Rows are 128 B apart, 8-row groups 1024 B apart (SBO); the swizzle is a
// function of the absolute smem address, so row-shifted starts need no base offset.
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
        : "r"(smem_addr(bar)), "r"(parity));
  }
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
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
      smem_addr(bar)));
}

__device__ __forceinline__ void tmem_ld32(uint32_t addr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
        "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
        "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
        "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// 16 sign bits -> 16 bytes of d = NOT(bit) in {0, 1} (byte i from bit i).
__device__ __forceinline__ uint4 expand_d16(uint32_t bits16) {
  const uint32_t d = ~bits16;
  uint4 r;
  r.x = ((d & 0xFu) * 0x00204081u) & 0x01010101u;
  r.y = (((d >> 4) & 0xFu) * 0x00204081u) & 0x01010101u;
  r.z = (((d >> 8) & 0xFu) * 0x00204081u) & 0x01010101u;
  r.w = (((d >> 12) & 0xFu) * 0x00204081u) & 0x01010101u;
  return r;
}

struct UmmaGeom {
  int C, H, W, O, kh, kw, pad, oh, ow, IC, Cw, KBn, NB, R, plane_bytes, n_mt, n_nb;
};

__global__ void __launch_bounds__(kUmmaThreads, 1) k_conv_umma(
    const uint32_t* __restrict__ bits, const uint8_t* __restrict__ wq, const int32_t* __restrict__ sw,
    const float* __restrict__ Kmap, const float* __restrict__ alpha, UmmaGeom g,
    float* __restrict__ y, int32_t* __restrict__ acc_out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  uint8_t* a_s = smem;                                          // KBn planes
  uint8_t* b_s = a_s + (size_t)g.KBn * g.plane_bytes;           // stages x NB*128
  const uint32_t b_stage_bytes = (uint32_t)g.NB * 128u;
  __shared__ __align__(8) uint64_t full_bar[kUmmaStages], empty_bar[kUmmaStages], done_bar;
  __shared__ uint32_t tmem_base_s;

  int bid = blockIdx.x;
  const int nb = bid % g.n_nb; bid /= g.n_nb;
  const int mt = bid % g.n_mt;
  const int n = bid / g.n_mt;
  const int m0 = mt * kUmmaMT;
  const int r0 = m0 / g.IC;
  const int off0 = m0 - r0 * g.IC;
  const int taps = g.kh * g.kw;
  const int nsteps = taps * g.KBn;
  const uint32_t tmem_cols = (2 * g.NB <= 32) ? 32 : (2 * g.NB <= 64) ? 64 : (2 * g.NB <= 128) ? 128
                            : (2 * g.NB <= 256) ? 256 : 512;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    for (int s = 0; s < kUmmaStages; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], 1); }
    mbar_init(&done_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_addr(&tmem_base_s)), "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_s;

  // ---- B producer: prefetch the first stages while everyone expands A
  const uint8_t* wq_nb = wq + (size_t)nb * nsteps * b_stage_bytes;
  if (tid == 0) {
    for (int st = 0; st < kUmmaStages && st < nsteps; ++st)
      bulk_load(b_s + st * b_stage_bytes, wq_nb + (size_t)st * b_stage_bytes, b_stage_bytes, &full_bar[st]);
  }

  // ---- A: expand packed sign bits of the padded input rows into u8 d-planes
  {
    const int pix = g.R * g.IC;
    const int items = pix * g.KBn * 8;  // 16-byte chunks
    const uint32_t* img = bits + (size_t)n * g.H * g.W * g.Cw;
    for (int it = tid; it < items; it += kUmmaThreads) {
      const int q = it & 7;
      const int rest = it >> 3;
      const int kb = rest % g.KBn;
      const int i = rest / g.KBn;
      const int pr = r0 + i / g.IC, pc = i % g.IC;
      const int iy = pr - g.pad, ix = pc - g.pad;
      uint4 v = make_uint4(0u, 0u, 0u, 0u);
      if (iy >= 0 && iy < g.H && ix >= 0 && ix < g.W) {
        const int wi = kb * 4 + (q >> 1);
        const uint32_t word = wi < g.Cw ? __ldg(img + ((size_t)iy * g.W + ix) * g.Cw + wi) : 0xFFFFFFFFu;
        v = expand_d16((word >> ((q & 1) * 16)) & 0xFFFFu);
      }
      *reinterpret_cast<uint4*>(a_s + (size_t)kb * g.plane_bytes + (size_t)i * 128 + ((q ^ (i & 7)) << 4)) = v;
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core
  __syncthreads();

  if (warp == 0) {
    // ---- B producer: steady state
    if (lane == 0) {
      for (int step = kUmmaStages; step < nsteps; ++step) {
        const int st = step % kUmmaStages;
        mbar_wait(&empty_bar[st], ((step / kUmmaStages) - 1) & 1);
        bulk_load(b_s + st * b_stage_bytes, wq_nb + (size_t)step * b_stage_bytes, b_stage_bytes,
                  &full_bar[st]);
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer
    if (lane == 0) {
      const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(g.NB >> 3) << 17) |
                             ((uint32_t)(128 >> 4) << 24);
      const uint32_t a_base = smem_addr(a_s), b_base = smem_addr(b_s);
      for (int step = 0; step < nsteps; ++step) {
        const int st = step % kUmmaStages;
        const int tap = step / g.KBn, kb = step - tap * g.KBn;
        const int ky = tap / g.kw, kx = tap - ky * g.kw;
        mbar_wait(&full_bar[st], (step / kUmmaStages) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t a_tap = a_base + (uint32_t)kb * g.plane_bytes +
                               (uint32_t)(off0 + ky * g.IC + kx) * 128u;
        const uint32_t b_st = b_base + (uint32_t)st * b_stage_bytes;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const uint64_t bd = umma_desc_sw128(b_st + s * 32);
#pragma unroll
          for (int h = 0; h < 2; ++h)
            umma_i8(tmem + h * g.NB, umma_desc_sw128(a_tap + h * 128 * 128 + s * 32), bd, idesc,
                    (step | s) != 0);
        }
        umma_commit(&empty_bar[st]);  // frees the B stage when these MMAs retire
      }
      umma_commit(&done_bar);
    }
  } else if (warp >= 4) {
    // ---- epilogue: TMEM -> registers -> decode + alpha*K -> y
    const int quad = warp & 3;
    mbar_wait(&done_bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int CKtot = g.C * taps;
    (void)CKtot;
    for (int h = 0; h < 2; ++h) {
      const int e = m0 + h * 128 + quad * 32 + lane;
      const int r = e / g.IC, c = e - (e / g.IC) * g.IC;
      const bool valid = (r < g.oh) && (c < g.ow);
      const float kv = (valid && y) ? __ldg(Kmap + ((size_t)n * g.oh + r) * g.ow + c) : 0.0f;
      for (int c0 = 0; c0 < g.NB; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(h * g.NB + c0), v);
        if (!valid) continue;
#pragma unroll 4
        for (int j = 0; j < 32; ++j) {
          const int o = nb * g.NB + c0 + j;
          if (o >= g.O) break;
          const int accv = __ldg(sw + o) - 2 * (int)v[j];
          const size_t idx = (((size_t)n * g.O + o) * g.oh + r) * g.ow + c;
          if (y) __stcs(y + idx, __fmul_rn(__fmul_rn((float)accv, kv), __ldg(alpha + o)));
          if (acc_out) acc_out[idx] = accv;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    __syncwarp();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols));
  }
}

// ---------------------------------------------------------------- weights
// wq[nb][tap][kb][row = filter within block][128 B], s8 signs (+1/-1, 0 for tail
// channels and filters >= O), each (tap, kb) chunk pre-swizzled for a 1024-aligned
// smem destination (16-byte chunk q of row r stored at q ^ (r & 7)).
// sw[o] = sum of the filter's signs over all taps and valid channels.
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

static int umma_nb(int O) { return O >= 256 ? 256 : (O <= 16 ? 16 : round_up(O, 16)); }

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

static bool umma_plan(int N, int C, int H, int W, int O, int kh, int kw, int pad, UmmaGeom& g,
                      size_t& smem) {
  g.C = C; g.H = H; g.W = W; g.O = O; g.kh = kh; g.kw = kw; g.pad = pad;
  g.oh = H + 2 * pad - kh + 1; g.ow = W + 2 * pad - kw + 1;
  g.IC = g.ow + kw - 1;  // = W + 2*pad
  g.Cw = cdiv(C, 32);
  g.KBn = cdiv(C, 128);
  g.NB = umma_nb(O);
  // rows of padded input a CTA touches: pixel indices off0 .. off0+255 + (kh-1)*IC + kw-1
  g.R = (g.IC - 1 + kUmmaMT - 1 + kw - 1) / g.IC + kh;
  g.plane_bytes = round_up(g.R * g.IC * 128, 1024);
  g.n_mt = cdiv(g.oh * g.IC, kUmmaMT);
  g.n_nb = cdiv(O, g.NB);
  smem = (size_t)g.KBn * g.plane_bytes + (size_t)kUmmaStages * g.NB * 128 + 1024;
  return smem <= 226 * 1024 && (long)N * g.n_mt * g.n_nb < 0x7fffffffL;
}

bool umma_supported(int N, int C, int H, int W, int O, int kh, int kw, int pad) {
  UmmaGeom g;
  size_t smem;
  return umma_plan(N, C, H, W, O, kh, kw, pad, g, smem);
}

int launch_conv_umma(const uint32_t* bits, const uint8_t* wq, const int32_t* sw, const float* K,
                     const float* alpha, int N, int C, int H, int W, int O, int kh, int kw, int pad,
                     float* y, int32_t* acc, cudaStream_t s) {
  UmmaGeom g;
  size_t smem;
  if (!umma_plan(N, C, H, W, O, kh, kw, pad, g, smem)) return XNC_ENOTSUP;
  static size_t attr_smem = 0;  // one-time (per size increase) shared-memory opt-in
  if (smem > attr_smem) {
    cudaError_t e = cudaFuncSetAttribute(k_conv_umma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return XNC_ECUDA_BASE + (int)e;
    attr_smem = smem;
  }
  const long blocks = (long)N * g.n_mt * g.n_nb;
  k_conv_umma<<<(unsigned)blocks, kUmmaThreads, smem, s>>>(bits, wq, sw, K, alpha, g, y, acc);
  return launch_status();
}

}  // namespace xnc
