// K3 variant: the legacy b1 tensor-core form, mma.sync.m16n8k256 .and.popc.
//
// The north star asks for the popcount path to be benchmarked against the b1
// mma.sync AND-popc form "wherever that form is exact".  AND-popc counts
// agreements of +1 bits only, so the XNOR sum is recovered with
//     acc = n - 2*popc(a) - 2*popc(b) + 4*popc(a & b)          (n = C*kh*kw)
// where popc(a) is the number of +1 input bits in the pixel's receptive field
// (padding words contribute C: they are all-ones over the valid channels) and
// popc(b) the number of +1 bits of the filter.  Tail channel bits are 0 in both
// operands and in the padding word, so the identity is exact for every C.
//
// On sm_100a ptxas lowers every m16n8k256 b1 MMA to a subroutine of 8x
// IMMA.16832.U8.U8 plus bit-unpacking; measured
// peak 734 bit-MAC/clk/SM (.and) vs 512 for POPC (profiles/int_peaks_r1.jsonl).
//
// Decomposition: CTA = one image, TR output rows x all W' columns (pixels taken
// in linear order, so a 16-row MMA tile may span two image rows and nothing is
// wasted on W' % 16), TO = 32 filters.  Each warp owns 2 m16 tiles x 4 n8 tiles.
// The GEMM K dimension is the flattened (ky, kx, j) word list padded to a
// multiple of 8 words (one k256 step); per-thread fragment addresses come from a
// small smem table indexed by the flattened word index.
#include "xnc_common.cuh"

namespace xnc {

constexpr int kB1TO = 32;       // filters per CTA (4 n8 tiles)
constexpr int kB1MT = 2;        // m16 tiles per warp

__device__ __forceinline__ void mma_b1_and(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                           uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__global__ void __launch_bounds__(512) k_conv_b1mma(
    const uint32_t* __restrict__ bits, const uint32_t* __restrict__ wbits,
    const float* __restrict__ Kmap, const float* __restrict__ alpha, int C, int H, int W, int O,
    int kh, int kw, int pad, int oh, int ow, int Cw, int TR, int SCs, int n_fb, int n_rt,
    int Kw8, float* __restrict__ y, int32_t* __restrict__ acc_out) {
  extern __shared__ uint4 smem_raw[];
  const int TRS = TR + kh - 1;
  const int taps = kh * kw;
  const int in_words = Cw * TRS * SCs;
  uint32_t* in_s = reinterpret_cast<uint32_t*>(smem_raw);   // [Cw][TRS][SCs] + 1 zero word
  uint32_t* w_s = in_s + in_words + 1;                        // [Cw][kh][kw][TO] + 1 zero word
  const int w_words = Cw * taps * kB1TO;
  int* kin = reinterpret_cast<int*>(w_s + w_words + 1);       // [Kw8*8] input offsets
  int* kwt = kin + Kw8 * 8;                                   // [Kw8*8] weight offsets
  int* cnt_s = kwt + Kw8 * 8;                                 // [TRS][SCs] popc per staged pixel
  int* pb_s = cnt_s + TRS * SCs;                              // [TO] popc per filter

  int bid = blockIdx.x;
  const int fb = bid % n_fb; bid /= n_fb;
  const int rt = bid % n_rt;
  const int n = bid / n_rt;
  const int y0 = rt * TR, o0 = fb * kB1TO;
  const int tid = threadIdx.x, nthr = blockDim.x;

  // ---- stage input tile (+1 padding words outside the image) and filters
  for (int i = tid; i < in_words; i += nthr) {
    const int j = i % Cw, rest = i / Cw;
    const int sc = rest % SCs, sr = rest / SCs;
    const int iy = y0 + sr - pad, ix = sc - pad;
    uint32_t v = (iy >= 0 && iy < H && ix >= 0 && ix < W)
                     ? __ldg(bits + (((long)n * H + iy) * W + ix) * Cw + j)
                     : pad_word(j, C);
    in_s[(j * TRS + sr) * SCs + sc] = v;
  }
  for (int i = tid; i < w_words; i += nthr) {
    const int t = i % kB1TO, q = i / kB1TO;
    const int o = o0 + t;
    w_s[i] = (o < O) ? __ldg(wbits + (long)q * O + o) : 0u;
  }
  if (tid == 0) { in_s[in_words] = 0u; w_s[w_words] = 0u; }
  for (int kidx = tid; kidx < Kw8 * 8; kidx += nthr) {
    if (kidx < taps * Cw) {
      const int tap = kidx / Cw, j = kidx - tap * Cw;
      const int ky = tap / kw, kx = tap - ky * kw;
      kin[kidx] = (j * TRS + ky) * SCs + kx;
      kwt[kidx] = ((j * kh + ky) * kw + kx) * kB1TO;
    } else {
      kin[kidx] = -1;
      kwt[kidx] = w_words;
    }
  }
  __syncthreads();
  // ---- popcount side terms of the AND identity
  for (int i = tid; i < TRS * SCs; i += nthr) {
    int s = 0;
    for (int j = 0; j < Cw; ++j) s += __popc(in_s[j * TRS * SCs + i]);
    cnt_s[i] = s;
  }
  for (int t = tid; t < kB1TO; t += nthr) {
    int s = 0;
    for (int q = 0; q < Cw * taps; ++q) s += __popc(w_s[q * kB1TO + t]);
    pb_s[t] = s;
  }
  __syncthreads();

  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int pix_tile = TR * ow;
  const int m_tiles = cdiv(pix_tile, 16);
  const int warps_m = cdiv(m_tiles, kB1MT);
  if (warp >= warps_m) return;  // (no __syncthreads below)
  const int mt0 = warp * kB1MT;

  // smem base offset of pixel rows g and g+8 of each m tile (linear pixel order)
  int pbase[kB1MT][2];
  bool pvalid[kB1MT][2];
#pragma unroll
  for (int m = 0; m < kB1MT; ++m)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int p = (mt0 + m) * 16 + g + 8 * h;
      pvalid[m][h] = p < pix_tile;
      const int pr = pvalid[m][h] ? p / ow : 0, pc = pvalid[m][h] ? p - (p / ow) * ow : 0;
      pbase[m][h] = pr * SCs + pc;
    }

  int d[kB1MT][4][4];
#pragma unroll
  for (int m = 0; m < kB1MT; ++m)
#pragma unroll
    for (int nn = 0; nn < 4; ++nn)
#pragma unroll
      for (int q = 0; q < 4; ++q) d[m][nn][q] = 0;

  for (int kc = 0; kc < Kw8; ++kc) {
    const int k0 = kin[kc * 8 + t], k1 = kin[kc * 8 + 4 + t];
    const int w0 = kwt[kc * 8 + t], w1 = kwt[kc * 8 + 4 + t];
    uint32_t a[kB1MT][4];
#pragma unroll
    for (int m = 0; m < kB1MT; ++m) {
      a[m][0] = k0 >= 0 ? in_s[k0 + pbase[m][0]] : 0u;
      a[m][1] = k0 >= 0 ? in_s[k0 + pbase[m][1]] : 0u;
      a[m][2] = k1 >= 0 ? in_s[k1 + pbase[m][0]] : 0u;
      a[m][3] = k1 >= 0 ? in_s[k1 + pbase[m][1]] : 0u;
    }
#pragma unroll
    for (int nn = 0; nn < 4; ++nn) {
      const uint32_t b0 = w_s[w0 + nn * 8 + g], b1 = w_s[w1 + nn * 8 + g];
#pragma unroll
      for (int m = 0; m < kB1MT; ++m) mma_b1_and(d[m][nn], a[m][0], a[m][1], a[m][2], a[m][3], b0, b1);
    }
  }

  // ---- epilogue: AND identity -> XNOR sum, then (f32(acc) * K) * alpha
  const int CK = C * kh * kw;
#pragma unroll
  for (int m = 0; m < kB1MT; ++m)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (!pvalid[m][h]) continue;
      const int p = (mt0 + m) * 16 + g + 8 * h;
      const int pr = p / ow, pc = p - pr * ow;
      const int yy = y0 + pr;
      if (yy >= oh) continue;
      int sa = 0;
      for (int ky = 0; ky < kh; ++ky)
        for (int kx = 0; kx < kw; ++kx) sa += cnt_s[(pr + ky) * SCs + pc + kx];
      const float kv = y ? __ldg(Kmap + ((long)n * oh + yy) * ow + pc) : 0.0f;
#pragma unroll
      for (int nn = 0; nn < 4; ++nn)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int ol = nn * 8 + 2 * t + q;
          const int o = o0 + ol;
          if (o >= O) continue;
          const int v = CK - 2 * sa - 2 * pb_s[ol] + 4 * d[m][nn][2 * h + q];
          const long idx = (((long)n * O + o) * oh + yy) * ow + pc;
          if (y) y[idx] = __fmul_rn(__fmul_rn((float)v, kv), __ldg(alpha + o));
          if (acc_out) acc_out[idx] = v;
        }
    }
}

int launch_conv_b1mma(const uint32_t* bits, const uint32_t* wbits, const float* K,
                      const float* alpha, int N, int C, int H, int W, int O, int kh, int kw,
                      int pad, float* y, int32_t* acc, cudaStream_t s) {
  const int oh = H + 2 * pad - kh + 1, ow = W + 2 * pad - kw + 1;
  const int Cw = cdiv(C, 32);
  const int taps = kh * kw;
  const int Kw8 = cdiv(taps * Cw, 8);
  // ~256-512 pixels per CTA (16-32 m16 tiles -> 8-16 warps)
  int TR = max(1, min(oh, 512 / ow));
  const int SCs = ow + kw - 1;
  auto smem_for = [&](int tr) {
    const int trs = tr + kh - 1;
    return (size_t)(Cw * trs * SCs + 1 + Cw * taps * kB1TO + 1 + 2 * Kw8 * 8 + trs * SCs + kB1TO) * 4;
  };
  while (TR > 1 && (smem_for(TR) > 160 * 1024 || cdiv(cdiv(TR * ow, 16), kB1MT) * 32 > 512)) --TR;
  const size_t smem = smem_for(TR);
  const int threads = cdiv(cdiv(TR * ow, 16), kB1MT) * 32;
  if (smem > 200 * 1024 || threads > 512) return XNC_ENOTSUP;
  const int n_fb = cdiv(O, kB1TO), n_rt = cdiv(oh, TR);
  const long blocks = (long)n_fb * n_rt * N;
  if (int rc = smem_opt_in(k_conv_b1mma, smem)) return rc;  // per device (xnc_runtime.cu)
  k_conv_b1mma<<<(unsigned)blocks, threads, smem, s>>>(bits, wbits, K, alpha, C, H, W, O, kh, kw, pad,
                                                       oh, ow, Cw, TR, SCs, n_fb, n_rt, Kw8, y, acc);
  return launch_status();
}

}  // namespace xnc
