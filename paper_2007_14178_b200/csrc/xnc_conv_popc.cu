// K3+K4: XNOR-popcount implicit-GEMM convolution with the alpha*K epilogue.
//
// GEMM view: M = N*H'*W' output pixels,
// N_gemm = O filters, K_gemm = kh*kw*Cw 32-bit words.  For every pixel p and
// filter o:  acc = C*kh*kw - 2 * sum_{ky,kx,j} popc(in[p+(ky,kx)][j] ^ w[o][ky][kx][j])
// which is the reference decode `k_area - 2*popc(diff)` summed over channels
// (_kernels_cy.pyx:100-104) regrouped 32 channels per word.  Tail channel bits
// are 0 in both operands; out-of-image taps read the +1 padding word
// (pad_word), exactly as zero_pad-then-binarize does (reference.py:87).
// Epilogue: y = (f32(acc) * K[n][y][x]) * alpha[o]  (_kernels_cy.pyx:349,
// two round-to-nearest multiplies, no FMA) -- bit-identical to the reference.
//
// Work decomposition (POPC-pipe bound: 16 lanes/clk/SM measured, see
// profiles/int_peaks_r1.json):
//  * CTA = one image n, TR output rows x TCg*P output columns, TO filters.
//  * The packed input tile (TR+kh-1 rows x (TCg*P+kw-1) cols x JC words) and
//    the filter block (JC x kh x kw x TO words) are staged in shared memory.
//  * Thread = P consecutive output columns x F filters held in P*F int32
//    registers.  Lanes of a warp walk consecutive column groups (conflict-free
//    16-byte smem reads of the input window) and share a filter group (the
//    filter words are warp-broadcast reads).
//  * For each (word j, kernel row ky) a thread loads its P+kw-1 input words
//    once and reuses them across the kw taps (register sliding window), so the
//    inner loop is LOP3 + POPC + IADD per word pair with ~3% load overhead.
#include "xnc_common.cuh"

namespace xnc {

constexpr int kP = 4;   // output columns per thread
constexpr int kF = 8;   // filters per thread

template <int KW>
__global__ void __launch_bounds__(256) k_conv_popc(
    const uint32_t* __restrict__ bits, const uint32_t* __restrict__ wbits,
    const float* __restrict__ Kmap, const float* __restrict__ alpha, int C, int H, int W, int O,
    int kh, int pad, int oh, int ow, int Cw, int JC, int TR, int TCg, int TO, int SCs,
    int n_fb, int n_ct, int n_rt, int vec_ok, float* __restrict__ y,
    int32_t* __restrict__ acc_out) {
  constexpr int P = kP, F = kF;
  constexpr int NWIN = ((P + KW - 1) + 3) / 4 * 4;
  extern __shared__ uint4 smem_raw[];
  const int TRS = TR + kh - 1;
  uint32_t* in_s = reinterpret_cast<uint32_t*>(smem_raw);  // [JC][TRS][SCs]
  uint32_t* w_s = in_s + (long)JC * TRS * SCs;              // [JC][kh][KW][TO]

  int bid = blockIdx.x;
  const int fb = bid % n_fb; bid /= n_fb;
  const int ct = bid % n_ct; bid /= n_ct;
  const int rt = bid % n_rt;
  const int n = bid / n_rt;
  const int y0 = rt * TR, x0 = ct * TCg * P, o0 = fb * TO;

  const int slots = TR * TCg;
  const int tid = threadIdx.x;
  const int slot = tid % slots, fg = tid / slots;
  const int r = slot / TCg, g = slot % TCg;

  int acc[P][F];
#pragma unroll
  for (int p = 0; p < P; ++p)
#pragma unroll
    for (int f = 0; f < F; ++f) acc[p][f] = 0;

  const int kkw = kh * KW;
  for (int j0 = 0; j0 < Cw; j0 += JC) {
    const int jn = min(JC, Cw - j0);
    if (j0 > 0) __syncthreads();
    // ---- stage the packed input tile (j fastest: coalesced global reads)
    const int in_elems = jn * TRS * SCs;
    for (int i = tid; i < in_elems; i += blockDim.x) {
      const int jj = i % jn;
      const int rest = i / jn;
      const int sc = rest % SCs, sr = rest / SCs;
      const int iy = y0 + sr - pad, ix = x0 + sc - pad;
      const int j = j0 + jj;
      uint32_t v;
      if (iy >= 0 && iy < H && ix >= 0 && ix < W)
        v = __ldg(bits + (((long)n * H + iy) * W + ix) * Cw + j);
      else
        v = pad_word(j, C);
      in_s[(jj * TRS + sr) * SCs + sc] = v;
    }
    // ---- stage the filter block (filters contiguous)
    const int w_elems = jn * kkw * TO;
    for (int i = tid; i < w_elems; i += blockDim.x) {
      const int t = i % TO;
      const int q = i / TO;  // (jj*kh + ky)*KW + kx
      const int o = o0 + t;
      w_s[i] = (o < O) ? __ldg(wbits + ((long)j0 * kkw + q) * O + o) : 0u;
    }
    __syncthreads();

    for (int jj = 0; jj < jn; ++jj) {
      for (int ky = 0; ky < kh; ++ky) {
        const uint32_t* rp = in_s + (jj * TRS + r + ky) * SCs + g * P;
        uint32_t win[NWIN];
#pragma unroll
        for (int q = 0; q < NWIN / 4; ++q) {
          uint4 t = reinterpret_cast<const uint4*>(rp)[q];
          win[4 * q + 0] = t.x; win[4 * q + 1] = t.y; win[4 * q + 2] = t.z; win[4 * q + 3] = t.w;
        }
        const uint32_t* wp = w_s + (jj * kh + ky) * KW * TO + fg * F;
#pragma unroll
        for (int kx = 0; kx < KW; ++kx) {
          uint32_t wv[F];
#pragma unroll
          for (int q = 0; q < F / 4; ++q) {
            uint4 t = reinterpret_cast<const uint4*>(wp + kx * TO)[q];
            wv[4 * q + 0] = t.x; wv[4 * q + 1] = t.y; wv[4 * q + 2] = t.z; wv[4 * q + 3] = t.w;
          }
#pragma unroll
          for (int p = 0; p < P; ++p)
#pragma unroll
            for (int f = 0; f < F; ++f) acc[p][f] += __popc(win[p + kx] ^ wv[f]);
        }
      }
    }
  }

  // ---- epilogue: decode + alpha*K (K4), fused
  const int yy = y0 + r;
  const int xb = x0 + g * P;
  if (yy >= oh || xb >= ow) return;
  const int CK = C * kh * KW;
  float kv[P];
  const float* kp = Kmap + ((long)n * oh + yy) * ow + xb;
#pragma unroll
  for (int p = 0; p < P; ++p) kv[p] = (y != nullptr && xb + p < ow) ? __ldg(kp + p) : 0.0f;
  const bool vec = vec_ok != 0;  // ow % 4 == 0 and 16-byte aligned outputs
#pragma unroll
  for (int f = 0; f < F; ++f) {
    const int o = o0 + fg * F + f;
    if (o >= O) break;
    const long base = (((long)n * O + o) * oh + yy) * ow + xb;
    int v[P];
#pragma unroll
    for (int p = 0; p < P; ++p) v[p] = CK - 2 * acc[p][f];
    if (y != nullptr) {
      const float a = __ldg(alpha + o);
      float out[P];
#pragma unroll
      for (int p = 0; p < P; ++p) out[p] = __fmul_rn(__fmul_rn((float)v[p], kv[p]), a);
      if (vec) {
        __stcs(reinterpret_cast<float4*>(y + base), make_float4(out[0], out[1], out[2], out[3]));
      } else {
#pragma unroll
        for (int p = 0; p < P; ++p)
          if (xb + p < ow) y[base + p] = out[p];
      }
    }
    if (acc_out != nullptr) {
      if (vec) {
        *reinterpret_cast<int4*>(acc_out + base) = make_int4(v[0], v[1], v[2], v[3]);
      } else {
#pragma unroll
        for (int p = 0; p < P; ++p)
          if (xb + p < ow) acc_out[base + p] = v[p];
      }
    }
  }
}

template <int KW>
static int launch_kw(const uint32_t* bits, const uint32_t* wbits, const float* K,
                     const float* alpha, int N, int C, int H, int W, int O, int kh, int pad,
                     float* y, int32_t* acc, cudaStream_t s) {
  constexpr int P = kP, F = kF;
  const int oh = H + 2 * pad - kh + 1, ow = W + 2 * pad - KW + 1;
  const int Cw = cdiv(C, 32);
  int TO = 32;
  while (TO > F && TO / 2 >= O) TO /= 2;  // small O: narrower filter blocks
  const int FG = TO / F;
  const int Gc = cdiv(ow, P);
  int TCg = Gc;
  while (TCg * FG > 256) TCg = cdiv(TCg, 2);
  int TR = max(1, min(oh, 256 / (TCg * FG)));
  const int NWIN = ((P + KW - 1) + 3) / 4 * 4;
  const int SCs = round_up((TCg - 1) * P + NWIN, 4);
  // words of the K dimension staged per pass: keep smem <= 96 KB so >= 2 CTAs fit
  auto smem_for = [&](int jc, int tr) {
    return (size_t)jc * ((size_t)(tr + kh - 1) * SCs + (size_t)kh * KW * TO) * 4;
  };
  int JC = Cw;
  while (JC > 1 && smem_for(JC, TR) > 96 * 1024) JC = cdiv(JC, 2);
  while (TR > 1 && smem_for(JC, TR) > 96 * 1024) --TR;
  const size_t smem = smem_for(JC, TR);
  if (smem > 200 * 1024) return XNC_ENOTSUP;
  const int n_fb = cdiv(O, TO), n_ct = cdiv(Gc, TCg), n_rt = cdiv(oh, TR);
  const long blocks = (long)n_fb * n_ct * n_rt * N;
  if (blocks > 0x7fffffffL) return XNC_ENOTSUP;
  const int threads = TR * TCg * FG;
  const int vec_ok = (ow % 4 == 0) && ((reinterpret_cast<uintptr_t>(y) & 15) == 0) &&
                     ((reinterpret_cast<uintptr_t>(acc) & 15) == 0);
  if (int rc = smem_opt_in(k_conv_popc<KW>, smem)) return rc;  // per device (xnc_runtime.cu)
  k_conv_popc<KW><<<(unsigned)blocks, threads, smem, s>>>(
      bits, wbits, K, alpha, C, H, W, O, kh, pad, oh, ow, Cw, JC, TR, TCg, TO, SCs, n_fb, n_ct,
      n_rt, vec_ok, y, acc);
  return launch_status();
}

int launch_conv_popc(const uint32_t* bits, const uint32_t* wbits, const float* K,
                     const float* alpha, int N, int C, int H, int W, int O, int kh, int kw,
                     int pad, float* y, int32_t* acc, cudaStream_t s) {
  switch (kw) {
    case 1: return launch_kw<1>(bits, wbits, K, alpha, N, C, H, W, O, kh, pad, y, acc, s);
    case 2: return launch_kw<2>(bits, wbits, K, alpha, N, C, H, W, O, kh, pad, y, acc, s);
    case 3: return launch_kw<3>(bits, wbits, K, alpha, N, C, H, W, O, kh, pad, y, acc, s);
    case 4: return launch_kw<4>(bits, wbits, K, alpha, N, C, H, W, O, kh, pad, y, acc, s);
    case 5: return launch_kw<5>(bits, wbits, K, alpha, N, C, H, W, O, kh, pad, y, acc, s);
    case 6: return launch_kw<6>(bits, wbits, K, alpha, N, C, H, W, O, kh, pad, y, acc, s);
    case 7: return launch_kw<7>(bits, wbits, K, alpha, N, C, H, W, O, kh, pad, y, acc, s);
    case 8: return launch_kw<8>(bits, wbits, K, alpha, N, C, H, W, O, kh, pad, y, acc, s);
    default: return XNC_EINVAL;
  }
}

}  // namespace xnc
