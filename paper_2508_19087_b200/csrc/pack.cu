// pack.cu — INT -> bipolar-INT bit-plane packing on the device (§4.1 Steps 1-3), and the
// fused fp16 -> symmetric per-token quantize + pack.
//
// Work item = one "quad" = 128 consecutive K elements of one row (4 output words per plane, one
// 16-byte store per plane).  A CTA owns R whole rows (so the row sums reduce in shared memory
// without global atomics) and its 256 threads stride over the R x Kpad/128 quads: rows fastest for
// the tile-major weight layout (a warp stores 32 rows x 16 B = 512 contiguous bytes per plane),
// quads fastest for the canonical layout (a warp stores 512 contiguous bytes of one row).  Each
// item reads its 128 codes as 8 x 16-byte loads, then per 32-element word:
//   signed -> offset digit  u = x + 2^(n-1) mod 2^n (the sign-bit flip of P:202), bytewise, no
//                           cross-byte carries;
//   natural -> slot order   two 4 x 4 byte transposes (16 PRMT, common.cuh to_slot_order): the
//                           digit view (activations) is exactly these registers;
//   slot order -> planes    unbuild8<BITS>, the inverse of the GEMMs' operand rebuild: a 2-3 stage
//                           butterfly bit transpose giving all BITS plane words at once (element c
//                           -> bit c, LSB first, reading Q5);
// row sums of the signed codes with dp4a.  ~60 integer ops per 32 elements at BITS <= 4 (~100 at
// BITS = 8) against ~40 per plane for a per-plane bit gather.
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "sync.cuh"

namespace apt {

constexpr int kPackThreads = 256;
constexpr int kPackWordThreads = 1024;  // one-word-per-thread activation packs: every item in one round
constexpr int kPackMaxRows = 256;  // rows per CTA (shared row-sum / row-max slots)
#ifndef APT_PACK_TILED_ROWS
#define APT_PACK_TILED_ROWS 16  // rows per CTA of a tile-major (weight) pack: one or a few quads per thread
#endif
#ifndef APT_PACK_WORD_ROWS
// activation packs up to this many rows take one word per thread (every activation pack: at M = 2048 the
// word path is 1.3-1.5x faster than quads, profiles/r2_pack_ab.jsonl)
#define APT_PACK_WORD_ROWS (1 << 30)
#endif

// bytewise: signed codes (4 per word) -> offset digits u (4 per word), modulo 2^BITS
template <int BITS>
__device__ __forceinline__ uint32_t to_offset4(uint32_t v) {
  if constexpr (BITS == 8) {
    return v ^ 0x80808080u;
  } else {
    constexpr uint32_t h = 1u << (BITS - 1);
    constexpr uint32_t mask = (1u << BITS) - 1u;
    // (x & 0x7F) + h < 256 never carries into the next byte; mod 2^BITS it equals x + h since 2^BITS | 128
    return ((v & 0x7F7F7F7Fu) + h * 0x01010101u) & (mask * 0x01010101u);
  }
}

// bytewise: offset digits -> sign-extended signed codes (used to detect out-of-range inputs)
template <int BITS>
__device__ __forceinline__ uint32_t from_offset4(uint32_t u) {
  if constexpr (BITS == 8) {
    return u ^ 0x80808080u;
  } else {
    constexpr uint32_t h = 1u << (BITS - 1);
    const uint32_t x = u ^ (h * 0x01010101u);                   // n-bit two's complement pattern
    const uint32_t s = (x >> (BITS - 1)) & 0x01010101u;         // sign bit of every byte
    return x | (s * (0x100u - 2u * h));                          // sign-extend (no cross-byte carry)
  }
}

// Stream order with programmatic dependent launch (include/apt.h "General contract"): the GEMMs
// read weight-side operands (planes, row sums, scales) BEFORE griddepcontrol.wait, so a kernel that
// writes a weight operand must not release its dependents early.  A pack with a digit view is an
// activation operand (apt_gemm rejects it as W, and reads activations only after the wait): it
// releases its dependents at entry, which hides the next launch.  Without a digit view the pack
// never triggers early (dependents launch once every CTA has exited) and fences its stores at GPU
// scope before exiting.
__device__ __forceinline__ void pack_release() { __threadfence(); }

// the 32 * WPI signed codes of one work item (WPI consecutive 32-element words) as 8 * WPI natural-order
// words (4 codes each)
template <bool QUANT, int WPI>
__device__ __forceinline__ void load_words(const PackArgs& p, const void* rowp, int c0, float s, int qmax,
                                           uint32_t (&v)[8 * WPI]) {
  constexpr int kE = 32 * WPI;  // codes per item
  if constexpr (!QUANT) {
    const int8_t* row = reinterpret_cast<const int8_t*>(rowp);
    if (((reinterpret_cast<uintptr_t>(row) & 15u) == 0) && c0 + kE <= p.k) {
#pragma unroll
      for (int j = 0; j < 2 * WPI; ++j) {
        const uint4 t = __ldg(reinterpret_cast<const uint4*>(row + c0) + j);
        v[4 * j] = t.x; v[4 * j + 1] = t.y; v[4 * j + 2] = t.z; v[4 * j + 3] = t.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8 * WPI; ++j) {
        uint32_t word = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int c = c0 + 4 * j + b;
          uint32_t byte = 0;  // pad = signed code 0 (reading Q6)
          if (c < p.k) {
            byte = (uint32_t)(uint8_t)row[c];
          } else if (p.enc == 1) {
            byte = 1u;  // bipolar pad x' = 1 -> signed 0
          }
          word |= byte << (8 * b);
        }
        v[j] = word;
      }
    }
  } else {
    // fp16 -> codes: x_hat = clamp(rint(RN_f32(x / s)), -qmax - 1, qmax), 0 where s == 0 (reading R-Q)
    const __half* row = reinterpret_cast<const __half*>(rowp);
    const bool vec = ((reinterpret_cast<uintptr_t>(row) & 15u) == 0) && c0 + kE <= p.k;
#pragma unroll
    for (int j = 0; j < 4 * WPI; ++j) {
      float f[8];
      if (vec) {
        const uint4 t = __ldg(reinterpret_cast<const uint4*>(row + c0) + j);
        const __half2* h = reinterpret_cast<const __half2*>(&t);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 g = __half22float2(h[e]);
          f[2 * e] = g.x;
          f[2 * e + 1] = g.y;
        }
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) f[e] = (c0 + 8 * j + e < p.k) ? __half2float(row[c0 + 8 * j + e]) : 0.f;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t word = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          float q = s > 0.f ? rintf(__fdiv_rn(f[4 * h + b], s)) : 0.f;
          q = fminf(fmaxf(q, -(float)qmax - 1.f), (float)qmax);
          word |= ((uint32_t)(int)q & 0xFFu) << (8 * b);
        }
        v[2 * j + h] = word;
      }
    }
  }
}

// WPI = words per work item: 4 (a 128-element quad, one 16-byte store per plane: the weight packs,
// bandwidth) or 1 (one 32-element word: the activation packs, a short per-thread critical path)
// The rows [cta * R, cta * R + R) of one pack (the body of pack_kernel and of pack_grouped_kernel).
template <int BITS, bool QUANT, int WPI>
__device__ __forceinline__ void pack_body(const PackArgs& p, const __half* __restrict__ x, float* scale,
                                          int rows_per_cta, int cta, int* s_sum, unsigned* s_amax) {
  const int R = rows_per_cta;
  const int r0 = cta * R;
  const int Q = p.k_words / WPI;  // work items per row
  const int items = R * Q;
  constexpr int kQmax = (1 << (BITS - 1)) - 1;
  for (int i = threadIdx.x; i < R; i += blockDim.x) {
    s_sum[i] = 0;
    s_amax[i] = 0u;
  }
  __syncthreads();
  auto item_rq = [&](int idx, int& rl, int& q) {
    if (p.tiled) { rl = idx % R; q = idx / R; } else { rl = idx / Q; q = idx % Q; }
  };
  if constexpr (QUANT) {
    // pass 1: row maxima of |x| (non-negative floats order like their bit patterns)
    for (int idx = threadIdx.x; idx < items; idx += blockDim.x) {
      int rl, q;
      item_rq(idx, rl, q);
      const int r = r0 + rl;
      if (r >= p.rows) continue;
      const __half* row = x + (int64_t)r * p.ld;
      float m = 0.f;
      const int c0 = 32 * WPI * q;
      if (((reinterpret_cast<uintptr_t>(row) & 15u) == 0) && c0 + 32 * WPI <= p.k) {
#pragma unroll
        for (int j = 0; j < 4 * WPI; ++j) {
          const uint4 t = __ldg(reinterpret_cast<const uint4*>(row + c0) + j);
          const __half2* h = reinterpret_cast<const __half2*>(&t);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 g = __half22float2(h[e]);
            m = fmaxf(m, fmaxf(fabsf(g.x), fabsf(g.y)));
          }
        }
      } else {
        for (int c = c0; c < c0 + 32 * WPI && c < p.k; ++c) m = fmaxf(m, fabsf(__half2float(row[c])));
      }
      atomicMax(&s_amax[rl], __float_as_uint(m));
    }
    __syncthreads();
  }
  for (int idx = threadIdx.x; idx < items; idx += blockDim.x) {
    int rl, q;
    item_rq(idx, rl, q);
    const int r = r0 + rl;
    if (r >= p.rows) continue;
    float s = 0.f;
    const void* rowp;
    if constexpr (QUANT) {
      s = __fdiv_rn(__uint_as_float(s_amax[rl]), (float)kQmax);
      if (q == 0) scale[r] = s;
      rowp = x + (int64_t)r * p.ld;
    } else {
      rowp = p.codes + (int64_t)r * p.ld;
    }
    uint32_t v[8 * WPI];
    load_words<QUANT, WPI>(p, rowp, 32 * WPI * q, s, kQmax, v);
    int sum = 0;
    uint32_t pw[BITS][WPI];
#pragma unroll
    for (int wi = 0; wi < WPI; ++wi) {
      const int c0 = 32 * (WPI * q + wi);
      uint32_t u[8];
      bool bad = false;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        uint32_t xw = v[8 * wi + j];
        if (!QUANT && p.enc == 1) {
          // bipolar x' (odd) -> signed x = (x' - 1) / 2 = x' >> 1 (arithmetic, bytewise)
          bad |= (xw & 0x01010101u) != 0x01010101u;
          xw = ((xw >> 1) & 0x7F7F7F7Fu) | (xw & 0x80808080u);
        }
        u[j] = to_offset4<BITS>(xw);
        if (!QUANT) bad |= from_offset4<BITS>(u[j]) != xw;
        sum = __dp4a((int)xw, 0x01010101, sum);
      }
      if (!QUANT && bad && p.range_error) {
        const int8_t* row = reinterpret_cast<const int8_t*>(rowp);
        for (int c = c0; c < c0 + 32 && c < p.k; ++c) {
          int xv = row[c];
          bool ok;
          if (p.enc == 1) {
            ok = (xv & 1) && xv >= -((1 << BITS) - 1) && xv <= (1 << BITS) - 1;
          } else {
            ok = xv >= -(1 << (BITS - 1)) && xv <= (1 << (BITS - 1)) - 1;
          }
          if (!ok) {
            const int64_t li = (int64_t)r * p.k + c + 1;
            atomicCAS(p.range_error, 0, li > 0x7FFFFFFF ? 0x7FFFFFFF : (int)li);
            break;
          }
        }
      }
      uint32_t o[8];
      to_slot_order(u, o);
      if (p.digits) {
        uint4* dd = reinterpret_cast<uint4*>(p.digits + ((int64_t)r * p.k_words + WPI * q + wi) * 32);
        dd[0] = make_uint4(o[0], o[1], o[2], o[3]);
        dd[1] = make_uint4(o[4], o[5], o[6], o[7]);
      }
      uint32_t w[BITS];
      unbuild8<BITS>(o, w);
#pragma unroll
      for (int i = 0; i < BITS; ++i) pw[i][wi] = w[i];
    }
    // plane stores: canonical [plane][row][k_words] or tile-major [plane][row/128][Kpad/256][2][128][4]
    // (word w of row r at slab w >> 3, half (w >> 2) & 1, column w & 3); a quad is one 16-byte store
    const int w0 = WPI * q;
    uint32_t* dst = p.tiled ? p.planes + ((int64_t)(r >> 7) * (p.k_words >> 3) + (w0 >> 3)) * 1024 + ((w0 >> 2) & 1) * 512 +
                                  (r & 127) * 4 + (w0 & 3)
                            : p.planes + (int64_t)r * p.k_words + w0;
#pragma unroll
    for (int i = 0; i < BITS; ++i) {
      if constexpr (WPI == 4)
        *reinterpret_cast<uint4*>(dst + (int64_t)i * p.plane_stride) = make_uint4(pw[i][0], pw[i][1], pw[i][2], pw[i][3]);
      else
        dst[(int64_t)i * p.plane_stride] = pw[i][0];
    }
    if constexpr (WPI == 1) {
      // one shared atomic per warp when the warp's words share a row (all but row boundaries)
      const unsigned act = __activemask();
      const int lead = __ffs(act) - 1;
      if (__all_sync(act, rl == __shfl_sync(act, rl, lead))) {
        sum = __reduce_add_sync(act, sum);
        if ((int)(threadIdx.x & 31) == lead) atomicAdd(&s_sum[rl], sum);
      } else {
        atomicAdd(&s_sum[rl], sum);
      }
    } else {
      atomicAdd(&s_sum[rl], sum);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < R; i += blockDim.x)
    if (r0 + i < p.rows) p.row_sum[r0 + i] = s_sum[i];
}

template <int BITS, bool QUANT, int WPI>
__global__ void __launch_bounds__(WPI == 1 ? kPackWordThreads : kPackThreads, WPI == 1 ? 1 : 2) pack_kernel(PackArgs p, const __half* __restrict__ x, float* scale,
                                                             int rows_per_cta) {
  if (p.digits) pdl_launch_dependents();  // activation operand: see pack_release()
  pdl_wait();  // our codes / output buffers may still be in use by the previous kernel
  __shared__ int s_sum[kPackMaxRows];
  __shared__ unsigned s_amax[kPackMaxRows];
  pack_body<BITS, QUANT, WPI>(p, x, scale, rows_per_cta, blockIdx.x, s_sum, s_amax);
  if (!p.digits) pack_release();
}

// Grouped activation packs (apt_pack_grouped): several independent packs WITH digit views in one launch;
// CTA b belongs to the problem i with cta_end[i - 1] <= b < cta_end[i] and packs that problem's rows
// exactly as its own pack_kernel launch would (one word per thread).  Activation operands only, so the
// launch releases its dependents at entry like every digit-view pack.
__global__ void __launch_bounds__(kPackWordThreads, 1) pack_grouped_kernel(const __grid_constant__ PackGroupArgs a) {
  pdl_launch_dependents();
  pdl_wait();
  __shared__ int s_sum[kPackMaxRows];
  __shared__ unsigned s_amax[kPackMaxRows];
  int i = 0;
  while (i + 1 < a.count && (int)blockIdx.x >= a.cta_end[i]) ++i;
  const int cta = (int)blockIdx.x - (i ? a.cta_end[i - 1] : 0);
  const PackArgs& p = a.p[i];
  const __half* x = reinterpret_cast<const __half*>(a.x[i]);
  const int R = a.rows_per_cta[i];
  switch (a.bits[i] * 2 + (a.x[i] ? 1 : 0)) {
#define APT_PG(B)                                                                          \
  case 2 * B: pack_body<B, false, 1>(p, x, a.scale[i], R, cta, s_sum, s_amax); break;      \
  case 2 * B + 1: if (B > 1) pack_body<B, true, 1>(p, x, a.scale[i], R, cta, s_sum, s_amax); break;
    APT_PG(1) APT_PG(2) APT_PG(3) APT_PG(4) APT_PG(5) APT_PG(6) APT_PG(7) APT_PG(8)
#undef APT_PG
    default: break;
  }
}

// rows per CTA: whole rows (row sums without global atomics); tile-major weights: 32 rows so a warp's
// store is 32 consecutive rows of one 16-byte column; otherwise enough rows to give every thread an item
static int pack_rows_per_cta(const PackArgs& p, int wpi) {
  const int Q = p.k_words / wpi;
  if (p.tiled && wpi == 4) return APT_PACK_TILED_ROWS;
  if (wpi == 1 && Q > kPackThreads) return 1;  // a whole row per CTA, one word per thread (pack_threads)
  int R = kPackThreads / (Q > 0 ? Q : 1);
  if (R < 1) R = 1;
  if (R > kPackMaxRows) R = kPackMaxRows;
  return R;
}

// threads per CTA: 256, or for a one-word-per-thread pack of a row longer than 256 words, the row's
// word count (rounded to a warp, at most 1024) so no thread walks two items in series
static int pack_threads(const PackArgs& p, int wpi) {
  const int Q = p.k_words / wpi;
  if (wpi != 1 || Q <= kPackThreads) return kPackThreads;
  return Q >= kPackWordThreads ? kPackWordThreads : (Q + 31) / 32 * 32;
}

template <bool QUANT, int WPI>
static cudaError_t launch_pack_w(const PackArgs& p, const void* x, float* scale, int bits, cudaStream_t stream) {
  const int R = pack_rows_per_cta(p, WPI);
  const dim3 grid((p.rows + R - 1) / R), block(pack_threads(p, WPI));
  const __half* xh = reinterpret_cast<const __half*>(x);
  switch (bits) {
    case 1: return launch_pdl(pack_kernel<1, QUANT, WPI>, grid, block, 0, stream, dim3(1, 1, 1), p, xh, scale, R);
    case 2: return launch_pdl(pack_kernel<2, QUANT, WPI>, grid, block, 0, stream, dim3(1, 1, 1), p, xh, scale, R);
    case 3: return launch_pdl(pack_kernel<3, QUANT, WPI>, grid, block, 0, stream, dim3(1, 1, 1), p, xh, scale, R);
    case 4: return launch_pdl(pack_kernel<4, QUANT, WPI>, grid, block, 0, stream, dim3(1, 1, 1), p, xh, scale, R);
    case 5: return launch_pdl(pack_kernel<5, QUANT, WPI>, grid, block, 0, stream, dim3(1, 1, 1), p, xh, scale, R);
    case 6: return launch_pdl(pack_kernel<6, QUANT, WPI>, grid, block, 0, stream, dim3(1, 1, 1), p, xh, scale, R);
    case 7: return launch_pdl(pack_kernel<7, QUANT, WPI>, grid, block, 0, stream, dim3(1, 1, 1), p, xh, scale, R);
    default: return launch_pdl(pack_kernel<8, QUANT, WPI>, grid, block, 0, stream, dim3(1, 1, 1), p, xh, scale, R);
  }
}

// activation packs (a digit view) take one word per thread; everything else quads
template <bool QUANT>
static cudaError_t launch_pack_t(const PackArgs& p, const void* x, float* scale, int bits, cudaStream_t stream) {
  if (p.digits && p.rows <= APT_PACK_WORD_ROWS) return launch_pack_w<QUANT, 1>(p, x, scale, bits, stream);
  return launch_pack_w<QUANT, 4>(p, x, scale, bits, stream);
}

int pack_group_rows_per_cta(const PackArgs& p) { return pack_rows_per_cta(p, 1); }
int pack_group_threads(const PackArgs& p) { return pack_threads(p, 1); }

cudaError_t launch_pack_grouped(const PackGroupArgs& a, int ctas, int threads, cudaStream_t stream) {
  return launch_pdl(pack_grouped_kernel, dim3(ctas), dim3(threads), 0, stream, dim3(1, 1, 1), a);
}

cudaError_t launch_pack(const PackArgs& p, int bits, cudaStream_t stream) {
  return launch_pack_t<false>(p, nullptr, nullptr, bits, stream);
}

// Fused activation quantize + pack (reading R-Q): fp16 rows -> per-row
// symmetric scale -> signed codes -> planes / digit view / row sums.  Linear quantization
// x = s * x_hat + z with z = 0:
//   s      = RN_f32( max_k |x| / (2^(n-1) - 1) )
//   x_hat  = clamp( rint( RN_f32(x / s) ), -2^(n-1), 2^(n-1) - 1 )   (0 where s == 0)
// in IEEE fp32 (division rounded to nearest, rint half-to-even), so the integer decision is taken in
// the same precision as the oracle's.  Pass 1 reads the CTA's rows for the maxima, pass 2 re-reads
// them (L1/L2) and packs.
cudaError_t launch_quant_pack(const PackArgs& p, const void* x, float* scale, int bits, cudaStream_t stream) {
  if (bits < 2 || bits > 8) return cudaErrorInvalidValue;
  return launch_pack_t<true>(p, x, scale, bits, stream);
}

}  // namespace apt
