// pack.cu — INT -> bipolar-INT bit-plane packing on the device (§4.1 Steps 1-3).
//
// One CTA per matrix row, one thread per 32-bit output word position (32 consecutive K
// elements) at a time and loads those 32 codes as two 16-byte vectors (a warp reads 1 KB of
// contiguous codes).  Per 4-byte group of codes:
//   signed -> offset bits   u = x + 2^(n-1) mod 2^n, i.e. the sign-bit flip of P:202, done
//                           bytewise without cross-byte carries;
//   plane i nibble          ((u >> i) & 0x01010101) * 0x01020408 >> 24 gathers bit i of the
//                           four bytes into 4 consecutive bits;
// and the eight nibbles of a plane form the output word (element c -> bit c%32, LSB first).
// Row sums of the signed codes use dp4a; the CTA reduces them without atomics.
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "sync.cuh"

namespace apt {


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

// One 32-element word of row r: offset digits u[8] (4 per uint32) -> the BITS plane words (element
// c -> bit c % 32, LSB first) and, when requested, the kernel-order u8 digit view.
template <int BITS>
__device__ __forceinline__ void store_word(const PackArgs& p, int r, int w, const uint32_t (&u)[8]) {
  // planes: bit i of every element, element c -> bit c % 32 (LSB first)
  uint32_t* dst = p.tiled ? p.planes + ((int64_t)(r >> 7) * (p.k_words >> 3) + (w >> 3)) * 1024 +
                                ((w >> 2) & 1) * 512 + (r & 127) * 4 + (w & 3)
                          : p.planes + (int64_t)r * p.k_words + w;
  uint32_t pw[BITS];
#pragma unroll
  for (int i = 0; i < BITS; ++i) {
    uint32_t word = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t nib = (((u[j] >> i) & 0x01010101u) * 0x01020408u) >> 24;
      word |= nib << (4 * j);
    }
    dst[(int64_t)i * p.plane_stride] = word;
    pw[i] = word;
  }
  if (p.digits) {
    // the optional digit view: the same word through the kernels' operand rebuild
    uint32_t d[8];
    rebuild8<BITS>(pw, d);
    uint4* dd = reinterpret_cast<uint4*>(p.digits + ((int64_t)r * p.k_words + w) * 32);
    dd[0] = make_uint4(d[0], d[1], d[2], d[3]);
    dd[1] = make_uint4(d[4], d[5], d[6], d[7]);
  }
}

// CTA reduction of a row's signed-code sum (pads contribute 0) into p.row_sum[r]
__device__ __forceinline__ void row_sum_store(const PackArgs& p, int r, int sum) {
  __shared__ int red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x < 32) {
    int v = threadIdx.x < (int)(blockDim.x >> 5) ? red[threadIdx.x] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) p.row_sum[r] = v;
  }
}

// Stream order with programmatic dependent launch (include/apt.h "General contract"): the GEMMs
// read weight-side operands (planes, row sums, scales) BEFORE griddepcontrol.wait, so a kernel that
// writes them must not release its dependents early.  The pack kernels therefore never execute
// griddepcontrol.launch_dependents (the dependents launch only once every CTA has exited) and make
// their stores visible at GPU scope before exiting (pack_release).
__device__ __forceinline__ void pack_release() { __threadfence(); }

template <int BITS>
__global__ void __launch_bounds__(1024) pack_kernel(PackArgs p) {
  pdl_wait();  // our codes / output buffers may still be in use by the previous kernel
  const int r = blockIdx.x;
  const int8_t* row = p.codes + (int64_t)r * p.ld;
  const bool vec_ok = ((reinterpret_cast<uintptr_t>(row) & 15u) == 0);
  int sum = 0;
  for (int w = threadIdx.x; w < p.k_words; w += blockDim.x) {
    const int c0 = w * 32;
    uint32_t v[8];
    if (vec_ok && c0 + 32 <= p.k) {
      const uint4 lo = __ldg(reinterpret_cast<const uint4*>(row + c0));
      const uint4 hi = __ldg(reinterpret_cast<const uint4*>(row + c0 + 16));
      v[0] = lo.x; v[1] = lo.y; v[2] = lo.z; v[3] = lo.w;
      v[4] = hi.x; v[5] = hi.y; v[6] = hi.z; v[7] = hi.w;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        uint32_t word = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int c = c0 + 4 * j + b;
          const uint32_t byte = (c < p.k) ? (uint32_t)(uint8_t)row[c] : 0u;  // pad = signed code 0
          word |= byte << (8 * b);
        }
        v[j] = word;
      }
      if (p.enc == 1) {
        // bipolar pads must also be neutral: pad positions hold x' = 1 (signed 0) after conversion
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
          for (int b = 0; b < 4; ++b)
            if (c0 + 4 * j + b >= p.k) v[j] |= 1u << (8 * b);
      }
    }
    uint32_t u[8];
    bool bad = false;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint32_t x = v[j];
      if (p.enc == 1) {
        // bipolar x' (odd) -> signed x = (x' - 1) / 2 = x' >> 1 (arithmetic, bytewise)
        bad |= (x & 0x01010101u) != 0x01010101u;
        x = ((x >> 1) & 0x7F7F7F7Fu) | (x & 0x80808080u);
      }
      u[j] = to_offset4<BITS>(x);
      bad |= from_offset4<BITS>(u[j]) != x;
      sum = __dp4a((int)x, 0x01010101, sum);
    }
    if (bad && p.range_error) {
      for (int c = c0; c < c0 + 32 && c < p.k; ++c) {
        int x = row[c];
        bool ok;
        if (p.enc == 1) {
          ok = (x & 1) && x >= -((1 << BITS) - 1) && x <= (1 << BITS) - 1;
          x = x >> 1;
        } else {
          ok = x >= -(1 << (BITS - 1)) && x <= (1 << (BITS - 1)) - 1;
        }
        if (!ok) {
          const int64_t li = (int64_t)r * p.k + c + 1;
          atomicCAS(p.range_error, 0, li > 0x7FFFFFFF ? 0x7FFFFFFF : (int)li);
          break;
        }
      }
    }
    store_word<BITS>(p, r, w, u);
  }
  row_sum_store(p, r, sum);
  pack_release();
}

cudaError_t launch_pack(const PackArgs& p, int bits, cudaStream_t stream) {
  // one CTA per row with (up to) one thread per 32-element word: a single latency round for K <= 32768
  int threads = ((p.k_words + 31) / 32) * 32;
  if (threads > 1024) threads = 1024;
  if (threads < 32) threads = 32;
  dim3 grid(p.rows), block(threads);
  switch (bits) {
    case 1: return launch_pdl(pack_kernel<1>, grid, block, 0, stream, dim3(1, 1, 1), p);
    case 2: return launch_pdl(pack_kernel<2>, grid, block, 0, stream, dim3(1, 1, 1), p);
    case 3: return launch_pdl(pack_kernel<3>, grid, block, 0, stream, dim3(1, 1, 1), p);
    case 4: return launch_pdl(pack_kernel<4>, grid, block, 0, stream, dim3(1, 1, 1), p);
    case 5: return launch_pdl(pack_kernel<5>, grid, block, 0, stream, dim3(1, 1, 1), p);
    case 6: return launch_pdl(pack_kernel<6>, grid, block, 0, stream, dim3(1, 1, 1), p);
    case 7: return launch_pdl(pack_kernel<7>, grid, block, 0, stream, dim3(1, 1, 1), p);
    default: return launch_pdl(pack_kernel<8>, grid, block, 0, stream, dim3(1, 1, 1), p);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Fused activation quantize + pack (reading R-Q): fp16 rows -> per-row
// symmetric scale -> signed codes -> planes / digit view / row sums, one read of the row from HBM
// (the second pass hits L1/L2).  Linear quantization x = s * x_hat + z with z = 0:
//   s      = RN_f32( max_k |x| / (2^(n-1) - 1) )
//   x_hat  = clamp( rint( RN_f32(x / s) ), -2^(n-1), 2^(n-1) - 1 )   (0 where s == 0)
// in IEEE fp32 (division rounded to nearest, rint half-to-even), so the integer decision is taken in
// the same precision as the oracle's.
template <int BITS>
__global__ void __launch_bounds__(1024) quant_pack_kernel(PackArgs p, const __half* __restrict__ x, float* scale) {
  pdl_wait();  // no early trigger: see pack_release()
  const int r = blockIdx.x;
  const __half* row = x + (int64_t)r * p.ld;
  const bool vec_ok = ((reinterpret_cast<uintptr_t>(row) & 15u) == 0);
  auto load32 = [&](int c0, float (&f)[32]) {
    if (vec_ok && c0 + 32 <= p.k) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(row + c0) + q);
        const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float2 g = __half22float2(h[t]);
          f[8 * q + 2 * t] = g.x;
          f[8 * q + 2 * t + 1] = g.y;
        }
      }
    } else {
#pragma unroll
      for (int e = 0; e < 32; ++e) f[e] = (c0 + e < p.k) ? __half2float(row[c0 + e]) : 0.f;
    }
  };
  // pass 1: the row's absolute maximum
  float amax = 0.f;
  for (int w = threadIdx.x; w < p.k_words; w += blockDim.x) {
    float f[32];
    load32(w * 32, f);
#pragma unroll
    for (int e = 0; e < 32; ++e) amax = fmaxf(amax, fabsf(f[e]));
  }
  __shared__ float s_red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = amax;
  __syncthreads();
  float m = 0.f;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) m = fmaxf(m, s_red[i]);
  constexpr float kQmax = (float)((1 << (BITS - 1)) - 1);
  const float s = __fdiv_rn(m, kQmax);
  if (threadIdx.x == 0) scale[r] = s;
  // pass 2: codes -> planes
  int sum = 0;
  for (int w = threadIdx.x; w < p.k_words; w += blockDim.x) {
    float f[32];
    load32(w * 32, f);
    uint32_t u[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint32_t word = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        float q = s > 0.f ? rintf(__fdiv_rn(f[4 * j + b], s)) : 0.f;
        q = fminf(fmaxf(q, -(kQmax + 1.f)), kQmax);
        word |= ((uint32_t)(int)q & 0xFFu) << (8 * b);
      }
      sum = __dp4a((int)word, 0x01010101, sum);
      u[j] = to_offset4<BITS>(word);
    }
    store_word<BITS>(p, r, w, u);
  }
  row_sum_store(p, r, sum);
  pack_release();
}

cudaError_t launch_quant_pack(const PackArgs& p, const void* x, float* scale, int bits, cudaStream_t stream) {
  int threads = ((p.k_words + 31) / 32) * 32;
  if (threads > 1024) threads = 1024;
  if (threads < 32) threads = 32;
  dim3 grid(p.rows), block(threads);
  const __half* xh = reinterpret_cast<const __half*>(x);
  switch (bits) {
    case 2: return launch_pdl(quant_pack_kernel<2>, grid, block, 0, stream, dim3(1, 1, 1), p, xh, scale);
    case 3: return launch_pdl(quant_pack_kernel<3>, grid, block, 0, stream, dim3(1, 1, 1), p, xh, scale);
    case 4: return launch_pdl(quant_pack_kernel<4>, grid, block, 0, stream, dim3(1, 1, 1), p, xh, scale);
    case 5: return launch_pdl(quant_pack_kernel<5>, grid, block, 0, stream, dim3(1, 1, 1), p, xh, scale);
    case 6: return launch_pdl(quant_pack_kernel<6>, grid, block, 0, stream, dim3(1, 1, 1), p, xh, scale);
    case 7: return launch_pdl(quant_pack_kernel<7>, grid, block, 0, stream, dim3(1, 1, 1), p, xh, scale);
    case 8: return launch_pdl(quant_pack_kernel<8>, grid, block, 0, stream, dim3(1, 1, 1), p, xh, scale);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace apt
