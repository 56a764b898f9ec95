// common.cuh — device helpers shared by the APT kernels (product path only; the CPU oracle
// under oracle/ shares nothing with this file).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace apt {

// ---------------------------------------------------------------------------------------------
// Operand rebuild: bit-planes -> full-width unsigned digits (the "shift" half of the paper's
// shift-add recovery, folded onto the operands).
//
// Input : Q plane words w[i] (i = plane = bit significance), each holding bit i of the
//         bipolar pattern u = x + 2^(Q-1) of 32 consecutive K elements (§4.1 Step 2).
// Output: 8 registers of 4 bytes; every byte is one element's u in [0, 2^Q), i.e. the digit
//         sum_i 2^i u_i.  The 32 elements land in the 32 byte slots through a fixed bijection
//         (a butterfly bit transpose).  The K order inside a word is irrelevant to the GEMM as long
//         as BOTH operands go through this same function for the same word (sum over K commutes),
//         so the exported packed format stays canonical while the kernel uses the cheapest order.
//
// Cost (after constant folding): about 20 ops for Q <= 2, 28 for Q = 4, 48 for Q = 8 per 32 elements.
// ---------------------------------------------------------------------------------------------
// (x & m) | (y & ~m) as ONE lop3 on the device (the compiler tends to emit two)
__host__ __device__ __forceinline__ uint32_t bit_select(uint32_t x, uint32_t y, uint32_t m) {
#ifdef __CUDA_ARCH__
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(d) : "r"(x), "r"(y), "r"(m));
  return d;
#else
  return (x & m) | (y & ~m);
#endif
}

__host__ __device__ __forceinline__ void bf_pair(uint32_t lo, uint32_t hi, int s, uint32_t m, uint32_t& a, uint32_t& b) {
  // a: even fields of lo in the low half, even fields of hi in the high half (field width s)
  // b: odd fields likewise.  m = mask of the low s bits of every 2s-bit field.
  a = bit_select(lo, hi << s, m);
  b = bit_select(lo >> s, hi, m);
}

// The element -> byte-slot bijection is the SAME for every Q (planes >= Q are zero and the
// compiler folds them away), so operands of different widths agree on the K order.
template <int Q>
__host__ __device__ __forceinline__ void rebuild8(const uint32_t* w, uint32_t (&o)[8]) {
  static_assert(Q >= 1 && Q <= 8, "bits");
  if constexpr (Q <= 4) {
    const uint32_t w1 = (Q >= 2) ? w[1] : 0u;
    const uint32_t w2 = (Q >= 3) ? w[2] : 0u;
    const uint32_t w3 = (Q >= 4) ? w[3] : 0u;
    uint32_t e01, f01, e23, f23, g[4];
    bf_pair(w[0], w1, 1, 0x55555555u, e01, f01);
    bf_pair(w2, w3, 1, 0x55555555u, e23, f23);
    bf_pair(e01, e23, 2, 0x33333333u, g[0], g[1]);
    bf_pair(f01, f23, 2, 0x33333333u, g[2], g[3]);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      o[2 * c] = g[c] & 0x0F0F0F0Fu;
      o[2 * c + 1] = (g[c] >> 4) & 0x0F0F0F0Fu;
    }
  } else {
    const uint32_t w5 = (Q >= 6) ? w[5] : 0u;
    const uint32_t w6 = (Q >= 7) ? w[6] : 0u;
    const uint32_t w7 = (Q >= 8) ? w[7] : 0u;
    uint32_t e01, f01, e23, f23, e45, f45, e67, f67, g[8];
    bf_pair(w[0], w[1], 1, 0x55555555u, e01, f01);
    bf_pair(w[2], w[3], 1, 0x55555555u, e23, f23);
    bf_pair(w[4], w5, 1, 0x55555555u, e45, f45);
    bf_pair(w6, w7, 1, 0x55555555u, e67, f67);
    bf_pair(e01, e23, 2, 0x33333333u, g[0], g[1]);
    bf_pair(e45, e67, 2, 0x33333333u, g[2], g[3]);
    bf_pair(f01, f23, 2, 0x33333333u, g[4], g[5]);
    bf_pair(f45, f67, 2, 0x33333333u, g[6], g[7]);
    bf_pair(g[0], g[2], 4, 0x0F0F0F0Fu, o[0], o[1]);
    bf_pair(g[1], g[3], 4, 0x0F0F0F0Fu, o[2], o[3]);
    bf_pair(g[4], g[6], 4, 0x0F0F0F0Fu, o[4], o[5]);
    bf_pair(g[5], g[7], 4, 0x0F0F0F0Fu, o[6], o[7]);
  }
}

// rebuild8's slot order is "strided": register j byte b holds element 8b + rev3(j) (rev3 = 3-bit
// reversal).  For 1- and 2-bit operands that order is cheaper to produce one register at a time with
// the digit placed in the TOP bits of its byte: register j = each plane shifted so that bit
// 8b + rev3(j) lands in bit 8 - Q + i of byte b, then masked.  The left shifts compile to IMAD.SHL
// (FMA pipe), leaving only the masks on the integer ALU pipe (8 LOP3 per word at Q = 1 against ~20
// for the butterfly).  Every byte is u * 2^(8-Q); the GEMM divides the exact sum by 2^(8-Q).
__host__ __device__ __forceinline__ constexpr int rev3(int j) { return ((j & 1) << 2) | (j & 2) | ((j >> 2) & 1); }

template <int S>
__host__ __device__ __forceinline__ uint32_t shl_signed(uint32_t v) {
  if constexpr (S >= 0) return v << S; else return v >> (-S);
}

template <int Q>
__host__ __device__ __forceinline__ void rebuild_hi(const uint32_t* w, uint32_t (&o)[8]) {
  static_assert(Q == 1 || Q == 2, "rebuild_hi covers 1- and 2-bit operands");
  if constexpr (Q == 1) {
    o[0] = shl_signed<7 - rev3(0)>(w[0]) & 0x80808080u;
    o[1] = shl_signed<7 - rev3(1)>(w[0]) & 0x80808080u;
    o[2] = shl_signed<7 - rev3(2)>(w[0]) & 0x80808080u;
    o[3] = shl_signed<7 - rev3(3)>(w[0]) & 0x80808080u;
    o[4] = shl_signed<7 - rev3(4)>(w[0]) & 0x80808080u;
    o[5] = shl_signed<7 - rev3(5)>(w[0]) & 0x80808080u;
    o[6] = shl_signed<7 - rev3(6)>(w[0]) & 0x80808080u;
    o[7] = shl_signed<7 - rev3(7)>(w[0]) & 0x80808080u;
  } else {
#define APT_HI2(j) o[j] = bit_select(shl_signed<6 - rev3(j)>(w[0]), shl_signed<7 - rev3(j)>(w[1]) & 0x80808080u, 0x40404040u)
    APT_HI2(0); APT_HI2(1); APT_HI2(2); APT_HI2(3); APT_HI2(4); APT_HI2(5); APT_HI2(6); APT_HI2(7);
#undef APT_HI2
  }
}

// rebuild8<Q> for Q = 3, 4 with every digit scaled by 16 (the nibble left in the high half of its
// byte): the last butterfly stage becomes one mask (+ one FMA-pipe left shift) per register instead of
// a right shift and a mask on the ALU pipe.  Same slots as rebuild8.
template <int Q>
__host__ __device__ __forceinline__ void rebuild_x16(const uint32_t* w, uint32_t (&o)[8]) {
  static_assert(Q == 3 || Q == 4, "rebuild_x16 covers 3- and 4-bit operands");
  const uint32_t w3 = (Q >= 4) ? w[3] : 0u;
  uint32_t e01, f01, e23, f23, g[4];
  bf_pair(w[0], w[1], 1, 0x55555555u, e01, f01);
  bf_pair(w[2], w3, 1, 0x55555555u, e23, f23);
  bf_pair(e01, e23, 2, 0x33333333u, g[0], g[1]);
  bf_pair(f01, f23, 2, 0x33333333u, g[2], g[3]);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    o[2 * c] = (g[c] << 4) & 0xF0F0F0F0u;
    o[2 * c + 1] = g[c] & 0xF0F0F0F0u;
  }
}

// Signed e2m1 (fp4) digits for the kind::mxf4 tensor-core path (1 <= Q <= 3): the signed code
// x = u - 2^(Q-1) in [-4, 3] is exactly representable in e2m1 (0, 0.5, 1, 1.5, 2, 3, 4, 6 and signs;
// nibble = sign << 3 | magnitude code, |x| 1 -> 2, 2 -> 4, 3 -> 5, 4 -> 6).  Each nibble bit is a boolean
// function of the Q plane bits (one lop3 per bit plane), then the first two butterfly stages of
// rebuild8 interleave the four bit planes into nibbles: g[c] nibble 2b = element 8b + rev3(2c), nibble
// 2b + 1 = element 8b + rev3(2c + 1) (rebuild8's slots, two per byte), so weights and tokens rebuilt
// with this function agree on K.  16 bytes per 32 elements.
template <int Q>
__host__ __device__ __forceinline__ void rebuild_e2m1(const uint32_t* w, uint32_t (&g)[4]) {
  static_assert(Q >= 1 && Q <= 3, "e2m1 holds signed codes of at most 3 bits");
  uint32_t b0, b1, b2, b3;
  if constexpr (Q == 1) {  // x = u0 - 1: -1 -> 1010, 0 -> 0000
    b3 = ~w[0];
    b2 = 0u;
    b1 = ~w[0];
    b0 = 0u;
  } else if constexpr (Q == 2) {  // x = u - 2: -2 -> 1100, -1 -> 1010, 0 -> 0000, 1 -> 0010
    b3 = ~w[1];
    b2 = ~(w[1] | w[0]);
    b1 = w[0];
    b0 = 0u;
  } else {  // x = u - 4: -4 1110, -3 1101, -2 1100, -1 1010, 0 0000, 1 0010, 2 0100, 3 0101
    const uint32_t u0 = w[0], u1 = w[1], u2 = w[2];
    b3 = ~u2;
    b2 = (u2 & u1) | (~u2 & ~(u1 & u0));
    b1 = (u2 & ~u1 & u0) | (~u2 & ~(u1 ^ u0));
    b0 = u0 & ~(u2 ^ u1);
  }
  uint32_t e01, f01, e23, f23;
  bf_pair(b0, b1, 1, 0x55555555u, e01, f01);
  bf_pair(b2, b3, 1, 0x55555555u, e23, f23);
  bf_pair(e01, e23, 2, 0x33333333u, g[0], g[1]);
  bf_pair(f01, f23, 2, 0x33333333u, g[2], g[3]);
}

// The inverse of rebuild8<Q> (the pack direction): 8 registers of digits in rebuild8's slot order
// -> Q plane words (element c -> bit c).  bf_pair is an involution for a fixed (s, m), so the
// inverse is the same butterfly run backwards.  Digits must be < 2^Q.
template <int Q>
__host__ __device__ __forceinline__ void unbuild8(const uint32_t (&o)[8], uint32_t* w) {
  static_assert(Q >= 1 && Q <= 8, "bits");
  if constexpr (Q <= 4) {
    uint32_t g[4], e01, f01, e23, f23;
#pragma unroll
    for (int c = 0; c < 4; ++c) g[c] = o[2 * c] | (o[2 * c + 1] << 4);
    bf_pair(g[0], g[1], 2, 0x33333333u, e01, e23);
    bf_pair(g[2], g[3], 2, 0x33333333u, f01, f23);
    uint32_t w0, w1, w2, w3;
    bf_pair(e01, f01, 1, 0x55555555u, w0, w1);
    bf_pair(e23, f23, 1, 0x55555555u, w2, w3);
    w[0] = w0;
    if (Q >= 2) w[1] = w1;
    if (Q >= 3) w[2] = w2;
    if (Q >= 4) w[3] = w3;
  } else {
    uint32_t g[8], e01, f01, e23, f23, e45, f45, e67, f67, x[8];
    bf_pair(o[0], o[1], 4, 0x0F0F0F0Fu, g[0], g[2]);
    bf_pair(o[2], o[3], 4, 0x0F0F0F0Fu, g[1], g[3]);
    bf_pair(o[4], o[5], 4, 0x0F0F0F0Fu, g[4], g[6]);
    bf_pair(o[6], o[7], 4, 0x0F0F0F0Fu, g[5], g[7]);
    bf_pair(g[0], g[1], 2, 0x33333333u, e01, e23);
    bf_pair(g[2], g[3], 2, 0x33333333u, e45, e67);
    bf_pair(g[4], g[5], 2, 0x33333333u, f01, f23);
    bf_pair(g[6], g[7], 2, 0x33333333u, f45, f67);
    bf_pair(e01, f01, 1, 0x55555555u, x[0], x[1]);
    bf_pair(e23, f23, 1, 0x55555555u, x[2], x[3]);
    bf_pair(e45, f45, 1, 0x55555555u, x[4], x[5]);
    bf_pair(e67, f67, 1, 0x55555555u, x[6], x[7]);
#pragma unroll
    for (int i = 0; i < Q; ++i) w[i] = x[i];
  }
}

__host__ __device__ __forceinline__ uint32_t byte_perm(uint32_t a, uint32_t b, uint32_t sel) {
#ifdef __CUDA_ARCH__
  return __byte_perm(a, b, sel);
#else
  const uint64_t v = ((uint64_t)b << 32) | a;
  uint32_t r = 0;
  for (int i = 0; i < 4; ++i) r |= (uint32_t)((v >> (8 * ((sel >> (4 * i)) & 7))) & 0xFF) << (8 * i);
  return r;
#endif
}

// 32 digits in natural order (register i byte c = element 4i + c) -> rebuild8's slot order
// (register j byte b = element 8b + rev3(j)): two 4 x 4 byte transposes, 16 PRMT.
__host__ __device__ __forceinline__ void to_slot_order(const uint32_t (&n)[8], uint32_t (&o)[8]) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint32_t t0 = byte_perm(n[h], n[2 + h], 0x5140u), t1 = byte_perm(n[h], n[2 + h], 0x7362u);
    const uint32_t t2 = byte_perm(n[4 + h], n[6 + h], 0x5140u), t3 = byte_perm(n[4 + h], n[6 + h], 0x7362u);
    // column c of the transpose holds elements 8b + 4h + c; slot register rev3(4h + c)
    o[h ? 1 : 0] = byte_perm(t0, t2, 0x5410u);
    o[h ? 5 : 4] = byte_perm(t0, t2, 0x7632u);
    o[h ? 3 : 2] = byte_perm(t1, t3, 0x5410u);
    o[h ? 7 : 6] = byte_perm(t1, t3, 0x7632u);
  }
}

// Runtime-width dispatch (used where the width is not a template parameter, e.g. token rebuild).
__host__ __device__ __forceinline__ void rebuild8_rt(const uint32_t* w, int q, uint32_t (&o)[8]) {
  switch (q) {
    case 1: rebuild8<1>(w, o); break;
    case 2: rebuild8<2>(w, o); break;
    case 3: rebuild8<3>(w, o); break;
    case 4: rebuild8<4>(w, o); break;
    case 5: rebuild8<5>(w, o); break;
    case 6: rebuild8<6>(w, o); break;
    case 7: rebuild8<7>(w, o); break;
    default: rebuild8<8>(w, o); break;
  }
}

// ---------------------------------------------------------------------------------------------
// Epilogue arithmetic (reading Q1/Q10; SURVEY §8c identities I2/I3).
// The kernels accumulate U = sum_{k<Kpad} u_a u_w over unsigned digits u = x + h (h = 2^(n-1)).
// Since pads are signed code 0 (u = h):
//     Y  = U - h_w * RA[m] - h_a * RW[n] - Kpad * h_a * h_w      (signed product)
//     Y' = 4Y + 2 RA[m] + 2 RW[n] + K                           (bipolar product)
// evaluated modulo 2^32 (the true values fit in int32 by the Q8 bound, so wraparound is exact).
// ---------------------------------------------------------------------------------------------
struct EpilogueArgs {
  const int32_t* w_rowsum;  // RW[N]
  const int32_t* a_rowsum;  // RA[M]
  const float* w_scale;     // [N]
  const float* a_scale;     // [M] or null
  void* out;
  int64_t ldo;
  int32_t kind;             // apt_out_kind
  int32_t layout;           // apt_layout
  int32_t M, N, K, kpad;
  int32_t h_w, h_a;         // 2^(wbits-1), 2^(abits-1)
};

// Epilogue with the rank-1 / scale operands already in registers.
__device__ __forceinline__ void epilogue_store_v(const EpilogueArgs& e, int m, int n, uint32_t U, int32_t ra_,
                                                 int32_t rw_, float wsc, float asc) {
  const uint32_t ra = (uint32_t)ra_, rw = (uint32_t)rw_;
  const uint32_t y = U - (uint32_t)e.h_w * ra - (uint32_t)e.h_a * rw -
                     (uint32_t)e.kpad * (uint32_t)e.h_a * (uint32_t)e.h_w;
  const int64_t off = e.layout == 0 ? (int64_t)m * e.ldo + n : (int64_t)n * e.ldo + m;
  if (e.kind == 0) {
    reinterpret_cast<int32_t*>(e.out)[off] = (int32_t)y;
  } else if (e.kind == 1) {
    const uint32_t yb = 4u * y + 2u * ra + 2u * rw + (uint32_t)e.K;
    reinterpret_cast<int32_t*>(e.out)[off] = (int32_t)yb;
  } else {
    const float v = ((float)(int32_t)y * wsc) * asc;
    unsigned short h;
    asm("cvt.rn.f16.f32 %0, %1;" : "=h"(h) : "f"(v));
    reinterpret_cast<unsigned short*>(e.out)[off] = h;
  }
}

// two fp32 -> two fp16 (round to nearest even each, IEEE overflow to inf), low half = a
__device__ __forceinline__ uint32_t pack_f16x2(float a, float b) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}

__device__ __forceinline__ void epilogue_store(const EpilogueArgs& e, int m, int n, uint32_t U) {
  epilogue_store_v(e, m, n, U, __ldg(e.a_rowsum + m), __ldg(e.w_rowsum + n),
                   e.kind == 2 ? __ldg(e.w_scale + n) : 0.f, (e.kind == 2 && e.a_scale) ? __ldg(e.a_scale + m) : 1.f);
}

// ---------------------------------------------------------------------------------------------
// Small PTX wrappers
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t ld_dsmem_u32(uint32_t local_smem_addr, uint32_t rank) {
  uint32_t remote, v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_smem_addr), "r"(rank));
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(remote) : "memory");
  return v;
}

}  // namespace apt
