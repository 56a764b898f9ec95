// Host-side check of the product's operand rebuild (paper_2508_19087_b200/csrc/common.cuh):
// for every width Q the 32 elements of a plane word land in the SAME byte slots (so operands of
// different widths agree on the K order) and every byte equals the element's offset digit u.
#include <cstdio>
#include <cstdlib>
#include "../../paper_2508_19087_b200/csrc/common.cuh"

template <int Q>
static int check(int ref_slot[32]) {
  int bad = 0;
  // slot of each element: set only plane 0 bit e
  for (int e = 0; e < 32; ++e) {
    uint32_t w[8] = {0}, o[8];
    w[0] = 1u << e;
    apt::rebuild8<Q>(w, o);
    int found = -1, count = 0;
    for (int r = 0; r < 8; ++r)
      for (int b = 0; b < 4; ++b)
        if ((o[r] >> (8 * b)) & 0xFF) { found = 4 * r + b; ++count; }
    if (count != 1) { ++bad; continue; }
    if (ref_slot[e] < 0) ref_slot[e] = found;
    else if (ref_slot[e] != found) ++bad;
  }
  // random words: byte at slot(e) == sum_i 2^i bit_e(w_i)
  srand(1234 + Q);
  for (int t = 0; t < 2000; ++t) {
    uint32_t w[8] = {0}, o[8];
    for (int i = 0; i < Q; ++i) w[i] = ((uint32_t)rand() << 16) ^ (uint32_t)rand();
    apt::rebuild8<Q>(w, o);
    for (int e = 0; e < 32; ++e) {
      uint32_t u = 0;
      for (int i = 0; i < Q; ++i) u |= ((w[i] >> e) & 1u) << i;
      const int s = ref_slot[e];
      if (((o[s / 4] >> (8 * (s % 4))) & 0xFF) != u) ++bad;
    }
    uint32_t o2[8];
    apt::rebuild8_rt(w, Q, o2);
    for (int r = 0; r < 8; ++r) if (o2[r] != o[r]) ++bad;
    // the pack direction: unbuild8 inverts rebuild8 exactly
    uint32_t back[8] = {0};
    apt::unbuild8<Q>(o, back);
    for (int i = 0; i < Q; ++i) if (back[i] != w[i]) ++bad;
    // natural-order digits -> slot order == rebuild8's slots
    uint32_t nat[8] = {0}, so[8];
    for (int e = 0; e < 32; ++e) {
      uint32_t u = 0;
      for (int i = 0; i < Q; ++i) u |= ((w[i] >> e) & 1u) << i;
      nat[e / 4] |= u << (8 * (e % 4));
    }
    apt::to_slot_order(nat, so);
    for (int r = 0; r < 8; ++r) if (so[r] != o[r]) ++bad;
    // the top-bit rebuild of 1- and 2-bit operands: same slots, digit * 2^(8-Q)
    if constexpr (Q == 3 || Q == 4) {
      uint32_t x16[8];
      apt::rebuild_x16<Q>(w, x16);
      for (int r = 0; r < 8; ++r) if (x16[r] != (o[r] << 4)) ++bad;
    }
    if constexpr (Q <= 3) {
      // e2m1 digits: the nibble at each element's slot decodes to the signed code u - 2^(Q-1)
      static const float kE2m1[8] = {0.f, 0.5f, 1.f, 1.5f, 2.f, 3.f, 4.f, 6.f};
      uint32_t g4[4];
      apt::rebuild_e2m1<Q>(w, g4);
      for (int e = 0; e < 32; ++e) {
        int u = 0;
        for (int i = 0; i < Q; ++i) u |= (int)((w[i] >> e) & 1u) << i;
        const int x = u - (1 << (Q - 1));
        const int s = ref_slot[e];  // rebuild8 slot 4 * reg + byte; reg = 2c + hi, nibble = 2 * byte + hi
        const int reg = s / 4, byte = s % 4, c = reg / 2, hi = reg % 2;
        const uint32_t nib = (g4[c] >> (4 * (2 * byte + hi))) & 0xFu;
        const float v = (nib & 8u ? -1.f : 1.f) * kE2m1[nib & 7u];
        if (v != (float)x) ++bad;
      }
    }
    if constexpr (Q <= 2) {
      uint32_t hi[8];
      apt::rebuild_hi<Q>(w, hi);
      for (int r = 0; r < 8; ++r)
        for (int b = 0; b < 4; ++b)
          if (((hi[r] >> (8 * b)) & 0xFF) != (((o[r] >> (8 * b)) & 0xFF) << (8 - Q))) ++bad;
    }
  }
  return bad;
}

int main() {
  int slot[32];
  for (int e = 0; e < 32; ++e) slot[e] = -1;
  int bad = check<1>(slot) + check<2>(slot) + check<3>(slot) + check<4>(slot) + check<5>(slot) +
            check<6>(slot) + check<7>(slot) + check<8>(slot);
  int seen[32] = {0};
  for (int e = 0; e < 32; ++e) if (slot[e] >= 0) seen[slot[e]]++;
  for (int s = 0; s < 32; ++s) if (seen[s] != 1) ++bad;
  printf("%s %d\n", bad ? "FAIL" : "OK", bad);
  return bad ? 1 : 0;
}
