// apt.cu — the C-ABI boundary (include/apt.h): argument validation, the config selector and
// kernel dispatch.  No torch types, no allocation, no synchronization.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>
#include <cuda_runtime.h>

#include "../../include/apt.h"
#include "kernels.h"
#include "sync.cuh"


namespace {

// The library's only global state (include/apt.h "Thread-safe"): the SM count of each device, queried
// once under a mutex.  Without a device (CPU-only hosts) the B200's 148 is assumed, so the selector
// stays a pure function of (M, N, K, p, q) on a given device.
std::mutex g_dev_mu;
int g_dev_sms[64] = {0};

int device_sms() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
    cudaGetLastError();
    return 148;
  }
  std::lock_guard<std::mutex> lk(g_dev_mu);
  if (g_dev_sms[dev] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) {
      cudaGetLastError();
      v = 148;
    }
    g_dev_sms[dev] = v;
  }
  return g_dev_sms[dev];
}


int64_t kpad_of(int64_t k) { return ((k + APT_KPAD_QUANTUM - 1) / APT_KPAD_QUANTUM) * APT_KPAD_QUANTUM; }

bool bound_ok(int64_t k, int wbits, int abits) {
  // reading Q8: Kpad * (2^abits - 1) * (2^wbits - 1) < 2^31 bounds |Y|, |Y'| and every unsigned partial sum
  return kpad_of(k) * ((1ll << abits) - 1) * ((1ll << wbits) - 1) < (1ll << 31);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

apt_status validate_packed(const apt_packed* P, int32_t rows, int32_t k, int32_t bits) {
  if (!P || !P->planes || !P->row_sum) return APT_ERR_INVALID_ARGUMENT;
  if (P->rows != rows || P->k != k || P->bits != bits) return APT_ERR_INVALID_ARGUMENT;
  if (P->k_words != kpad_of(k) / 32) return APT_ERR_INVALID_ARGUMENT;
  if (!aligned16(P->planes)) return APT_ERR_INVALID_ARGUMENT;
  if (P->layout != APT_PACK_ROWS && P->layout != APT_PACK_TILED) return APT_ERR_INVALID_ARGUMENT;
  return APT_OK;
}

apt_status validate_config(const apt_config* c, int32_t M, int32_t N, int32_t K, int32_t wbits, int32_t abits) {
  const int kw = (int)(kpad_of(K) / 32);
  if (c->w_digit != wbits || c->a_digit != abits) return APT_ERR_UNSUPPORTED;  // full-width digits only
  if (c->mma_kind != APT_MMA_I8 && c->mma_kind != APT_MMA_MXF4) return APT_ERR_UNSUPPORTED;
  if (c->kernel == APT_KERNEL_PF) {
    if (c->bm != 128 || (c->bn != 128 && c->bn != 192 && c->bn != 256) || c->bk != 128 ||
        c->stages != (c->bn == 128 ? 6 : c->bn == 192 ? 4 : 3) || c->split_k != 1 || c->cluster_n != 1 || c->cta_pair != 0)
      return APT_ERR_UNSUPPORTED;
    // 2 x 192 accumulator + A ring = 512 TMEM columns; 2 x 256 with the A ring in shared memory: i8 only
    if (c->bn != 128 && c->mma_kind != APT_MMA_I8) return APT_ERR_UNSUPPORTED;
    if (c->mma_kind == APT_MMA_MXF4 && (wbits > 3 || abits > 3 || kpad_of(K) * 16ll >= (1ll << 24)))
      return APT_ERR_UNSUPPORTED;
    // i8: weight digits scaled by 2^s (<= 255 each) accumulate in s32: Kpad * 255 * 255 < 2^31
    if (c->mma_kind == APT_MMA_I8 && kpad_of(K) * 255ll * 255ll >= (1ll << 31)) return APT_ERR_UNSUPPORTED;
    return APT_OK;
  }
  if (c->mma_kind == APT_MMA_MXF4) {
    // signed e2m1 digits: codes of at most 3 bits; the tcgen05 prefill tile, one K range, no cluster;
    // f32 accumulation exact while every partial sum is an integer below 2^24 (|x y| <= 16)
    if (wbits > 3 || abits > 3 || c->kernel != APT_KERNEL_TC) return APT_ERR_UNSUPPORTED;
    if ((c->bn != 128 && c->bn != 256) || c->split_k != 1 || c->cluster_n != 1 || c->bm != 128 || c->bk != 128)
      return APT_ERR_UNSUPPORTED;
    if (c->stages != apt::tc_stages(wbits, c->bn) || c->cta_pair != 0) return APT_ERR_UNSUPPORTED;
    if (kpad_of(K) * 16ll >= (1ll << 24)) return APT_ERR_UNSUPPORTED;
    return APT_OK;
  }
  if (c->kernel == APT_KERNEL_GEMV) {
    if (M > 4 || c->bm != 32 || c->bn != M || c->bk != 128 || (c->split_k != 8 && c->split_k != 16) ||
        c->stages != 1)
      return APT_ERR_UNSUPPORTED;
    if (c->cta_pair != 0 || c->cluster_n != 1) return APT_ERR_UNSUPPORTED;
    return APT_OK;
  }
  if (c->kernel == APT_KERNEL_SKINNY) {
    if (c->bm != 16 || (c->bn != 8 && c->bn != 16) || c->bk != 256 || c->stages != 1) return APT_ERR_UNSUPPORTED;
    if (c->split_k != 4 && c->split_k != 8 && c->split_k != 16) return APT_ERR_UNSUPPORTED;
    if (c->cta_pair != 0 || c->cluster_n != 1) return APT_ERR_UNSUPPORTED;
    return APT_OK;
  }
  if (c->kernel == APT_KERNEL_DEC) {
    if (M > 16 || c->bm != 32 || c->bn != (M <= 8 ? 8 : 16) || c->bk != 256) return APT_ERR_UNSUPPORTED;
    if ((c->stages != 4 && c->stages != 8) || c->split_k < 1 || c->split_k > 32) return APT_ERR_UNSUPPORTED;
    if (c->cta_pair != 0 || c->cluster_n != 1) return APT_ERR_UNSUPPORTED;
    // 1-4-bit weight digits are u * 2^s (gemm_dec.cu): the unsigned sum must stay below 2^32
    if (kpad_of(K) * 255ll * 255ll >= (1ll << 32)) return APT_ERR_UNSUPPORTED;
    if ((N + c->bm - 1) / c->bm > APT_WS_TICKETS) return APT_ERR_UNSUPPORTED;  // one ticket per row tile
    return APT_OK;
  }
  if (c->kernel == APT_KERNEL_TC) {
    if (c->bm != 128 || c->bk != 128) return APT_ERR_UNSUPPORTED;
    if (c->bn != 16 && c->bn != 64 && c->bn != 128 && c->bn != 256) return APT_ERR_UNSUPPORTED;
    if (c->stages != apt::tc_stages(wbits, c->bn) || c->cta_pair != 0) return APT_ERR_UNSUPPORTED;
    if (c->cluster_n != 1 && c->cluster_n != 2 && c->cluster_n != 4) return APT_ERR_UNSUPPORTED;
    if (c->split_k < 1 || c->split_k > 8) return APT_ERR_UNSUPPORTED;
    if (c->split_k > 1 && (c->bn > 64 || c->cluster_n != 1)) return APT_ERR_UNSUPPORTED;
    if (c->cluster_n > 1 && c->bn < 128) return APT_ERR_UNSUPPORTED;
    if (c->bn == 16) {  // the up-front token slab holds at most 16 K steps per CTA
      if ((kw / 4 + c->split_k - 1) / c->split_k > 16) return APT_ERR_UNSUPPORTED;
    }
    return APT_OK;
  }
  return APT_ERR_UNSUPPORTED;
}

// the product kernels behind apt_gemm (defined after the C ABI)
apt_status launch_product(const apt_config& c, const apt_packed* W, const apt_packed* A, const apt::EpilogueArgs& e,
                          int32_t M, int32_t N, int32_t wbits, int32_t abits, void* workspace, cudaStream_t s);

}  // namespace

// ---------------------------------------------------------------------------------------------
// Autotuned configuration table (the paper's lookup table + Best Kernel Search +
// Approximate Matching, §5.2).  The table is filled offline by measuring every legal config
// (apt_enumerate_configs) per problem key (tools/tune.py) and loaded with apt_table_load.  Lookup: the
// exact key (M, N, K, wbits, abits), else the nearest key by d = |log2 M - log2 M'| + |log2 N - log2 N'| +
// |log2 K - log2 K'| among entries with the same (wbits, abits) — any (wbits, abits) if none — ties broken
// by the smaller measured time, then the smaller key.  A found config is used only if it is legal for the
// queried shape; otherwise the analytic rules decide.
namespace {
struct TableEntry {
  int32_t M, N, K, wbits, abits;
  apt_config cfg;
  double us;
};
std::mutex g_tab_mu;
std::vector<TableEntry> g_tab;

double key_dist(const TableEntry& e, int32_t M, int32_t N, int32_t K) {
  return std::fabs(std::log2((double)M) - std::log2((double)e.M)) + std::fabs(std::log2((double)N) - std::log2((double)e.N)) +
         std::fabs(std::log2((double)K) - std::log2((double)e.K));
}

bool key_less(const TableEntry& a, const TableEntry& b) {
  if (a.M != b.M) return a.M < b.M;
  if (a.N != b.N) return a.N < b.N;
  if (a.K != b.K) return a.K < b.K;
  if (a.wbits != b.wbits) return a.wbits < b.wbits;
  return a.abits < b.abits;
}

// token-count regime of a key: decode (M <= 16), small batch (M <= 64), prefill; rows of another regime
// are never matched (their kernels answer a different bound: HBM vs tensor)
int m_class(int32_t M) { return M <= 16 ? 0 : M <= 64 ? 1 : 2; }

// nearest entry (see above); false if no row of the query's M regime exists
bool table_find(int32_t M, int32_t N, int32_t K, int32_t wbits, int32_t abits, TableEntry* hit, double* dist) {
  std::lock_guard<std::mutex> lk(g_tab_mu);
  bool any = false, same_pq = false;
  for (const TableEntry& e : g_tab) {
    if (m_class(e.M) != m_class(M)) continue;
    any = true;
    same_pq |= (e.wbits == wbits && e.abits == abits);
  }
  if (!any) return false;
  const TableEntry* best = nullptr;
  double bd = 0;
  for (const TableEntry& e : g_tab) {
    if (m_class(e.M) != m_class(M)) continue;
    if (same_pq && (e.wbits != wbits || e.abits != abits)) continue;
    const double d = key_dist(e, M, N, K) + ((e.wbits == wbits && e.abits == abits) ? 0.0 : 0.0);
    bool better = !best || d < bd - 1e-12;
    if (best && std::fabs(d - bd) <= 1e-12) better = e.us < best->us || (e.us == best->us && key_less(e, *best));
    if (better) { best = &e; bd = d; }
  }
  *hit = *best;
  *dist = bd;
  return true;
}

bool table_select(int32_t M, int32_t N, int32_t K, int32_t wbits, int32_t abits, apt_config* out) {
  TableEntry e;
  double d;
  if (!table_find(M, N, K, wbits, abits, &e, &d)) return false;
  apt_config c = e.cfg;
  c.w_digit = wbits;  // digit widths follow the operand widths (full-width digits)
  c.a_digit = abits;
  if (c.kernel == APT_KERNEL_TC) c.stages = apt::tc_stages(wbits, c.bn);
  if (validate_config(&c, M, N, K, wbits, abits) != APT_OK) return false;
  *out = c;
  return true;
}

apt_status select_analytic(int32_t M, int32_t N, int32_t K, int32_t wbits, int32_t abits, apt_config* out);
}  // namespace


extern "C" {

int32_t apt_abi_version(void) { return APT_ABI_VERSION; }

const char* apt_status_string(apt_status s) {
  switch (s) {
    case APT_OK: return "APT_OK";
    case APT_ERR_INVALID_ARGUMENT: return "APT_ERR_INVALID_ARGUMENT";
    case APT_ERR_UNSUPPORTED: return "APT_ERR_UNSUPPORTED";
    case APT_ERR_WORKSPACE: return "APT_ERR_WORKSPACE";
    case APT_ERR_CUDA: return "APT_ERR_CUDA";
  }
  return "APT_ERR_UNKNOWN";
}

size_t apt_packed_plane_bytes(int32_t rows, int32_t k, int32_t bits, int32_t layout) {
  if (rows <= 0 || k <= 0 || bits < 1 || bits > 8) return 0;
  if (layout != APT_PACK_ROWS && layout != APT_PACK_TILED) return 0;
  const size_t prow = layout == APT_PACK_TILED ? (size_t)((rows + 127) / 128) * 128 : (size_t)rows;
  return (size_t)bits * prow * (size_t)(kpad_of(k) / 32) * 4u;
}

apt_status apt_pack_bipolar(const int8_t* codes, int32_t rows, int32_t k, int64_t ld, int32_t bits,
                            apt_encoding enc, apt_packed* out, int32_t* range_error, void* stream) {
  if (!codes || !out || !out->planes || !out->row_sum) return APT_ERR_INVALID_ARGUMENT;
  if (rows <= 0 || k <= 0 || ld < k || bits < 1 || bits > 8) return APT_ERR_INVALID_ARGUMENT;
  if (enc != APT_ENC_SIGNED && enc != APT_ENC_BIPOLAR) return APT_ERR_INVALID_ARGUMENT;
  if (enc == APT_ENC_BIPOLAR && bits > 7) return APT_ERR_INVALID_ARGUMENT;
  if (!aligned16(out->planes)) return APT_ERR_INVALID_ARGUMENT;
  if (out->layout != APT_PACK_ROWS && out->layout != APT_PACK_TILED) return APT_ERR_INVALID_ARGUMENT;
  out->rows = rows;
  out->k = k;
  out->k_words = (int32_t)(kpad_of(k) / 32);
  out->bits = bits;
  apt::PackArgs p;
  p.codes = codes;
  p.ld = ld;
  p.rows = rows;
  p.k = k;
  p.k_words = out->k_words;
  p.enc = (int32_t)enc;
  p.planes = out->planes;
  p.tiled = out->layout == APT_PACK_TILED ? 1 : 0;
  p.plane_stride = (int64_t)(p.tiled ? (rows + 127) / 128 * 128 : rows) * out->k_words;
  p.row_sum = out->row_sum;
  p.range_error = range_error;
  p.digits = out->digits;
  if (out->digits && !aligned16(out->digits)) return APT_ERR_INVALID_ARGUMENT;
  cudaError_t err = apt::launch_pack(p, bits, reinterpret_cast<cudaStream_t>(stream));
  return err == cudaSuccess ? APT_OK : APT_ERR_CUDA;
}

apt_status apt_quantize_pack(const uint16_t* x, int32_t rows, int32_t k, int64_t ld, int32_t bits,
                             apt_packed* out, float* scale, void* stream) {
  if (!x || !out || !out->planes || !out->row_sum || !scale) return APT_ERR_INVALID_ARGUMENT;
  if (rows <= 0 || k <= 0 || ld < k || bits < 2 || bits > 8) return APT_ERR_INVALID_ARGUMENT;
  if (!aligned16(out->planes)) return APT_ERR_INVALID_ARGUMENT;
  if (out->digits && !aligned16(out->digits)) return APT_ERR_INVALID_ARGUMENT;
  if (out->layout != APT_PACK_ROWS && out->layout != APT_PACK_TILED) return APT_ERR_INVALID_ARGUMENT;
  out->rows = rows;
  out->k = k;
  out->k_words = (int32_t)(kpad_of(k) / 32);
  out->bits = bits;
  apt::PackArgs p;
  p.codes = nullptr;
  p.ld = ld;
  p.rows = rows;
  p.k = k;
  p.k_words = out->k_words;
  p.enc = APT_ENC_SIGNED;
  p.planes = out->planes;
  p.tiled = out->layout == APT_PACK_TILED ? 1 : 0;
  p.plane_stride = (int64_t)(p.tiled ? (rows + 127) / 128 * 128 : rows) * out->k_words;
  p.row_sum = out->row_sum;
  p.range_error = nullptr;
  p.digits = out->digits;
  cudaError_t err = apt::launch_quant_pack(p, x, scale, bits, reinterpret_cast<cudaStream_t>(stream));
  return err == cudaSuccess ? APT_OK : APT_ERR_CUDA;
}

apt_status apt_pack_grouped(int32_t count, const apt_pack_problem* problems, void* stream) {
  if (count < 1 || count > APT_GROUP_MAX || count > apt::kPackGroupMax || !problems) return APT_ERR_INVALID_ARGUMENT;
  static apt::PackGroupArgs ga_zero;  // zero-initialised template (the struct is ~10 KB)
  apt::PackGroupArgs ga = ga_zero;
  ga.count = count;
  int ctas = 0, threads = 32;
  for (int i = 0; i < count; ++i) {
    const apt_pack_problem& P = problems[i];
    apt_packed* out = P.out;
    const bool quant = P.quantize != 0;
    if (!P.src || !out || !out->planes || !out->row_sum || !out->digits) return APT_ERR_INVALID_ARGUMENT;
    if (P.rows <= 0 || P.rows > APT_PACK_GROUP_MAX_ROWS || P.k <= 0 || P.ld < P.k) return APT_ERR_INVALID_ARGUMENT;
    if (P.bits < (quant ? 2 : 1) || P.bits > 8 || (quant && !P.scale)) return APT_ERR_INVALID_ARGUMENT;
    if (!aligned16(out->planes) || !aligned16(out->digits) || out->layout != APT_PACK_ROWS) return APT_ERR_INVALID_ARGUMENT;
    out->rows = P.rows;
    out->k = P.k;
    out->k_words = (int32_t)(kpad_of(P.k) / 32);
    out->bits = P.bits;
    apt::PackArgs& p = ga.p[i];
    p.codes = quant ? nullptr : reinterpret_cast<const int8_t*>(P.src);
    p.ld = P.ld;
    p.rows = P.rows;
    p.k = P.k;
    p.k_words = out->k_words;
    p.enc = APT_ENC_SIGNED;
    p.planes = out->planes;
    p.tiled = 0;
    p.plane_stride = (int64_t)P.rows * out->k_words;
    p.row_sum = out->row_sum;
    p.range_error = quant ? nullptr : P.range_error;
    p.digits = out->digits;
    ga.x[i] = quant ? P.src : nullptr;
    ga.scale[i] = quant ? P.scale : nullptr;
    ga.bits[i] = P.bits;
    ga.rows_per_cta[i] = apt::pack_group_rows_per_cta(p);
    ctas += (P.rows + ga.rows_per_cta[i] - 1) / ga.rows_per_cta[i];
    ga.cta_end[i] = ctas;
    threads = std::max(threads, apt::pack_group_threads(p));
  }
  cudaError_t err = apt::launch_pack_grouped(ga, ctas, threads, reinterpret_cast<cudaStream_t>(stream));
  return err == cudaSuccess ? APT_OK : APT_ERR_CUDA;
}

apt_status apt_select_config(int32_t M, int32_t N, int32_t K, int32_t wbits, int32_t abits, apt_config* out) {
  if (!out || M <= 0 || N <= 0 || K <= 0 || wbits < 1 || wbits > 8 || abits < 1 || abits > 8)
    return APT_ERR_INVALID_ARGUMENT;
  if (!bound_ok(K, wbits, abits)) return APT_ERR_UNSUPPORTED;
  // the autotuned table first (NEXT-3, §5.2): exact key or nearest key, if legal for the shape
  if (table_select(M, N, K, wbits, abits, out)) return APT_OK;
  return select_analytic(M, N, K, wbits, abits, out);
}

}  // extern "C"

namespace {
apt_status select_analytic(int32_t M, int32_t N, int32_t K, int32_t wbits, int32_t abits, apt_config* out) {
  std::memset(out, 0, sizeof(*out));
  const int kNumSMs = device_sms();
  const int kw = (int)(kpad_of(K) / 32);
  out->w_digit = wbits;
  out->a_digit = abits;
  out->kernel = APT_KERNEL_TC;
  out->bm = 128;
  out->bk = 128;
  out->cta_pair = 0;
  if (M > 64) {
    // token-rich: 128 weight rows x 256 tokens per tile, no cluster.  The weight rebuild (converter
    // warps, integer ALU) is paid once per 256 tokens instead of 128 (profiles/r1_prefill_bn_sweep.txt:
    // 1.0-1.4x faster than 2 x (128 x 128) CTAs per SM with a 4-CTA token multicast).  The persistent
    // tile (one CTA per SM walking the tiles, epilogue overlapped with the next tile's MMAs) where its
    // s32 accumulation of scaled digits is exact: 0.95-1.25x the one-tile-per-CTA kernel on the
    // prefill, Llama-3-70B and sweep shapes (profiles/r2_pf256_ab.jsonl)
    out->bn = 256;
    out->split_k = 1;
    out->cluster_n = 1;
    if (kpad_of(K) * 255ll * 255ll < (1ll << 31)) {
      out->kernel = APT_KERNEL_PF;
      out->stages = 3;
      return APT_OK;
    }
  } else if (M <= 2) {
    // one or two tokens: the SIMT dp4a GEMV (SURVEY §8 a9 "pick by measurement"; 1.2-2.2x faster
    // than the tensor-core decode tile on every Llama-2-7B decode linear at M = 1, 2).
    // 16 warps per 32-row CTA when the row tiles do not fill the SMs, else 8 warps, 3 CTAs per SM.
    out->kernel = APT_KERNEL_GEMV;
    out->bm = 32;
    out->bn = M;
    out->split_k = ceil_div(N, 32) <= kNumSMs ? 16 : 8;
    out->cluster_n = 1;
    out->stages = 1;
    return APT_OK;
  } else if (M <= 8 && K <= 4096) {
    // up to 8 tokens, K <= 4096: the mma.sync skinny GEMM fed from registers (1.07-1.48x faster than
    // the tcgen05 tile at M = 8 on 4096x4096 and 11008x4096; slower at K = 11008 and at M = 16,
    // profiles/r1_skinny_vs_tc.txt).  8 warps per 16-row CTA while the row tiles fit twice on the
    // SMs, else 4.
    out->kernel = APT_KERNEL_SKINNY;
    out->bm = 16;
    out->bn = 8;
    out->bk = 256;
    out->split_k = ceil_div(N, 16) <= 2 * kNumSMs ? 8 : 4;
    out->cluster_n = 1;
    out->stages = 1;
    return APT_OK;
  } else {
    // decode: 16 (or 64) tokens per tile, K split over a cluster of up to 8 CTAs so that about two
    // CTAs per SM stream weights
    out->bn = M <= 16 ? 16 : 64;
    out->cluster_n = 1;
    const int64_t tiles = (int64_t)ceil_div(N, 128) * ceil_div(M, out->bn);
    const int steps = kw / 4;  // 128-element K steps
    int split = (int)((2 * kNumSMs + tiles / 2) / tiles);
    if (split > 8) split = 8;
    if (split > steps) split = steps;
    if (split < 1) split = 1;
    if (out->bn == 16) {  // at most 16 K steps per CTA, else the ring-buffered 64-token tile
      while (split < 8 && (steps + split - 1) / split > 16) ++split;
      if ((steps + split - 1) / split > 16) out->bn = 64;
    }
    out->split_k = split;
  }
  out->stages = apt::tc_stages(wbits, out->bn);
  return APT_OK;
}
}  // namespace

extern "C" {

// workspace areas (include/apt.h apt_gemm_workspace_bytes), offsets fixed per (cfg, M, N, K):
// [split-K tickets, APT_WS_TICKETS uint32, the same place for every call][token digit expansion]
// [DEC split-K partials]
static size_t ws_expand_bytes(int32_t M, int32_t K) { return apt::tc_workspace_bytes(M, (int)(kpad_of(K) / 32)); }
static size_t ws_dec_off(int32_t M, int32_t K) { return APT_WS_TICKET_BYTES + (ws_expand_bytes(M, K) + 15) / 16 * 16; }
static size_t ws_dec_bytes(const apt_config* cfg, int32_t N) {
  return cfg->kernel == APT_KERNEL_DEC ? apt::dec_workspace_bytes(N, cfg->split_k) : 0;
}

size_t apt_gemm_workspace_bytes(const apt_config* cfg, int32_t M, int32_t N, int32_t K) {
  if (!cfg || M <= 0 || N <= 0 || K <= 0) return 0;
  return ws_dec_off(M, K) + ws_dec_bytes(cfg, N);
}

size_t apt_gemm_zp_workspace_bytes(const apt_config* cfg, int32_t M, int32_t N, int32_t K) {
  if (!cfg || M <= 0 || N <= 0 || K <= 0) return 0;
  return (apt_gemm_workspace_bytes(cfg, M, N, K) + 15) / 16 * 16 + (size_t)M * (size_t)N * 4u;
}

static apt_status grp_gemm(int32_t M, int32_t N, int32_t K, int32_t wbits, int32_t abits, const apt_packed* W,
                           const apt_packed* A, const apt_scales* scales, apt_out_kind kind, apt_layout layout,
                           void* out, int64_t ldo, void* workspace, size_t ws_bytes, cudaStream_t s);

apt_status apt_gemm(int32_t M, int32_t N, int32_t K, int32_t wbits, int32_t abits, const apt_packed* W,
                    const apt_packed* A, const apt_scales* scales, apt_out_kind kind, apt_layout layout,
                    void* out, int64_t ldo, const apt_config* cfg, void* workspace, size_t ws_bytes,
                    void* stream) {
  if (M <= 0 || N <= 0 || K <= 0 || wbits < 1 || wbits > 8 || abits < 1 || abits > 8 || !out)
    return APT_ERR_INVALID_ARGUMENT;
  apt_status st = validate_packed(W, N, K, wbits);
  if (st != APT_OK) return st;
  // a packed matrix with a digit view is an activation operand (its pack releases dependents early,
  // include/apt.h "General contract"); it may not serve as the weight operand
  if (W->digits) return APT_ERR_INVALID_ARGUMENT;
  st = validate_packed(A, M, K, abits);
  if (st != APT_OK) return st;
  if (kind != APT_OUT_I32_SIGNED && kind != APT_OUT_I32_BIPOLAR && kind != APT_OUT_F16_SCALED)
    return APT_ERR_INVALID_ARGUMENT;
  if (layout != APT_LAYOUT_ROW && layout != APT_LAYOUT_COL) return APT_ERR_INVALID_ARGUMENT;
  if (layout == APT_LAYOUT_ROW ? ldo < N : ldo < M) return APT_ERR_INVALID_ARGUMENT;
  if (kind == APT_OUT_F16_SCALED && (!scales || (!scales->w_scale && scales->group_size == 0)))
    return APT_ERR_INVALID_ARGUMENT;
  if (!bound_ok(K, wbits, abits)) return APT_ERR_UNSUPPORTED;
  apt_config c;
  if (cfg) {
    c = *cfg;
  } else {
    st = apt_select_config(M, N, K, wbits, abits, &c);
    if (st != APT_OK) return st;
  }
  st = validate_config(&c, M, N, K, wbits, abits);
  if (st != APT_OK) return st;
  const size_t dec_ws = ws_dec_bytes(&c, N);
  const bool expand = !A->digits || c.mma_kind == APT_MMA_MXF4;  // the token expansion area is used
  const size_t need0 = dec_ws ? ws_dec_off(M, K) + dec_ws : (expand ? APT_WS_TICKET_BYTES + ws_expand_bytes(M, K) : 0);
  // zero points (NEXT-2): exact int32 Y into the workspace after the digit-expansion area, then the
  // elementwise zero-point epilogue
  const bool zp = kind == APT_OUT_F16_SCALED && (scales->w_zero || scales->a_zero);
  // group-wise scales (NEXT-2): the grouped kernel's signed-digit path, M in chunks of 16 tokens
  if (scales && scales->group_size != 0) {
    if (kind != APT_OUT_F16_SCALED || scales->group_size != 128 || !scales->w_gscale || zp) return APT_ERR_INVALID_ARGUMENT;
    if (W->layout != APT_PACK_TILED || !A->digits || A->layout != APT_PACK_ROWS) return APT_ERR_UNSUPPORTED;
    if (!workspace || ws_bytes < apt_gemm_grouped_workspace_bytes(1) || !aligned16(workspace)) return APT_ERR_WORKSPACE;
    return grp_gemm(M, N, K, wbits, abits, W, A, scales, kind, layout, out, ldo, workspace, ws_bytes,
                    reinterpret_cast<cudaStream_t>(stream));
  }
  // zero points at decode token counts: fused into the grouped kernel's epilogue (one launch, no int32 Y
  // round trip) when the operands and the workspace allow it and no config was forced
  if (zp && !cfg && M <= 16 && W->layout == APT_PACK_TILED && A->digits && A->layout == APT_PACK_ROWS && workspace &&
      ws_bytes >= apt_gemm_grouped_workspace_bytes(1) && aligned16(workspace))
    return grp_gemm(M, N, K, wbits, abits, W, A, scales, kind, layout, out, ldo, workspace, ws_bytes,
                    reinterpret_cast<cudaStream_t>(stream));
  // (never inside the ticket area, which every call leaves zero for the next one)
  const size_t y_off = (std::max<size_t>(need0, APT_WS_TICKET_BYTES) + 15) / 16 * 16;
  const size_t need = zp ? y_off + (size_t)M * (size_t)N * 4u : need0;
  if (need > 0 && (!workspace || ws_bytes < need || !aligned16(workspace))) return APT_ERR_WORKSPACE;
  if (A->digits && !aligned16(A->digits)) return APT_ERR_INVALID_ARGUMENT;

  apt::EpilogueArgs e;
  e.w_rowsum = W->row_sum;
  e.a_rowsum = A->row_sum;
  e.w_scale = scales ? scales->w_scale : nullptr;
  e.a_scale = scales ? scales->a_scale : nullptr;
  e.out = out;
  e.ldo = ldo;
  e.kind = (int32_t)kind;
  e.layout = (int32_t)layout;
  e.M = M;
  e.N = N;
  e.K = K;
  e.kpad = (int32_t)kpad_of(K);
  e.h_w = 1 << (wbits - 1);
  e.h_a = 1 << (abits - 1);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (zp) {
    e.out = reinterpret_cast<uint8_t*>(workspace) + y_off;
    e.ldo = N;
    e.kind = APT_OUT_I32_SIGNED;
    e.layout = APT_LAYOUT_ROW;
  }
  st = launch_product(c, W, A, e, M, N, wbits, abits, workspace, s);
  if (st != APT_OK || !zp) return st;
  apt::ZpArgs z;
  z.y = reinterpret_cast<const int32_t*>(reinterpret_cast<uint8_t*>(workspace) + y_off);
  z.w_rowsum = W->row_sum;
  z.a_rowsum = A->row_sum;
  z.w_scale = scales->w_scale;
  z.a_scale = scales->a_scale;
  z.w_zero = scales->w_zero;
  z.a_zero = scales->a_zero;
  z.out = reinterpret_cast<__half*>(out);
  z.ldo = ldo;
  z.layout = (int32_t)layout;
  z.M = M;
  z.N = N;
  z.K = K;
  return apt::launch_zp_epilogue(z, s) == cudaSuccess ? APT_OK : APT_ERR_CUDA;
}


apt_status apt_table_load(const char* path) {
  if (!path) return APT_ERR_INVALID_ARGUMENT;
  FILE* f = std::fopen(path, "r");
  if (!f) return APT_ERR_INVALID_ARGUMENT;
  std::vector<TableEntry> rows;
  char line[512];
  bool ok = true;
  while (std::fgets(line, sizeof(line), f)) {
    const char* q = line;
    while (*q == ' ' || *q == '\t') ++q;
    if (*q == '#' || *q == '\n' || *q == '\0') continue;
    TableEntry e;
    std::memset(&e, 0, sizeof(e));
    apt_config& c = e.cfg;
    const int n = std::sscanf(q, "%d %d %d %d %d %d %d %d %d %d %d %d %d %d %d %d %lf", &e.M, &e.N, &e.K, &e.wbits,
                              &e.abits, &c.kernel, &c.w_digit, &c.a_digit, &c.bm, &c.bn, &c.bk, &c.stages, &c.split_k,
                              &c.cta_pair, &c.cluster_n, &c.mma_kind, &e.us);
    if (n != 17 || e.M <= 0 || e.N <= 0 || e.K <= 0 || e.wbits < 1 || e.wbits > 8 || e.abits < 1 || e.abits > 8) {
      ok = false;
      break;
    }
    rows.push_back(e);
  }
  std::fclose(f);
  if (!ok) return APT_ERR_INVALID_ARGUMENT;
  std::lock_guard<std::mutex> lk(g_tab_mu);
  // a later row for the same key replaces an earlier one
  for (const TableEntry& e : rows) {
    bool replaced = false;
    for (TableEntry& o : g_tab)
      if (o.M == e.M && o.N == e.N && o.K == e.K && o.wbits == e.wbits && o.abits == e.abits) { o = e; replaced = true; }
    if (!replaced) g_tab.push_back(e);
  }
  return APT_OK;
}

void apt_table_clear(void) {
  std::lock_guard<std::mutex> lk(g_tab_mu);
  g_tab.clear();
}

int32_t apt_table_size(void) {
  std::lock_guard<std::mutex> lk(g_tab_mu);
  return (int32_t)g_tab.size();
}

apt_status apt_table_lookup(int32_t M, int32_t N, int32_t K, int32_t wbits, int32_t abits, apt_config* out,
                            double* distance) {
  if (!out || M <= 0 || N <= 0 || K <= 0 || wbits < 1 || wbits > 8 || abits < 1 || abits > 8)
    return APT_ERR_INVALID_ARGUMENT;
  TableEntry e;
  double d;
  if (!table_find(M, N, K, wbits, abits, &e, &d)) return APT_ERR_UNSUPPORTED;
  *out = e.cfg;
  if (distance) *distance = d;
  return APT_OK;
}

int32_t apt_enumerate_configs(int32_t M, int32_t N, int32_t K, int32_t wbits, int32_t abits, apt_config* out,
                              int32_t cap) {
  if (M <= 0 || N <= 0 || K <= 0 || wbits < 1 || wbits > 8 || abits < 1 || abits > 8) return 0;
  if (!bound_ok(K, wbits, abits)) return 0;
  std::vector<apt_config> v;
  auto add = [&](int kernel, int bm, int bn, int bk, int stages, int split, int cn) {
    apt_config c;
    std::memset(&c, 0, sizeof(c));
    c.kernel = kernel; c.w_digit = wbits; c.a_digit = abits; c.bm = bm; c.bn = bn; c.bk = bk; c.stages = stages;
    c.split_k = split; c.cta_pair = 0; c.cluster_n = cn; c.mma_kind = APT_MMA_I8;
    if (validate_config(&c, M, N, K, wbits, abits) == APT_OK) v.push_back(c);
  };
  for (int sp : {8, 16}) add(APT_KERNEL_GEMV, 32, M, 128, 1, sp, 1);
  for (int bn : {8, 16})
    for (int w : {4, 8, 16}) add(APT_KERNEL_SKINNY, 16, bn, 256, 1, w, 1);
  for (int w : {4, 8})
    for (int sp : {1, 2, 3, 4, 6, 8}) add(APT_KERNEL_DEC, 32, M <= 8 ? 8 : 16, 256, w, sp, 1);
  for (int bn : {16, 64, 128, 256})
    for (int cn : {1, 2, 4})
      for (int sp = 1; sp <= 8; ++sp) add(APT_KERNEL_TC, 128, bn, 128, apt::tc_stages(wbits, bn), sp, cn);
  for (int bn : {128, 192, 256})  // the persistent tile
    for (int mk : {APT_MMA_I8, APT_MMA_MXF4}) {
      apt_config c;
      std::memset(&c, 0, sizeof(c));
      c.kernel = APT_KERNEL_PF; c.w_digit = wbits; c.a_digit = abits; c.bm = 128; c.bn = bn; c.bk = 128;
      c.stages = bn == 128 ? 6 : bn == 192 ? 4 : 3; c.split_k = 1; c.cluster_n = 1; c.mma_kind = mk;
      if (validate_config(&c, M, N, K, wbits, abits) == APT_OK) v.push_back(c);
    }
  for (int bn : {128, 256}) {  // kind::mxf4 (wbits, abits <= 3)
    apt_config c;
    std::memset(&c, 0, sizeof(c));
    c.kernel = APT_KERNEL_TC; c.w_digit = wbits; c.a_digit = abits; c.bm = 128; c.bn = bn; c.bk = 128;
    c.stages = apt::tc_stages(wbits, bn); c.split_k = 1; c.cluster_n = 1; c.mma_kind = APT_MMA_MXF4;
    if (validate_config(&c, M, N, K, wbits, abits) == APT_OK) v.push_back(c);
  }
  const int n = (int)v.size();
  for (int i = 0; i < n && i < cap && out; ++i) out[i] = v[i];
  return n;
}

// ---- grouped decode GEMM (include/apt.h apt_gemm_grouped, gemm_grp.cu)
static int grp_max_workers() { return device_sms() * 4; }  // one worker per CTA, at most 4 CTAs per SM

size_t apt_gemm_grouped_workspace_bytes(int32_t count) {
  if (count < 1 || count > APT_GROUP_MAX) return 0;
  // tickets, then int32 partials [worker][2][4 warps][16 x 32]
  return APT_WS_TICKET_BYTES + (size_t)grp_max_workers() * 2u * 4u * 512u * 4u;
}

// The grouped launch behind apt_gemm_grouped and apt_gemm's group-scale / fused zero-point routes.
// a_gs_ld[i] (nullable): leading dimension of problem i's a_gscale ([Kpad/128][a_gs_ld]); default its M.
static apt_status grp_run(int32_t count, const apt_gemm_problem* problems, const int64_t* a_gs_ld, void* workspace,
                          size_t ws_bytes, cudaStream_t stream) {
  if (count < 1 || count > APT_GROUP_MAX || count > apt::kGrpMax || !problems) return APT_ERR_INVALID_ARGUMENT;
  static_assert(APT_GROUP_MAX <= apt::kGrpMax, "group size");
  static apt::GrpArgs ga_zero;  // zero-initialised template (the struct is ~19 KB)
  apt::GrpArgs ga = ga_zero;
  int64_t blocks = 0, cost = 0;
  int wbmax = 1, cmax = 1;
  const bool gs = problems[0].scales.group_size != 0;
  for (int i = 0; i < count; ++i) {
    const apt_gemm_problem& P = problems[i];
    // group-wise scales (NEXT-2): fp16 output, groups of 128, the weights' [Kpad/128][N] scales required,
    // no zero points, and all problems of a launch alike
    if ((P.scales.group_size != 0) != gs) return APT_ERR_INVALID_ARGUMENT;
    if (gs && (P.scales.group_size != 128 || P.kind != APT_OUT_F16_SCALED || !P.scales.w_gscale ||
               P.scales.w_zero || P.scales.a_zero))
      return APT_ERR_INVALID_ARGUMENT;
    const int32_t M = P.M, N = P.N, K = P.K;
    if (M <= 0 || M > 16 || N <= 0 || K <= 0 || P.wbits < 1 || P.wbits > 8 || P.abits < 1 || P.abits > 8 || !P.out)
      return APT_ERR_INVALID_ARGUMENT;
    if (validate_packed(&P.W, N, K, P.wbits) != APT_OK || P.W.layout != APT_PACK_TILED || P.W.digits)
      return APT_ERR_INVALID_ARGUMENT;
    if (validate_packed(&P.A, M, K, P.abits) != APT_OK || !P.A.digits || !aligned16(P.A.digits))
      return APT_ERR_INVALID_ARGUMENT;
    if (P.kind != APT_OUT_I32_SIGNED && P.kind != APT_OUT_I32_BIPOLAR && P.kind != APT_OUT_F16_SCALED)
      return APT_ERR_INVALID_ARGUMENT;
    if (P.layout != APT_LAYOUT_ROW && P.layout != APT_LAYOUT_COL) return APT_ERR_INVALID_ARGUMENT;
    if (P.layout == APT_LAYOUT_ROW ? P.ldo < N : P.ldo < M) return APT_ERR_INVALID_ARGUMENT;
    if (P.kind == APT_OUT_F16_SCALED && !gs && !P.scales.w_scale) return APT_ERR_INVALID_ARGUMENT;
    if (!bound_ok(K, P.wbits, P.abits)) return APT_ERR_UNSUPPORTED;
    if (kpad_of(K) * 255ll * 255ll >= (1ll << 32)) return APT_ERR_UNSUPPORTED;  // u * 2^s digits (gemm_dec.cu)
    apt::GrpProblem& q = ga.p[i];
    {
      // token digit view [M][Kpad] u8, 128-byte swizzle
      apt::PFN_encodeTiled_t enc = apt::tensor_map_encoder();
      if (!enc) return APT_ERR_CUDA;
      const cuuint64_t kp = (cuuint64_t)P.A.k_words * 32;
      // [Kpad / 128 chunks][M rows][128 bytes]; a box = the 2 chunks of a 256-element block x 8 / 16 rows
      cuuint64_t dims[3] = {128, (cuuint64_t)M, kp / 128};
      cuuint64_t strides[2] = {kp, 128};
      cuuint32_t box[3] = {128, M <= 8 ? 8u : 16u, 2};
      cuuint32_t es[3] = {1, 1, 1};
      if (enc(&q.tok, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, P.A.digits, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return APT_ERR_INVALID_ARGUMENT;
    }
    q.wp = P.W.planes;
    q.w_pstride = (int64_t)((N + 127) / 128 * 128) * P.W.k_words;
    q.adig = P.A.digits;
    apt::EpilogueArgs& e = q.e;
    e.w_rowsum = P.W.row_sum;
    e.a_rowsum = P.A.row_sum;
    e.w_scale = P.scales.w_scale;
    e.a_scale = P.scales.a_scale;
    e.out = P.out;
    e.ldo = P.ldo;
    e.kind = P.kind;
    e.layout = P.layout;
    e.M = M;
    e.N = N;
    e.K = K;
    e.kpad = (int32_t)kpad_of(K);
    e.h_w = 1 << (P.wbits - 1);
    e.h_a = 1 << (P.abits - 1);
    if (P.n_peers < 0 || P.n_peers > APT_MAX_PEERS) return APT_ERR_INVALID_ARGUMENT;
    q.n_peers = P.n_peers;
    for (int j = 0; j < P.n_peers; ++j) {
      if (!P.out_peers[j]) return APT_ERR_INVALID_ARGUMENT;
      q.peers[j] = P.out_peers[j];
    }
    q.w_zero = P.kind == APT_OUT_F16_SCALED ? P.scales.w_zero : nullptr;
    q.a_zero = P.kind == APT_OUT_F16_SCALED ? P.scales.a_zero : nullptr;
    q.w_gs = gs ? P.scales.w_gscale : nullptr;
    q.a_gs = gs ? P.scales.a_gscale : nullptr;
    q.a_gs_ld = a_gs_ld ? a_gs_ld[i] : M;
    q.k_words = P.W.k_words;
    q.nb = P.W.k_words / 8;  // units of 128 rows x 256 K per 128-row tile
    q.tiles = (N + 127) / 128;
    q.wbits = P.wbits;
    // unit cost = 4 KB per weight plane + a fixed share for the consumers' per-unit work (token tile,
    // MMAs, barriers), twice as large at M > 8 (the two-token-tile orientation: twice the MMAs and token
    // bytes).  Coefficients fitted on the bench's 36-problem launch (tools/grp_bench.py): 4 / 2 per plane
    // + 16 / 8 ran it in 120 us, 4 + 2 (bytes only) in 150 us, 4 + 8 / 2 in 132 us
#ifndef APT_GRP_CW
#define APT_GRP_CW 4
#define APT_GRP_CM16 16
#define APT_GRP_CM8 8
#endif
    q.cost = APT_GRP_CW * P.wbits + (M > 8 ? APT_GRP_CM16 : APT_GRP_CM8);
    q.blk0 = blocks;
    q.cost0 = cost;
    blocks += (int64_t)q.tiles * q.nb;
    cost += (int64_t)q.tiles * q.nb * q.cost;
    wbmax = std::max(wbmax, P.wbits);
    cmax = std::max(cmax, q.cost);
  }
  // every worker owns at least one block when workers * max cost <= total cost (gemm_grp.cu grp_owner)
#ifdef APT_GRP_CPS
  const int cps = APT_GRP_CPS;
#else
  const int cps = apt::grp_ctas_per_sm(wbmax, gs);
#endif
  int64_t workers = std::min<int64_t>((int64_t)device_sms() * cps, cost / cmax);
  workers = std::max<int64_t>(workers, 1);
  if (workers > grp_max_workers() || workers * 4 > APT_WS_TICKETS) return APT_ERR_UNSUPPORTED;  // a ticket per warp slice
  if (!workspace || ws_bytes < apt_gemm_grouped_workspace_bytes(count) || !aligned16(workspace))
    return APT_ERR_WORKSPACE;
  ga.count = count;
  ga.workers = (int32_t)workers;
  ga.total_blocks = blocks;
  ga.total_cost = cost;
  // every worker's first block: the first block whose owner (midpoint rule, gemm_grp.cu grp_owner) is that
  // worker; owners are non-decreasing along the blocks and take every value (workers * max cost <= total)
  if (workers > apt::kGrpMaxWorkers || blocks >= (1ll << 32)) return APT_ERR_UNSUPPORTED;
  {
    int next = 0;
    for (int i = 0; i < count && next < workers; ++i) {
      apt::GrpProblem& q = ga.p[i];
      const int64_t nblk = (int64_t)q.tiles * q.nb;
      auto owner = [&](int64_t b) { return (int)((2 * q.cost0 + (2 * b + 1) * (int64_t)q.cost) * workers / (2 * cost)); };
      q.w_hi = owner(nblk - 1);
      while (next < workers && next <= q.w_hi) {
        // smallest b with owner(b) >= next (binary search over the problem's blocks)
        int64_t lo = 0, hi = nblk - 1;
        while (lo < hi) {
          const int64_t mid = (lo + hi) / 2;
          if (owner(mid) >= next) hi = mid; else lo = mid + 1;
        }
        ga.wstart[next++] = (uint32_t)(q.blk0 + lo);
      }
    }
    for (; next <= workers; ++next) ga.wstart[next] = (uint32_t)blocks;
  }
  ga.tickets = reinterpret_cast<uint32_t*>(workspace);
  ga.partials = reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(workspace) + APT_WS_TICKET_BYTES);
  bool peers = false;
  for (int i = 0; i < count; ++i) peers |= ga.p[i].n_peers > 0;
  cudaError_t err = apt::launch_gemm_grp(ga, wbmax, (int)workers, gs, peers, stream);
  return err == cudaSuccess ? APT_OK : APT_ERR_CUDA;
}

apt_status apt_gemm_grouped(int32_t count, const apt_gemm_problem* problems, void* workspace, size_t ws_bytes,
                            void* stream) {
  return grp_run(count, problems, nullptr, workspace, ws_bytes, reinterpret_cast<cudaStream_t>(stream));
}

// apt_gemm through the grouped kernel: the M tokens in chunks of at most 16 rows, each chunk one problem
// (A, its row sums, scales, zero points and group scales offset to the chunk; the output offset to its
// rows / columns), up to APT_GROUP_MAX chunks per launch
static apt_status grp_gemm(int32_t M, int32_t N, int32_t K, int32_t wbits, int32_t abits, const apt_packed* W,
                           const apt_packed* A, const apt_scales* scales, apt_out_kind kind, apt_layout layout,
                           void* out, int64_t ldo, void* workspace, size_t ws_bytes, cudaStream_t s) {
  const int esz = kind == APT_OUT_F16_SCALED ? 2 : 4;
  const int64_t kp = kpad_of(K);
  apt_gemm_problem pr[APT_GROUP_MAX];
  int64_t ld[APT_GROUP_MAX];
  int n = 0;
  for (int32_t m0 = 0; m0 < M; m0 += 16) {
    apt_gemm_problem& P = pr[n];
    std::memset(&P, 0, sizeof(P));
    const int32_t mc = std::min(16, M - m0);
    P.M = mc;
    P.N = N;
    P.K = K;
    P.wbits = wbits;
    P.abits = abits;
    P.W = *W;
    P.A = *A;
    P.A.rows = mc;
    P.A.row_sum = A->row_sum + m0;
    P.A.digits = A->digits + (int64_t)m0 * kp;
    if (scales) {
      P.scales = *scales;
      if (scales->a_scale) P.scales.a_scale = scales->a_scale + m0;
      if (scales->a_zero) P.scales.a_zero = scales->a_zero + m0;
      if (scales->a_gscale) P.scales.a_gscale = scales->a_gscale + m0;
    }
    P.kind = kind;
    P.layout = layout;
    P.out = reinterpret_cast<uint8_t*>(out) + (layout == APT_LAYOUT_ROW ? (int64_t)m0 * ldo : (int64_t)m0) * esz;
    P.ldo = ldo;
    ld[n] = M;
    if (++n == APT_GROUP_MAX || m0 + 16 >= M) {
      const apt_status st = grp_run(n, pr, ld, workspace, ws_bytes, s);
      if (st != APT_OK) return st;
      n = 0;
    }
  }
  return APT_OK;
}

apt_status apt_recombine_plane_products(const int32_t* parts, int32_t abits, int32_t wbits, int64_t part_stride,
                                        int64_t count, int32_t* out, void* stream) {
  if (!parts || !out || abits < 1 || abits > 8 || wbits < 1 || wbits > 8 || count <= 0 || part_stride < count)
    return APT_ERR_INVALID_ARGUMENT;
  return apt::launch_recombine_planes(parts, abits, wbits, part_stride, count, out,
                                      reinterpret_cast<cudaStream_t>(stream)) == cudaSuccess
             ? APT_OK
             : APT_ERR_CUDA;
}
}  // extern "C"

namespace {
apt_status launch_product(const apt_config& c, const apt_packed* W, const apt_packed* A, const apt::EpilogueArgs& e,
                          int32_t M, int32_t N, int32_t wbits, int32_t abits, void* workspace, cudaStream_t s) {
  // the TC kernel reads the activation operand as kernel-order u8 digits: the packed view, or
  // expanded now into the workspace
  if (c.kernel == APT_KERNEL_PF) {
    apt::TcArgs p;
    p.wp = W->planes;
    p.w_tiled = W->layout == APT_PACK_TILED ? 1 : 0;
    p.w_pstride = (int64_t)(p.w_tiled ? (N + 127) / 128 * 128 : N) * W->k_words;
    p.k_words = W->k_words;
    p.e = e;
    const bool mx = c.mma_kind == APT_MMA_MXF4;
    if (mx || !A->digits) {
      if (A->layout != APT_PACK_ROWS) return APT_ERR_UNSUPPORTED;
      uint8_t* xp = reinterpret_cast<uint8_t*>(workspace) + APT_WS_TICKET_BYTES;
      cudaError_t err = mx ? apt::launch_expand_tokens_mx(A->planes, (int64_t)M * A->k_words, M, A->k_words, abits, xp, s)
                           : apt::launch_expand_tokens(A->planes, (int64_t)M * A->k_words, M, A->k_words, abits, xp, s);
      if (err != cudaSuccess) return APT_ERR_CUDA;
      p.adig = xp;
    } else {
      p.adig = A->digits;
    }
    if (mx) {
      p.e.h_w = 0;
      p.e.h_a = 0;
    }
    return apt::launch_gemm_pf(p, wbits, mx ? 1 : 0, c.bn, s) == cudaSuccess ? APT_OK : APT_ERR_CUDA;
  }
  if (c.mma_kind == APT_MMA_MXF4) {
    // kind::mxf4: tokens as signed e2m1 nibbles, expanded from the activation planes into the workspace;
    // the f32 accumulator is already the signed product (no offset-digit correction: h_w = h_a = 0)
    if (A->layout != APT_PACK_ROWS) return APT_ERR_UNSUPPORTED;
    uint8_t* xp = reinterpret_cast<uint8_t*>(workspace) + APT_WS_TICKET_BYTES;
    cudaError_t err = apt::launch_expand_tokens_mx(A->planes, (int64_t)M * A->k_words, M, A->k_words, abits, xp, s);
    if (err != cudaSuccess) return APT_ERR_CUDA;
    apt::TcArgs p;
    p.wp = W->planes;
    p.w_tiled = W->layout == APT_PACK_TILED ? 1 : 0;
    p.w_pstride = (int64_t)(p.w_tiled ? (N + 127) / 128 * 128 : N) * W->k_words;
    p.adig = xp;
    p.k_words = W->k_words;
    p.e = e;
    p.e.h_w = 0;
    p.e.h_a = 0;
    err = apt::launch_gemm_tc(p, wbits, c.bn, 1, 1, 1, s);
    return err == cudaSuccess ? APT_OK : APT_ERR_CUDA;
  }
  const uint8_t* adig = A->digits;
  if (!adig && A->layout != APT_PACK_ROWS) return APT_ERR_UNSUPPORTED;
  if (!adig) {
    uint8_t* xp = reinterpret_cast<uint8_t*>(workspace) + APT_WS_TICKET_BYTES;
    cudaError_t err = apt::launch_expand_tokens(A->planes, (int64_t)M * A->k_words, M, A->k_words, abits, xp, s);
    if (err != cudaSuccess) return APT_ERR_CUDA;
    adig = xp;
  }
  if (c.kernel == APT_KERNEL_GEMV || c.kernel == APT_KERNEL_SKINNY) {
    apt::GemvArgs p;
    p.wp = W->planes;
    p.w_tiled = W->layout == APT_PACK_TILED ? 1 : 0;
    p.w_pstride = (int64_t)(p.w_tiled ? (N + 127) / 128 * 128 : N) * W->k_words;
    p.adig = adig;
    p.k_words = W->k_words;
    p.e = e;
    cudaError_t err = c.kernel == APT_KERNEL_GEMV ? apt::launch_gemv(p, wbits, c.split_k, s)
                                                  : apt::launch_gemm_skinny(p, wbits, c.bn, c.split_k, s);
    return err == cudaSuccess ? APT_OK : APT_ERR_CUDA;
  }
  if (c.kernel == APT_KERNEL_DEC) {
    apt::DecArgs p;
    p.wp = W->planes;
    p.w_tiled = W->layout == APT_PACK_TILED ? 1 : 0;
    p.w_pstride = (int64_t)(p.w_tiled ? (N + 127) / 128 * 128 : N) * W->k_words;
    p.adig = adig;
    p.k_words = W->k_words;
    p.e = e;
    p.partials = nullptr;
    p.counters = nullptr;
    if (c.split_k > 1) {
      p.partials = reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(workspace) + ws_dec_off(M, e.K));
      p.counters = reinterpret_cast<uint32_t*>(workspace);
    }
    cudaError_t err = apt::launch_gemm_dec(p, wbits, c.stages, c.split_k, s);
    return err == cudaSuccess ? APT_OK : APT_ERR_CUDA;
  }
  if (c.kernel == APT_KERNEL_TC) {
    apt::TcArgs p;
    p.wp = W->planes;
    p.w_tiled = W->layout == APT_PACK_TILED ? 1 : 0;
    p.w_pstride = (int64_t)(p.w_tiled ? (N + 127) / 128 * 128 : N) * W->k_words;
    p.adig = adig;
    p.k_words = W->k_words;
    p.e = e;
    cudaError_t err = apt::launch_gemm_tc(p, wbits, c.bn, c.cluster_n, c.split_k, 0, s);
    return err == cudaSuccess ? APT_OK : APT_ERR_CUDA;
  }
  return APT_ERR_UNSUPPORTED;
}
}  // namespace
