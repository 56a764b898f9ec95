// Throughput probes for the decode-kernel design choice: how many weight digits per
// clock per SM each multiply path can consume.
//   legacy mma.sync.m16n8k32 u8 (registers), __dp4a, __popc, LOP3 (integer ALU),
//   tcgen05.mma kind::i8 M=128 x N x K=32 with A in TMEM or SMEM,
//   tcgen05.mma kind::mxf4.block_scale M=128 x N x K=64 (e2m1, unit UE8M0 scales), A in SMEM / TMEM.
// One JSON line per probe.  Operand values are irrelevant (rates are data independent).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rates mma_rates.cu && ./mma_rates
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("{\"error\": \"%s line %d\"}\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

__device__ unsigned long long g_sink;
__device__ long long g_cyc[1024];

// ------------------------------------------------------------------------------------ legacy IMMA
template <int NACC>
__global__ void imma_kernel(int iters) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 9, b1 = a0 ^ 11;
  int c[NACC][4] = {};
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < NACC; ++q)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(c[q][0]), "+r"(c[q][1]), "+r"(c[q][2]), "+r"(c[q][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  __syncthreads();
  const long long t1 = clock64();
  int s = 0;
#pragma unroll
  for (int q = 0; q < NACC; ++q) s += c[q][0] + c[q][1] + c[q][2] + c[q][3];
  if (s == 0x12345) g_sink = s;
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = t1 - t0;
}

// ------------------------------------------------------------------------------------ integer ALU
template <int OP>
__global__ void alu_kernel(int iters) {
  uint32_t x[8], acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) { x[j] = threadIdx.x * (j + 3); acc[j] = j; }
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) acc[j] = __dp4a(x[j], acc[j], acc[j]);
      if (OP == 1) acc[j] += __popc(acc[j] ^ x[j]);
      if (OP == 2) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(acc[j]) : "r"(x[j]), "r"(x[(j + 1) & 7]));
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += acc[j];
  if (s == 0x12345) g_sink = s;
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = t1 - t0;
}

// ------------------------------------------------------------------------------------ tcgen05
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t a) {
  uint64_t d = 0;
  d |= (uint64_t)((a >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// KIND 0 = i8 (K=32 per instruction), 1 = mxf4 block_scale scale_vec::2X (K=64)
template <int N, bool ATMEM, int KIND>
__global__ void __launch_bounds__(128, 1) tc_kernel(int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const uint32_t sA = base, sB = base + 16384;
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 8192; i += 128) reinterpret_cast<uint32_t*>(smem + (base - smem_u32(smem)))[i] = 0x3C3C3C3Cu;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  // fill TMEM columns 256..511 (A operand / scale factors) with 0x7F bytes = UE8M0 2^0
  {
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    uint32_t r[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) r[j] = 0x7F7F7F7Fu;
#pragma unroll 1
    for (int c = 256; c < 512; c += 32)
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
          "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tmem + lane_off + c),
          "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
          "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
          "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
          "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
          : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    uint32_t idesc;
    if (KIND == 0) idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    else idesc = (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t bd = desc_sw128(sB), ad = desc_sw128(sA);
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t acc = (i | kk) != 0;
        if (KIND == 0) {
          if (ATMEM)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                         "r"(tmem + 256 + 8 * kk), "l"(bd + 2 * kk), "r"(idesc), "r"(acc) : "memory");
          else
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                         "l"(ad + 2 * kk), "l"(bd + 2 * kk), "r"(idesc), "r"(acc) : "memory");
        } else {
          if (ATMEM)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], [%1], %2, %3, [%5], [%6], p;\n\t}"
                         ::"r"(tmem), "r"(tmem + 256 + 8 * kk), "l"(bd + 2 * kk), "r"(idesc), "r"(acc),
                         "r"(tmem + 480), "r"(tmem + 496) : "memory");
          else
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%5], [%6], p;\n\t}"
                         ::"r"(tmem), "l"(ad + 2 * kk), "l"(bd + 2 * kk), "r"(idesc), "r"(acc),
                         "r"(tmem + 480), "r"(tmem + 496) : "memory");
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(smem_u32(&bar)) : "memory");
    t1 = clock64();
    g_cyc[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

static long long max_cyc(int n) {
  long long h[1024];
  cudaMemcpyFromSymbol(h, g_cyc, sizeof(long long) * n);
  long long m = 0;
  for (int i = 0; i < n; ++i) m = h[i] > m ? h[i] : m;
  return m;
}

template <int NACC>
static int run_imma(int warps, int ctas_per_sm) {
  const int iters = 4096, grid = 148 * ctas_per_sm;
  imma_kernel<NACC><<<grid, 32 * warps>>>(iters);
  CK(cudaDeviceSynchronize());
  imma_kernel<NACC><<<grid, 32 * warps>>>(iters);
  CK(cudaDeviceSynchronize());
  const double cyc = (double)max_cyc(grid);
  const double macs_sm = (double)iters * NACC * 4096.0 * warps * ctas_per_sm;
  printf("{\"probe\": \"imma_m16n8k32_u8\", \"warps_per_sm\": %d, \"acc_chains\": %d, \"mac_per_clk_sm\": %.1f}\n",
         warps * ctas_per_sm, NACC, macs_sm / cyc);
  return 0;
}

template <int OP>
static int run_alu(const char* name, int warps) {
  const int iters = 4096, grid = 148;
  alu_kernel<OP><<<grid, 32 * warps>>>(iters);
  CK(cudaDeviceSynchronize());
  alu_kernel<OP><<<grid, 32 * warps>>>(iters);
  CK(cudaDeviceSynchronize());
  const double cyc = (double)max_cyc(grid);
  printf("{\"probe\": \"%s\", \"warps_per_sm\": %d, \"lane_ops_per_clk_sm\": %.1f}\n", name, warps,
         (double)iters * 8 * 32 * warps / cyc);
  return 0;
}

template <int N, bool ATMEM, int KIND>
static int run_tc() {
  const int iters = 256, grid = 148;
  auto k = tc_kernel<N, ATMEM, KIND>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
  k<<<grid, 128, 64 * 1024>>>(iters);
  CK(cudaDeviceSynchronize());
  k<<<grid, 128, 64 * 1024>>>(iters);
  CK(cudaDeviceSynchronize());
  const double cyc = (double)max_cyc(grid);
  const int kper = KIND == 0 ? 32 : 64;
  const double per = cyc / (iters * 4.0);
  printf("{\"probe\": \"tcgen05_%s\", \"M\": 128, \"N\": %d, \"K\": %d, \"A\": \"%s\", \"clk_per_mma\": %.2f, "
         "\"mac_per_clk_sm\": %.1f, \"weight_elems_per_clk_sm\": %.1f}\n",
         KIND == 0 ? "i8" : "mxf4", N, kper, ATMEM ? "tmem" : "smem", per, 128.0 * N * kper / per, 128.0 * kper / per);
  return 0;
}

int main() {
  int dev = 0, clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"probe\": \"device\", \"sm_clock_khz\": %d}\n", clk);
  if (run_imma<4>(4, 1)) return 1;
  if (run_imma<4>(8, 1)) return 1;
  if (run_imma<8>(16, 1)) return 1;
  if (run_imma<2>(32, 1)) return 1;
  if (run_alu<0>("dp4a", 16)) return 1;
  if (run_alu<1>("popc_xor_add", 16)) return 1;
  if (run_alu<2>("lop3", 16)) return 1;
  if (run_tc<16, true, 0>()) return 1;
  if (run_tc<16, false, 0>()) return 1;
  if (run_tc<8, false, 0>()) return 1;
  if (run_tc<32, true, 0>()) return 1;
  if (run_tc<64, true, 0>()) return 1;
  if (run_tc<256, true, 0>()) return 1;
  if (run_tc<256, false, 0>()) return 1;
  if (run_tc<16, false, 1>()) return 1;
  if (run_tc<16, true, 1>()) return 1;
  if (run_tc<8, false, 1>()) return 1;
  if (run_tc<64, false, 1>()) return 1;
  if (run_tc<256, false, 1>()) return 1;
  return 0;
}
