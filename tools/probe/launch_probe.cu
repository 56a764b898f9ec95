// Launch-overhead probe: back-to-back launches (CUDA graph, PDL) of a kernel that only spins for a
// fixed time, for cluster sizes 1/2/4/8 and per-CTA shared memory sizes.  Reports the per-launch
// period and the CTA entry spread, to separate launch/cluster-scheduling cost from kernel work.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o launch_probe launch_probe.cu && ./launch_probe
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ unsigned long long g_entry[16][1024];
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void probe(int launch, unsigned spin_ns, int tmem) {
  extern __shared__ char sm[];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const unsigned long long t0 = gt();
  if (threadIdx.x == 0) g_entry[launch & 15][blockIdx.x + gridDim.x * blockIdx.z] = t0;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (tmem && threadIdx.x < 32) {
    __shared__ unsigned slot;
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" :: "r"((unsigned)__cvta_generic_to_shared(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    __syncwarp();
    const unsigned t = *(volatile unsigned*)&slot;
    while (gt() - t0 < spin_ns) {}
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" :: "r"(t) : "memory");
  } else {
    while (gt() - t0 < spin_ns) {}
  }
  sm[threadIdx.x] = 0;
}

int main() {
  const int ctas = 256, L = 16;
  int dev = 0; cudaSetDevice(dev);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaStream_t s; cudaStreamCreate(&s);
  printf("%8s %8s %6s %6s %10s %10s %10s\n", "cluster", "smemKB", "spin", "tmem", "us/launch", "entry_p50", "entry_p90");
  for (int tmem = 0; tmem < 2; ++tmem)
  for (unsigned spin : {500u, 3000u})
  for (int smem_kb : {60, 113}) for (int cl : {1, 2, 4, 8}) {
    auto launch = [&](int i) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(ctas / 8, 1, 8); cfg.blockDim = dim3(384); cfg.dynamicSmemBytes = smem_kb * 1024; cfg.stream = s;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = cl;
      at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[1].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at; cfg.numAttrs = 2;
      return cudaLaunchKernelEx(&cfg, probe, i, spin, tmem);
    };
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < L; ++i) launch(i);
    cudaStreamEndCapture(s, &g);
    if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("instantiate failed cl=%d\n", cl); return 1; }
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, s);
    cudaEventRecord(e0, s); cudaGraphLaunch(ge, s); cudaEventRecord(e1, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) { printf("err %s\n", cudaGetErrorString(cudaGetLastError())); return 1; }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    static unsigned long long h[16][1024];
    cudaMemcpyFromSymbol(h, g_entry, sizeof(h));
    std::vector<double> sp50, sp90;
    for (int i = 1; i < L; ++i) {
      std::vector<unsigned long long> v(h[i], h[i] + ctas);
      std::sort(v.begin(), v.end());
      sp50.push_back((double)(v[ctas / 2] - v[0])); sp90.push_back((double)(v[ctas * 9 / 10] - v[0]));
    }
    std::sort(sp50.begin(), sp50.end()); std::sort(sp90.begin(), sp90.end());
    printf("%8d %8d %6u %6d %10.3f %10.0f %10.0f\n", cl, smem_kb, spin, tmem, ms * 1e3 / L, sp50[sp50.size() / 2], sp90[sp90.size() / 2]);
    cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
  }
  return 0;
}
