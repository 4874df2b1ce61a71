// dev microbenchmark: per-iteration floor of a cluster-resident CG loop (DSMEM + cluster
// barriers), and whether a 16-CTA cluster kernel co-runs with a cooperative kernel.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cluster_bench cluster_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

constexpr int NT = 512;

__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cl_size() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned mapa(const void* p, unsigned rank) {
  unsigned a = (unsigned)__cvta_generic_to_shared(p), d;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(rank));
  return d;
}
__device__ __forceinline__ double ld_dsmem(unsigned a) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_dsmem(unsigned a, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int R, int NB>
__global__ void __launch_bounds__(NT, 1) cl_loop(int iters, double* out, long long* stamps) {
  extern __shared__ double sm[];
  double* p_s = sm;                       // [R * NT]
  double* slots = sm + R * NT;            // [2][16][8]
  __shared__ double red[NT / 32][5];
  __shared__ double tot[5];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const unsigned rank = cl_rank(), C = cl_size();
  if (t == 0) stamps[2 * blockIdx.x] = gtimer();
  double p[R], q[R], r[R], d[R];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    p[k] = 1e-3 * (t + k);
    r[k] = 1.0;
    d[k] = 0.5;
    q[k] = 0.0;
  }
  double a = 0.001, b = 0.5;
  const unsigned nbr = mapa(p_s, (rank + 1) % C);
  cl_sync();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < R; ++k) {
      r[k] = __fma_rn(-a, q[k], r[k]);
      p[k] = __fma_rn(d[k], r[k], b * p[k]);
      p_s[k * NT + t] = p[k];
    }
    if (NB == 2) cl_sync();
    else __syncthreads();
    double acc[5] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < R; ++k) {
      double pl = __shfl_up_sync(0xffffffffu, p[k], 1);
      double pr = __shfl_down_sync(0xffffffffu, p[k], 1);
      if (lane == 0) pl = t > 0 ? p_s[k * NT + t - 1] : 0.0;
      if (lane == 31) pr = t + 1 < NT ? p_s[k * NT + t + 1] : ld_dsmem(nbr + 8u * (unsigned)(k * NT));
      q[k] = 3.0 * p[k] + (p[k] - pl) + (p[k] - pr);
      acc[0] += p[k] * q[k];
      acc[1] += r[k] * r[k];
      acc[2] += d[k] * r[k] * r[k];
      acc[3] += d[k] * r[k] * q[k];
      acc[4] += d[k] * q[k] * q[k];
    }
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      double s = acc[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) red[w][k] = s;
    }
    __syncthreads();
    double* sl = slots + (it & 1) * 128;
    if (w == 0) {
      // lane = 5 * dst + k for dst < C ... C <= 16 -> 80 (dst, k) pairs over 32 lanes
      double v[5];
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < NT / 32; ++i) s += red[i][k];
        v[k] = s;
      }
      for (int e = lane; e < 5 * (int)C; e += 32) {
        const int dst = e / 5, k = e % 5;
        double val = v[0];
        if (k == 1) val = v[1];
        if (k == 2) val = v[2];
        if (k == 3) val = v[3];
        if (k == 4) val = v[4];
        st_dsmem(mapa(sl + rank * 8 + k, dst), val);
      }
    }
    cl_sync();
    if (w == 0 && lane < 5) {
      double s = 0.0;
      for (unsigned c = 0; c < C; ++c) s += sl[c * 8 + lane];
      tot[lane] = s;
    }
    __syncthreads();
    a = 1e-9 * tot[0];
    b = 0.5 + 1e-12 * tot[2];
  }
  cl_sync();
  if (t == 0) {
    stamps[2 * blockIdx.x + 1] = gtimer();
    out[blockIdx.x] = a + b + p[0];
  }
}

// cooperative companion: G CTAs spinning through a counter barrier for `iters` rounds
__global__ void __launch_bounds__(256, 2) coop_loop(unsigned long long* ctr, int iters, long long* stamps) {
  if (threadIdx.x == 0) stamps[2 * blockIdx.x] = gtimer();
  for (int it = 0; it < iters; ++it) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(ctr, 1ull);
      const unsigned long long target = (unsigned long long)(it + 1) * gridDim.x;
      while (*(volatile unsigned long long*)ctr < target) {
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) stamps[2 * blockIdx.x + 1] = gtimer();
}

template <int R, int NB>
float run_cl(int C, int iters, double* out, long long* stamps, cudaStream_t s, bool timeit = true) {
  const size_t smem = (size_t)R * NT * 8 + 2 * 128 * 8;
  cudaFuncSetAttribute(cl_loop<R, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(cl_loop<R, NB>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, s);
  cudaError_t e = cudaLaunchKernelEx(&cfg, cl_loop<R, NB>, iters, out, stamps);
  cudaEventRecord(b, s);
  if (!timeit) return 0.f;
  cudaEventSynchronize(b);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) printf("err C=%d: %s\n", C, cudaGetErrorString(e));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  double* out;
  long long *st1, *st2;
  unsigned long long* ctr;
  cudaMalloc(&out, 4096 * 8);
  cudaMalloc(&st1, 4096 * 8);
  cudaMalloc(&st2, 4096 * 8);
  cudaMalloc(&ctr, 64);
  {
    int ncl = 0;
    const size_t smem = (size_t)9 * NT * 8 + 2 * 128 * 8;
    cudaFuncSetAttribute(cl_loop<9, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(cl_loop<9, 2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int C : {8, 16}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(C);
      cfg.blockDim = dim3(NT);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = C;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, cl_loop<9, 2>, &cfg);
      printf("max active clusters of %d (smem %zu): %d (%s)\n", C, smem, ncl, cudaGetErrorString(e));
    }
  }
  const int iters = 20000;
  for (int C : {1, 2, 4, 8, 16}) {
    run_cl<9, 2>(C, 100, out, st1, 0);
    float t2 = run_cl<9, 2>(C, iters, out, st1, 0);
    float t1 = run_cl<9, 1>(C, iters, out, st1, 0);
    float t4 = run_cl<4, 2>(C, iters, out, st1, 0);
    printf("C=%2d  R=9 2 cluster barriers %.3f us/iter   R=9 1 barrier (+syncthreads) %.3f   R=4 2 barriers %.3f\n", C,
           t2 * 1e3f / iters, t1 * 1e3f / iters, t4 * 1e3f / iters);
  }
  // co-residency: cluster kernel (16 x 1 CTA/SM, ~37 KB... big smem) first, then a cooperative kernel
  cudaStream_t sa, sb;
  cudaStreamCreateWithFlags(&sa, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking);
  cudaFuncSetAttribute(coop_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(ctr, 0, 64);
    cudaDeviceSynchronize();
    run_cl<9, 2>(16, 50000, out, st1, sb, false);
    int G = 2 * (148 - 16), it2 = 20000;
    void* args[] = {&ctr, &it2, &st2};
    cudaError_t e = cudaLaunchCooperativeKernel((void*)coop_loop, G, 256, args, 70000, sa);
    cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaGetLastError();
    long long h1[32], h2[600];
    cudaMemcpy(h1, st1, 32 * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2, st2, 2 * G * 8, cudaMemcpyDeviceToHost);
    long long c0 = h1[0], c1 = h1[1], k0 = h2[0], k1 = h2[1];
    for (int i = 0; i < 16; ++i) { c0 = c0 < h1[2 * i] ? c0 : h1[2 * i]; c1 = c1 > h1[2 * i + 1] ? c1 : h1[2 * i + 1]; }
    for (int i = 0; i < G; ++i) { k0 = k0 < h2[2 * i] ? k0 : h2[2 * i]; k1 = k1 > h2[2 * i + 1] ? k1 : h2[2 * i + 1]; }
    printf("coresidency rep %d (%s): cluster [%.1f, %.1f] us  coop(G=%d) [%.1f, %.1f] us\n", rep, cudaGetErrorString(e),
           0.0, (c1 - c0) * 1e-3, G, (k0 - c0) * 1e-3, (k1 - c0) * 1e-3);
  }
  return 0;
}
