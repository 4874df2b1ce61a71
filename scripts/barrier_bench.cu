// dev microbenchmark: cost of one grid-wide all-reduce barrier on B200 vs CTA count.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o barrier_bench barrier_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// mode 0: counter barrier only; 1: + 5 partials write/read (redundant reduce); 2: + dummy L2 load chain
template <int MODE>
__global__ void __launch_bounds__(256, 4) bar_kernel(unsigned long long* ctr, double* part, int iters, double* out) {
  __shared__ double sh[8][5];
  __shared__ double tot[5];
  const int G = gridDim.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    double v[5];
    for (int k = 0; k < 5; ++k) v[k] = threadIdx.x * 1e-3 + it;
    if (MODE >= 1) {
      for (int k = 0; k < 5; ++k) {
        double s = v[k];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) sh[w][k] = s;
      }
      __syncthreads();
    }
    double* pp = part + (size_t)(it & 1) * 5 * G;
    if (threadIdx.x == 0) {
      if (MODE >= 1)
        for (int k = 0; k < 5; ++k) {
          double s = 0;
          for (int i = 0; i < 8; ++i) s += sh[i][k];
          __stcg(pp + k * G + blockIdx.x, s);
        }
      if (MODE != 3) __threadfence();
      const unsigned long long target = (unsigned long long)(it + 1) * G;
      if (MODE == 3) {   // release-atomic, acquire spin, no full fences
        unsigned long long one = 1, old;
        asm volatile("atom.add.release.gpu.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(ctr), "l"(one) : "memory");
        while (ld_acquire(ctr) < target) {
        }
      } else if (MODE == 2) {   // last arriver releases a flag on another line
        unsigned long long old = atomicAdd(ctr, 1ull);
        unsigned long long* flag = ctr + 32;
        if (old == target - 1) { __threadfence(); atomicExch(flag, (unsigned long long)(it + 1)); }
        else while (ld_acquire(flag) < (unsigned long long)(it + 1)) { }
      } else {
        atomicAdd(ctr, 1ull);
        while (ld_acquire(ctr) < target) {
        }
      }
      if (MODE != 3) __threadfence();
    }
    __syncthreads();
    if (MODE >= 1) {
      if (w < 5) {
        double s = 0;
        for (int i = lane; i < G; i += 32) s += __ldcg(pp + w * G + i);
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) tot[w] = s;
      }
      __syncthreads();
      acc += tot[0];
      __syncthreads();
    }
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = acc;
}

// LL-style: each CTA publishes its 5 partials as 10 x (32-bit half, 32-bit epoch) 8-byte words;
// readers poll the words until every epoch matches (no counter, no atomics).
template <int FENCE>
__global__ void __launch_bounds__(256, 4) ll_kernel(unsigned long long* slots, int iters, double* out) {
  __shared__ double sh[8][5];
  __shared__ double tot[5];
  const int G = gridDim.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    const unsigned ep = (unsigned)it + 1u;
    for (int k = 0; k < 5; ++k) {
      double s = threadIdx.x * 1e-3 + it;
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) sh[w][k] = s;
    }
    __syncthreads();
    unsigned long long* sl = slots + (size_t)(it & 1) * 10 * G;
    if (w == 0) {
      double v = 0.0;
      if (lane < 10) for (int i = 0; i < 8; ++i) v += sh[i][lane >> 1];
      if (FENCE) __threadfence();
      if (lane < 10) {
        unsigned long long bits = __double_as_longlong(v);
        unsigned half = (lane & 1) ? (unsigned)(bits >> 32) : (unsigned)bits;
        unsigned long long word = ((unsigned long long)ep << 32) | half;
        asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(sl + (size_t)lane * G + blockIdx.x), "l"(word) : "memory");
      }
    }
    if (w < 5) {
      double s = 0.0;
      for (int i = lane; i < G; i += 32) {
        unsigned long long lo, hi;
        do { asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(lo) : "l"(sl + (size_t)(2 * w) * G + i) : "memory"); } while ((unsigned)(lo >> 32) != ep);
        do { asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(hi) : "l"(sl + (size_t)(2 * w + 1) * G + i) : "memory"); } while ((unsigned)(hi >> 32) != ep);
        s += __longlong_as_double((long long)((hi << 32) | (lo & 0xffffffffull)));
      }
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) tot[w] = s;
      if (FENCE) __threadfence();
    }
    __syncthreads();
    acc += tot[0];
    __syncthreads();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = acc;
}

// mode 4: release-atomic barrier, parallel partial publish, all-thread partial fetch
__global__ void __launch_bounds__(256, 4) fast_kernel(unsigned long long* ctr, double* part, int iters, double* out) {
  __shared__ double sh[8][5];
  __shared__ double tot[5];
  const int G = gridDim.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    for (int k = 0; k < 5; ++k) {
      double s = threadIdx.x * 1e-3 + it;
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) sh[w][k] = s;
    }
    __syncthreads();
    double* pp = part + (size_t)(it & 1) * 5 * G;
    if (w == 0) {
      if (lane < 5) {
        double s = 0;
        for (int i = 0; i < 8; ++i) s += sh[i][lane];
        __stcg(pp + (size_t)blockIdx.x * 5 + lane, s);
      }
      __syncwarp();
      if (lane == 0) {
        const unsigned long long target = (unsigned long long)(it + 1) * G;
        unsigned long long one = 1, old;
        asm volatile("atom.add.release.gpu.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(ctr), "l"(one) : "memory");
        while (ld_acquire(ctr) < target) {
        }
      }
    }
    __syncthreads();
    double v[5] = {0, 0, 0, 0, 0};
    for (int i = threadIdx.x; i < G; i += 256) {
      double t[5];
      for (int k = 0; k < 5; ++k) t[k] = __ldcg(pp + (size_t)i * 5 + k);
      for (int k = 0; k < 5; ++k) v[k] += t[k];
    }
    for (int k = 0; k < 5; ++k) {
      double s = v[k];
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) sh[w][k] = s;
    }
    __syncthreads();
    if (threadIdx.x < 5) {
      double s = 0;
      for (int i = 0; i < 8; ++i) s += sh[i][threadIdx.x];
      tot[threadIdx.x] = s;
    }
    __syncthreads();
    acc += tot[0];
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = acc;
}

float run_fast(int G, int iters, unsigned long long* ctr, double* part, double* out) {
  cudaMemset(ctr, 0, 512);
  void* args[] = {&ctr, &part, &iters, &out};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaLaunchCooperativeKernel((void*)fast_kernel, G, 256, args, 0, 0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.f / iters;
}

template <int FENCE>
float run_ll(int G, int iters, unsigned long long* slots, double* out) {
  cudaMemset(slots, 0, 2 * 10 * 1024 * 8);
  void* args[] = {&slots, &iters, &out};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaLaunchCooperativeKernel((void*)ll_kernel<FENCE>, G, 256, args, 0, 0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
  return ms * 1000.f / iters;
}

template <int MODE>
float run(int G, int iters, unsigned long long* ctr, double* part, double* out) {
  cudaMemset(ctr, 0, 512);
  void* args[] = {&ctr, &part, &iters, &out};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaLaunchCooperativeKernel((void*)bar_kernel<MODE>, G, 256, args, 0, 0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
  return ms * 1000.f / iters;
}

int main() {
  unsigned long long* ctr;
  double *part, *out;
  cudaMalloc(&ctr, 512);
  cudaMalloc(&part, 2 * 5 * 1024 * 8);
  cudaMalloc(&out, 8);
  unsigned long long* slots;
  cudaMalloc(&slots, 2 * 10 * 1024 * 8);
  int Gs[] = {1, 8, 16, 32, 64, 74, 148, 296, 444, 592};
  for (int G : Gs) {
    run<0>(G, 100, ctr, part, out);
    float t0 = run<0>(G, 20000, ctr, part, out);
    float t1 = run<1>(G, 20000, ctr, part, out);
    float t3 = run<3>(G, 20000, ctr, part, out);
    float t4 = run_fast(G, 20000, ctr, part, out);
    printf("G=%4d  barrier %.3f  barrier+reduce %.3f  release-atomic+reduce %.3f  fast %.3f us\n", G, t0, t1, t3, t4);
  }
  return 0;
}
