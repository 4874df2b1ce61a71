// dev microbenchmark: one group all-reduce of 5 fp64 partials per iteration across G CTAs.
//   cur : the step kernel's protocol (CTA tree -> st.cg partials -> red.release counter ->
//         ld.acquire spin -> partial reads)
//   ll  : flag-in-word protocol: every CTA publishes each partial as two 64-bit words
//         (epoch << 32 | 32-bit half); readers poll the words until every epoch matches.
//         No fences, no atomics; 64-bit accesses are single-copy atomic, so a word whose
//         epoch matches carries that epoch's half.
//   llh : ll + a halo exchange per iteration: every thread publishes 2 rows x 3 doubles
//         as flagged words and reads 2 rows of another CTA (validated the same way)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ll_bench ll_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ ulonglong2 ldv2(const ulonglong2* p) {
  ulonglong2 v;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void stv2(ulonglong2* p, ulonglong2 v) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(v.x), "l"(v.y) : "memory");
}
__device__ __forceinline__ ulonglong2 ll_pack(double d, unsigned ep) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(d);
  const unsigned long long e = (unsigned long long)ep << 32;
  return make_ulonglong2(e | (b & 0xffffffffull), e | (b >> 32));
}
__device__ __forceinline__ bool ll_ok(ulonglong2 w, unsigned ep) {
  return (unsigned)(w.x >> 32) == ep && (unsigned)(w.y >> 32) == ep;
}
__device__ __forceinline__ double ll_val(ulonglong2 w) {
  return __longlong_as_double((long long)((w.y << 32) | (w.x & 0xffffffffull)));
}

constexpr int GMAX = 1024;

__global__ void __launch_bounds__(256, 2) cur_kernel(unsigned long long* ctr, double* part, int iters, double* out) {
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
    if (threadIdx.x == 0) {
      for (int k = 0; k < 5; ++k) {
        double s = 0;
        for (int i = 0; i < 8; ++i) s += sh[i][k];
        __stcg(pp + k * G + blockIdx.x, s);
      }
      red_release_add(ctr, 1ull);
      const unsigned long long target = (unsigned long long)(it + 1) * G;
      while (ld_acquire(ctr) < target) {
      }
    }
    __syncthreads();
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
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = acc;
}

// HALO: 0 none, 1 flagged halo words, 2 plain halo stores + loads (current kernel's pattern,
// ordered by the counter barrier)
template <int HALO>
__global__ void __launch_bounds__(256, 2) ll_kernel(ulonglong2* slots, ulonglong2* halo, int iters, unsigned ep0,
                                                    double* out) {
  __shared__ double sh[8][5];
  __shared__ double tot[5];
  const int G = gridDim.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double acc = 0.0;
  double hv = 0.0;
  const int peer = (blockIdx.x + 1) % G;
  for (int it = 0; it < iters; ++it) {
    const unsigned ep = ep0 + (unsigned)it + 1u;
    if (HALO == 1 && it > 0) {
      // previous iteration's rows of the peer CTA (2 rows x 3 values per thread)
      const ulonglong2* src = halo + ((size_t)((it - 1) & 1) * G + peer) * 256 * 6 + threadIdx.x * 6;
      ulonglong2 v[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) v[k] = ldv2(src + k);
#pragma unroll
      for (int k = 0; k < 6; ++k)
        while (!ll_ok(v[k], ep - 1)) v[k] = ldv2(src + k);
#pragma unroll
      for (int k = 0; k < 6; ++k) hv += ll_val(v[k]);
    }
    if (HALO == 1) {
      ulonglong2* dst = halo + ((size_t)(it & 1) * G + blockIdx.x) * 256 * 6 + threadIdx.x * 6;
#pragma unroll
      for (int k = 0; k < 6; ++k) stv2(dst + k, ll_pack(hv + k, ep));
    }
    for (int k = 0; k < 5; ++k) {
      double s = threadIdx.x * 1e-3 + it + hv * 1e-30;
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) sh[w][k] = s;
    }
    __syncthreads();
    ulonglong2* sl = slots + (size_t)(it & 1) * 5 * GMAX;
    if (w == 0 && lane < 5) {
      double s = 0;
      for (int i = 0; i < 8; ++i) s += sh[i][lane];
      stv2(sl + (size_t)lane * GMAX + blockIdx.x, ll_pack(s, ep));
    }
    if (w < 5) {
      const ulonglong2* src = sl + (size_t)w * GMAX;
      double s = 0.0;
      for (int i0 = 0; i0 < G; i0 += 128) {
        ulonglong2 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + lane + 32 * u;
          v[u] = i < G ? ldv2(src + i) : ll_pack(0.0, ep);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + lane + 32 * u;
          while (!ll_ok(v[u], ep)) v[u] = ldv2(src + i);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) s += ll_val(v[u]);
      }
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) tot[w] = s;
    }
    __syncthreads();
    acc += tot[0];
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = acc + hv;
}

// current protocol + plain halo (stores of 6 doubles per thread, loads of the peer's after the barrier)
__global__ void __launch_bounds__(256, 2) curh_kernel(unsigned long long* ctr, double* part, double* halo, int iters,
                                                      double* out) {
  __shared__ double sh[8][5];
  __shared__ double tot[5];
  const int G = gridDim.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double acc = 0.0, hv = 0.0;
  const int peer = (blockIdx.x + 1) % G;
  for (int it = 0; it < iters; ++it) {
    if (it > 0) {
      const double* src = halo + ((size_t)((it - 1) & 1) * G + peer) * 256 * 6 + threadIdx.x * 6;
      double v[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) v[k] = src[k];
#pragma unroll
      for (int k = 0; k < 6; ++k) hv += v[k];
    }
    {
      double* dst = halo + ((size_t)(it & 1) * G + blockIdx.x) * 256 * 6 + threadIdx.x * 6;
#pragma unroll
      for (int k = 0; k < 6; ++k) __stcg(dst + k, hv + k);
    }
    for (int k = 0; k < 5; ++k) {
      double s = threadIdx.x * 1e-3 + it + hv * 1e-30;
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) sh[w][k] = s;
    }
    __syncthreads();
    double* pp = part + (size_t)(it & 1) * 5 * G;
    if (threadIdx.x == 0) {
      for (int k = 0; k < 5; ++k) {
        double s = 0;
        for (int i = 0; i < 8; ++i) s += sh[i][k];
        __stcg(pp + k * G + blockIdx.x, s);
      }
      red_release_add(ctr, 1ull);
      const unsigned long long target = (unsigned long long)(it + 1) * G;
      while (ld_acquire(ctr) < target) {
      }
    }
    __syncthreads();
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
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = acc + hv;
}

// ll2: one 128-B line per CTA (5 flagged values), ONE warp per CTA polls all G lines with
// warp-uniform retries (only words not yet current are reloaded); HALO as in ll_kernel.
template <int HALO, int SLEEP>
__global__ void __launch_bounds__(256, 2) ll2_kernel(ulonglong2* slots, ulonglong2* halo, int iters, unsigned ep0,
                                                     double* out) {
  __shared__ double sh[8][5];
  __shared__ double tot[5];
  const int G = gridDim.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double acc = 0.0;
  double hv = 0.0;
  const int peer = (blockIdx.x + 1) % G;
  for (int it = 0; it < iters; ++it) {
    const unsigned ep = ep0 + (unsigned)it + 1u;
    if (HALO == 1 && it > 0) {
      const ulonglong2* src = halo + ((size_t)((it - 1) & 1) * G + peer) * 256 * 6 + threadIdx.x * 6;
      ulonglong2 v[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) v[k] = ldv2(src + k);
#pragma unroll
      for (int k = 0; k < 6; ++k)
        while (!ll_ok(v[k], ep - 1)) v[k] = ldv2(src + k);
#pragma unroll
      for (int k = 0; k < 6; ++k) hv += ll_val(v[k]);
    }
    if (HALO == 1) {
      ulonglong2* dst = halo + ((size_t)(it & 1) * G + blockIdx.x) * 256 * 6 + threadIdx.x * 6;
#pragma unroll
      for (int k = 0; k < 6; ++k) stv2(dst + k, ll_pack(hv + k, ep));
    }
    for (int k = 0; k < 5; ++k) {
      double s = threadIdx.x * 1e-3 + it + hv * 1e-30;
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) sh[w][k] = s;
    }
    __syncthreads();
    ulonglong2* sl = slots + (size_t)(it & 1) * 8 * GMAX;      // [cta][8] lines of 128 B
    if (w == 0) {
      if (lane < 5) {
        double s = 0;
        for (int i = 0; i < 8; ++i) s += sh[i][lane];
        stv2(sl + (size_t)blockIdx.x * 8 + lane, ll_pack(s, ep));
      }
      // lane l polls CTAs l, l+32, ... (<= 8 per lane: G <= 256)
      double s[5] = {0, 0, 0, 0, 0};
      for (int i0 = 0; i0 < G; i0 += 32) {
        const int i = i0 + lane;
        ulonglong2 v[5];
        bool ok = true;
        if (i < G) {
#pragma unroll
          for (int k = 0; k < 5; ++k) v[k] = ldv2(sl + (size_t)i * 8 + k);
#pragma unroll
          for (int k = 0; k < 5; ++k) ok = ok && ll_ok(v[k], ep);
        }
        while (!__all_sync(0xffffffffu, ok)) {
          if (SLEEP) __nanosleep(SLEEP);
          if (!ok) {
#pragma unroll
            for (int k = 0; k < 5; ++k) v[k] = ldv2(sl + (size_t)i * 8 + k);
            ok = true;
#pragma unroll
            for (int k = 0; k < 5; ++k) ok = ok && ll_ok(v[k], ep);
          }
        }
        if (i < G) {
#pragma unroll
          for (int k = 0; k < 5; ++k) s[k] += ll_val(v[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        double t = s[k];
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) tot[k] = t;
      }
    }
    __syncthreads();
    acc += tot[0];
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = acc + hv;
}

static float timed(void* fn, int G, void** args) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaError_t e = cudaLaunchCooperativeKernel(fn, G, 256, args, 0, 0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  unsigned long long* ctr;
  double *part, *out, *hplain;
  ulonglong2 *slots, *halo;
  cudaMalloc(&ctr, 512);
  cudaMalloc(&part, 2 * 5 * GMAX * 8);
  cudaMalloc(&out, 8);
  cudaMalloc(&slots, 2 * 8 * GMAX * 16);
  cudaMalloc(&halo, (size_t)2 * GMAX * 256 * 6 * 16);
  cudaMalloc(&hplain, (size_t)2 * GMAX * 256 * 6 * 8);
  cudaMemset(slots, 0, 2 * 8 * GMAX * 16);
  cudaMemset(halo, 0, (size_t)2 * GMAX * 256 * 6 * 16);
  unsigned ep = 0;
  const int iters = 20000;
  int Gs[] = {1, 8, 16, 32, 64, 74, 128, 143, 148, 296};
  for (int G : Gs) {
    cudaMemset(ctr, 0, 512);
    int it = iters;
    void* a0[] = {&ctr, &part, &it, &out};
    float t0 = timed((void*)cur_kernel, G, a0);
    cudaMemset(ctr, 0, 512);
    void* a0h[] = {&ctr, &part, &hplain, &it, &out};
    float t0h = timed((void*)curh_kernel, G, a0h);
    void* a1[] = {&slots, &halo, &it, &ep, &out};
    float t1 = timed((void*)ll_kernel<0>, G, a1);
    ep += iters + 2;
    void* a2[] = {&slots, &halo, &it, &ep, &out};
    float t2 = timed((void*)ll_kernel<1>, G, a2);
    ep += iters + 2;
    float t3 = timed((void*)ll2_kernel<0, 0>, G, a2);
    ep += iters + 2;
    float t4 = timed((void*)ll2_kernel<1, 0>, G, a2);
    ep += iters + 2;
    float t5 = timed((void*)ll2_kernel<0, 64>, G, a2);
    ep += iters + 2;
    float t6 = timed((void*)ll2_kernel<1, 64>, G, a2);
    ep += iters + 2;
    printf("G=%4d  cur %.3f  cur+halo %.3f  ll %.3f  ll+halo %.3f  ll2 %.3f  ll2+halo %.3f  ll2s %.3f  ll2s+halo %.3f us/iter\n",
           G, t0 * 1e3f / iters, t0h * 1e3f / iters, t1 * 1e3f / iters, t2 * 1e3f / iters, t3 * 1e3f / iters,
           t4 * 1e3f / iters, t5 * 1e3f / iters, t6 * 1e3f / iters);
  }
  return 0;
}
