// dev microbenchmark: practical HBM ceiling on B200 for the CG pass access patterns.
//   copy   : 1 read stream, 1 write stream            (the MEASURED_PEAKS.json pattern)
//   cgpass : 8 read streams, 4 write streams, 16-B vectors (the grid / ELL CG pass pattern)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_bench stream_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void copy_k(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

__global__ void cg_k(const double2* __restrict__ r, const double2* __restrict__ q, const double2* __restrict__ p,
                     const double2* __restrict__ d, double2* __restrict__ x, const double2* __restrict__ t1,
                     const double2* __restrict__ t2, const double2* __restrict__ s, double2* __restrict__ ro,
                     double2* __restrict__ po, double2* __restrict__ qo, size_t n, double a, double b) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 rr = __ldcg(r + i), qq = __ldcg(q + i), pp = __ldcg(p + i), dd = __ldg(d + i), xx = x[i];
    double2 aa = __ldg(t1 + i), bb = __ldg(t2 + i), ss = __ldg(s + i);
    double2 rn = make_double2(rr.x - a * qq.x, rr.y - a * qq.y);
    double2 pn = make_double2(dd.x * rn.x + b * pp.x, dd.y * rn.y + b * pp.y);
    x[i] = make_double2(xx.x + a * pp.x, xx.y + a * pp.y);
    __stcg(ro + i, rn);
    __stcg(po + i, pn);
    __stcg(qo + i, make_double2(ss.x * pn.x + aa.x + bb.x, ss.y * pn.y + aa.y + bb.y));
  }
}

int main() {
  const size_t n = (size_t)67108864 / 2;   // double2 elements: 67M doubles per array (config 4 grid)
  double2* buf[12];
  for (int k = 0; k < 12; ++k) {
    cudaMalloc(&buf[k], n * sizeof(double2));
    cudaMemset(buf[k], 0, n * sizeof(double2));
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int bps : {2, 4, 8}) {
    float ms;
    copy_k<<<sms * bps, 256>>>(buf[0], buf[1], n);
    cudaEventRecord(e0);
    for (int it = 0; it < 10; ++it) copy_k<<<sms * bps, 256>>>(buf[0], buf[1], n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("copy   blocks/SM %d: %.1f GB/s\n", bps, 10 * 2.0 * n * 16 / (ms * 1e-3) / 1e9);
    cudaEventRecord(e0);
    for (int it = 0; it < 10; ++it)
      cg_k<<<sms * bps, 256>>>(buf[0], buf[1], buf[2], buf[3], buf[4], buf[5], buf[6], buf[7], buf[8], buf[9],
                                buf[10], n, 0.5, 0.25);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("cgpass blocks/SM %d: %.1f GB/s  (%.3f ms per 67M-cell pass)\n", bps, 10 * 12.0 * n * 16 / (ms * 1e-3) / 1e9, ms / 10);
  }
  return 0;
}
