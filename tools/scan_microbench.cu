// Microbenchmark of the screening inner loop's instruction mix (register only):
// per k: 8 x scalars (broadcast) x 4 float2 y -> 32 FADD2 + 32 FFMA2.
// Measures achievable pair throughput vs occupancy, to bound the scan kernel.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void __launch_bounds__(256) mb(float* out, int iters, int d) {
  float2 acc[8][4];
#pragma unroll
  for (int r = 0; r < 8; r++)
#pragma unroll
    for (int q = 0; q < 4; q++) acc[r][q] = make_float2(0, 0);
  float xr[8];
  float2 yc[4];
#pragma unroll
  for (int r = 0; r < 8; r++) xr[r] = threadIdx.x * 1e-3f + r;
#pragma unroll
  for (int q = 0; q < 4; q++) yc[q] = make_float2(q * 0.25f, q * 0.5f + threadIdx.x * 1e-4f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll 1
    for (int k = 0; k < d; ++k) {
#pragma unroll
      for (int r = 0; r < 8; r++)
#pragma unroll
        for (int q = 0; q < 4; q++) {
          if (MODE == 0) {
            float2 dd = __fadd2_rn(yc[q], make_float2(-xr[r], -xr[r]));
            acc[r][q] = __ffma2_rn(dd, dd, acc[r][q]);
          } else {
            acc[r][q] = __ffma2_rn(yc[q], make_float2(xr[r], xr[r]), acc[r][q]);
          }
        }
#pragma unroll
      for (int r = 0; r < 8; r++) xr[r] += 1e-7f;
    }
  }
  float s = 0;
#pragma unroll
  for (int r = 0; r < 8; r++)
#pragma unroll
    for (int q = 0; q < 4; q++) s += acc[r][q].x + acc[r][q].y;
  if (s == 1.2345f) out[0] = s;
}
int main() {
  float* out;
  cudaMalloc(&out, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int d = 25, iters = 400;
  for (int mode = 0; mode < 2; ++mode)
    for (int ctas = 1; ctas <= 4; ctas *= 2) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (mode == 0) mb<0><<<sms * ctas, 256>>>(out, iters, d);
        else mb<1><<<sms * ctas, 256>>>(out, iters, d);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double pairs = 64.0 * 256 * sms * ctas * (double)iters * d / d;  // pairs x d-steps / d
        double lane_ops = 64.0 * 256 * sms * ctas * (double)iters * d * (mode == 0 ? 2 : 1);
        if (rep) printf("{\"mode\":\"%s\",\"ctas_per_sm\":%d,\"pairs_per_s\":%.3e,\"fma_lane_ops_T\":%.2f}\n",
                        mode ? "dot" : "direct", ctas, pairs / (ms * 1e-3), lane_ops / (ms * 1e-3) / 1e12);
      }
    }
  return 0;
}
