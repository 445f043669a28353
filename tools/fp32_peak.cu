// FP32 pipe microbenchmark: measures sustained FFMA and FFMA2 throughput on this GPU.
// Used to derive the FP32 roofline denominator (MEASURED_PEAKS.json has no fp32 entry).
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1;}}while(0)
template<int ILP>
__global__ void ffma_scalar(float* out, int iters, float a, float b) {
  float r[ILP];
#pragma unroll
  for (int i = 0; i < ILP; i++) r[i] = threadIdx.x * 1e-7f + i;
  for (int t = 0; t < iters; t++) {
#pragma unroll
    for (int i = 0; i < ILP; i++) r[i] = fmaf(r[i], a, b);
  }
  float s = 0; 
#pragma unroll
  for (int i = 0; i < ILP; i++) s += r[i];
  if (s == 12345.f) out[0] = s;
}
template<int ILP>
__global__ void ffma_x2(float* out, int iters, float a, float b) {
  float2 r[ILP];
  float2 A = make_float2(a, a), B = make_float2(b, b);
#pragma unroll
  for (int i = 0; i < ILP; i++) r[i] = make_float2(threadIdx.x * 1e-7f + i, i * 0.5f);
  for (int t = 0; t < iters; t++) {
#pragma unroll
    for (int i = 0; i < ILP; i++) r[i] = __ffma2_rn(r[i], A, B);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < ILP; i++) s += r[i].x + r[i].y;
  if (s == 12345.f) out[0] = s;
}
int main() {
  float* out; CK(cudaMalloc(&out, 4));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 1 << 16; int blocks = sms * 8, threads = 256;
  for (int rep = 0; rep < 3; rep++) {
    ffma_scalar<16><<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
    cudaEventRecord(e0);
    ffma_scalar<16><<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * iters * (double)blocks * threads;
    printf("{\"kernel\":\"ffma_scalar\",\"tflops\":%.2f,\"ms\":%.3f}\n", fl / ms / 1e9, ms);
    ffma_x2<8><<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
    cudaEventRecord(e0);
    ffma_x2<8><<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 2 * 8 * iters * (double)blocks * threads;
    printf("{\"kernel\":\"ffma_x2\",\"tflops\":%.2f,\"ms\":%.3f}\n", fl / ms / 1e9, ms);
  }
  return 0;
}
