// nnm_diag.cu -- diagnostics exported next to the hot path: the FP32 pipe peak
// used as the roofline denominator (MEASURED_PEAKS.json has no FP32 entry).
#include <cuda_runtime.h>

#include "../../include/nnm.h"

namespace {
template <int ILP>
__global__ void ffma2_peak_kernel(float* out, int iters, float a, float b) {
  float2 r[ILP];
  const float2 A = make_float2(a, a), B = make_float2(b, b);
#pragma unroll
  for (int i = 0; i < ILP; i++) r[i] = make_float2(threadIdx.x * 1e-7f + i, i * 0.5f);
  for (int t = 0; t < iters; t++) {
#pragma unroll
    for (int i = 0; i < ILP; i++) r[i] = __ffma2_rn(r[i], A, B);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < ILP; i++) s += r[i].x + r[i].y;
  if (s == 12345.f) out[0] = s;
}
}  // namespace

extern "C" int nnm_measure_fp32_peak(int32_t device, double* tflops) {
  if (cudaSetDevice(device) != cudaSuccess) return NNM_E_CUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  float* out = nullptr;
  if (cudaMalloc(&out, sizeof(float)) != cudaSuccess) return NNM_E_CUDA;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 1 << 15, blocks = sms * 8, threads = 256;
  double best = 0.0;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    ffma2_peak_kernel<8><<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
    cudaEventRecord(e1);
    if (cudaEventSynchronize(e1) != cudaSuccess) return NNM_E_CUDA;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 2 * 8 * (double)iters * blocks * threads;
    if (rep > 0 && fl / (ms * 1e-3) / 1e12 > best) best = fl / (ms * 1e-3) / 1e12;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  *tflops = best;
  return cudaGetLastError() == cudaSuccess ? NNM_OK : NNM_E_CUDA;
}
