// alert_probe.cu — instrumentation: measured FP32 issue peak of this GPU
// (independent FFMA chains, immediate-free register form, full occupancy),
// the denominator of the FP32 roofline reported by bench.py.
#include <cuda_runtime.h>

#include "../../include/alert_b200.h"

__global__ void __launch_bounds__(256) ffma_probe_kernel(float* out, int iters, float a, float b) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
      x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
    }
  }
  float s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 1234.5f) out[0] = s;  // keep the chains alive
}

// FFMA lane-ops per second (one lane-op = one FP32 issue slot).
int alert_probe_fp32_peak(int device, double* slots_per_s) {
  if (!slots_per_s) return ALERT_ERR_INVALID_ARGUMENT;
  if (cudaSetDevice(device) != cudaSuccess) return ALERT_ERR_CUDA;
  cudaDeviceProp p;
  if (cudaGetDeviceProperties(&p, device) != cudaSuccess) return ALERT_ERR_CUDA;
  float* out = nullptr;
  if (cudaMalloc(&out, 4) != cudaSuccess) return ALERT_ERR_CUDA;
  const int blocks = p.multiProcessorCount * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  ffma_probe_kernel<<<blocks, threads>>>(out, 64, 0.999f, 0.001f);  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    ffma_probe_kernel<<<blocks, threads>>>(out, iters, 0.999f, 0.001f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaError_t e = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (e != cudaSuccess) return ALERT_ERR_CUDA;
  *slots_per_s = (double)blocks * threads * iters * 16.0 * 8.0 / (best * 1e-3);
  return ALERT_OK;
}

#include "alert_device.cuh"

__global__ void phi32_probe_kernel(const float* x, float* out, long long n) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = alert::phi32_x(x[i]);
}

// The FP32 normal CDF of the scan, Phi(sqrt(2) * x[i]) -> out[i] (device
// pointers): lets the tests bound its error against FP64 (instrumentation).
int alert_probe_phi32(const float* x, float* out, int64_t n, void* cuda_stream) {
  if (!x || !out || n < 0) return ALERT_ERR_INVALID_ARGUMENT;
  if (n == 0) return ALERT_OK;
  phi32_probe_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)cuda_stream>>>(x, out, n);
  return cudaGetLastError() == cudaSuccess ? ALERT_OK : ALERT_ERR_CUDA;
}

__global__ void erfc_rel_probe_kernel(const float* x, float* out, long long n) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = alert::erfc_rel(x[i]);
}

// The relatively accurate FP32 erfc of the max-accuracy tail ordering ->
// out[i] (device pointers): lets the tests bound its RELATIVE error.
int alert_probe_erfc_rel(const float* x, float* out, int64_t n, void* cuda_stream) {
  if (!x || !out || n < 0) return ALERT_ERR_INVALID_ARGUMENT;
  if (n == 0) return ALERT_OK;
  erfc_rel_probe_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)cuda_stream>>>(x, out, n);
  return cudaGetLastError() == cudaSuccess ? ALERT_OK : ALERT_ERR_CUDA;
}
