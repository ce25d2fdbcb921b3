// fp32_peak.cu -- measured FP32 CUDA-core peak on this B200 (the c3 roofline
// denominator) plus the cluster-placement numbers the large-bin fit kernel is
// sized by.  Build + run (GPU box):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/fp32_peak tools/fp32_peak.cu
//   build/fp32_peak
// Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      return 1;                                                                     \
    }                                                                               \
  } while (0)

constexpr int kIters = 4096;

// 3-register FFMA: 16 independent chains per thread.
__global__ void __launch_bounds__(256) ffma_kernel(float* out, float a, float b) {
  float v[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = threadIdx.x * 1e-3f + k;
  float c = a + threadIdx.x * 1e-7f, d = b - threadIdx.x * 1e-7f;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = fmaf(v[k], c, d);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += v[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Packed FFMA2 (fma.rn.f32x2): 16 independent float2 chains per thread.
__global__ void __launch_bounds__(256) ffma2_kernel(float* out, float a, float b) {
  float2 v[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = make_float2(threadIdx.x * 1e-3f + k, k - threadIdx.x * 1e-3f);
  const float2 c = make_float2(a + threadIdx.x * 1e-7f, a - threadIdx.x * 1e-7f);
  const float2 d = make_float2(b, -b);
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = __ffma2_rn(v[k], c, d);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += v[k].x + v[k].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// MUFU.RCP throughput.
__global__ void __launch_bounds__(256) rcp_kernel(float* out, float a) {
  float v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = a + threadIdx.x * 1e-3f + k;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(v[k]));
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += v[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void cluster_probe(int* out) {
  extern __shared__ int sm[];
  sm[threadIdx.x] = threadIdx.x;
  if (threadIdx.x == 0) out[blockIdx.x] = sm[0];
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  const int blocks = sms * 8, threads = 256;
  float* out;
  CK(cudaMalloc(&out, sizeof(float) * blocks * threads));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto time_it = [&](auto launch) {
    for (int w = 0; w < 3; ++w) launch();
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    return best;
  };
  const double lanes = double(blocks) * threads;
  const float t1 = time_it([&] { ffma_kernel<<<blocks, threads>>>(out, 0.999f, 1e-3f); });
  const float t2 = time_it([&] { ffma2_kernel<<<blocks, threads>>>(out, 0.999f, 1e-3f); });
  const float t3 = time_it([&] { rcp_kernel<<<blocks, threads>>>(out, 1.5f); });
  CK(cudaGetLastError());
  const double ffma_tf = lanes * kIters * 16 * 2 / (t1 * 1e-3) / 1e12;
  const double ffma2_tf = lanes * kIters * 32 * 2 / (t2 * 1e-3) / 1e12;
  const double rcp_g = lanes * kIters * 8 / (t3 * 1e-3) / 1e9;
  // Max co-resident clusters for a 1-CTA-per-SM shared-memory footprint.
  const int smem = 220 * 1024;
  CK(cudaFuncSetAttribute(cluster_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(cluster_probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  int ncl[9] = {0};
  for (int c = 1; c <= 8; ++c) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(c * 64);
    cfg.blockDim = dim3(448);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaOccupancyMaxActiveClusters(&ncl[c], cluster_probe, &cfg));
  }
  printf("{\"sms\": %d, \"clock_khz\": %d, \"ffma_tflops\": %.2f, \"ffma2_tflops\": %.2f, "
         "\"rcp_gops\": %.1f, \"ffma_ms\": %.3f, \"ffma2_ms\": %.3f, \"max_active_clusters_220KB\": "
         "{\"1\": %d, \"2\": %d, \"3\": %d, \"4\": %d, \"5\": %d, \"6\": %d, \"7\": %d, \"8\": %d}}\n",
         sms, clk, ffma_tf, ffma2_tf, rcp_g, t1, t2, ncl[1], ncl[2], ncl[3], ncl[4], ncl[5], ncl[6],
         ncl[7], ncl[8]);
  return 0;
}
