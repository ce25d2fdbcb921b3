// tmem_bw.cu -- tensor-memory load/store throughput per SM with 32x32b
// register transfers (the large-bin kernel keeps per-frame state in TMEM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/tmem_bw tools/tmem_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kWarps = 16, kIters = 4096;

__global__ void __launch_bounds__(kWarps * 32, 1) tmem_kernel(unsigned* out, long long* cyc, int mode) {
  __shared__ unsigned base_s;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        unsigned(__cvta_generic_to_shared(&base_s))));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const unsigned base = base_s;
  const unsigned taddr = base + ((32u * (warp & 3)) << 16) + 128u * (warp >> 2);
  unsigned v[8];
  for (int k = 0; k < 8; ++k) v[k] = threadIdx.x + k;
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
  asm volatile("tcgen05.wait::st.sync.aligned;\n");
  __syncthreads();
  long long t0 = clock64();
  unsigned acc = 0;
  for (int i = 0; i < kIters; ++i) {
    const unsigned a = taddr + 8u * (i & 15);
    if (mode == 0) {
      unsigned r[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                     "=r"(r[7])
                   : "r"(a));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
      for (int k = 0; k < 8; ++k) acc += r[k];
    } else {
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(a),
                   "r"(v[0] + i), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]),
                   "r"(v[7]));
    }
  }
  if (mode != 0) asm volatile("tcgen05.wait::st.sync.aligned;\n");
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(base));
}

int main() {
  unsigned* out;
  long long* cyc;
  cudaMalloc(&out, 148 * kWarps * 32 * 4);
  cudaMalloc(&cyc, 148 * 8);
  for (int mode = 0; mode < 2; ++mode) {
    tmem_kernel<<<148, kWarps * 32>>>(out, cyc, mode);
    tmem_kernel<<<148, kWarps * 32>>>(out, cyc, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
      return 1;
    }
    long long c[148];
    cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < 148; ++i) mean += c[i] / 148.0;
    const double bytes = double(kWarps) * 32 * 8 * 4 * kIters;  // per SM
    printf("{\"mode\": \"%s\", \"cycles\": %.0f, \"bytes_per_cycle_per_sm\": %.1f}\n",
           mode == 0 ? "ld32x32b.x8+wait" : "st32x32b.x8", mean, bytes / mean);
  }
  return 0;
}
