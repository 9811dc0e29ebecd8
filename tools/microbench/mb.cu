// Microbenchmarks that ground the K1 design on B200 (sm_100a):
// shared-memory atomic throughput (u32 add, u64 add, u64 CAS, f64 add = CAS loop),
// fp64 DFMA / DADD.RM / F2F.F64.F32 issue rates, and L2-resident streaming read bandwidth.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s at %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

template<int MODE>
__global__ void smem_atomics(unsigned long long* out, int iters) {
  extern __shared__ unsigned char sm[];
  unsigned int* u32 = (unsigned int*)sm;
  unsigned long long* u64 = (unsigned long long*)sm;
  double* f64 = (double*)sm;
  const int slots = 8192;
  for (int i = threadIdx.x; i < slots; i += blockDim.x) u64[i] = 0;
  __syncthreads();
  unsigned int h = threadIdx.x * 2654435761u + blockIdx.x;
  unsigned long long acc = 0;
  for (int it = 0; it < iters; ++it) {
    h = h * 1664525u + 1013904223u;
    int s = (h >> 8) & (slots - 1);
    if (MODE == 0) atomicAdd(&u32[s], 1u);
    else if (MODE == 1) atomicAdd(&u64[s], 3ull);
    else if (MODE == 2) acc += atomicCAS(&u64[s], 0ull, (unsigned long long)h);
    else if (MODE == 3) atomicAdd(&f64[s], 1.5);
    else if (MODE == 4) acc += u64[s];  // plain LDS.64 random
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = u64[7] + acc;
}

__global__ void fp64_rate(double* out, int iters, int mode) {
  double a = threadIdx.x * 1e-3, b = 1.0000001, c = 0.5, d = 0.25, e = 0.125, f = 2.0;
  float fa = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    if (mode == 0) {  // 4 independent DFMA chains
      a = fma(a, b, c); d = fma(d, b, c); e = fma(e, b, c); f = fma(f, b, c);
    } else if (mode == 1) {
      a = __dadd_rd(a, 6755399441055744.0); d = __dadd_rd(d, 3.0); e = __dadd_rd(e, 5.0); f = __dadd_rd(f, 7.0);
    } else {
      a += (double)fa; d += (double)(fa + 1.f); e += (double)(fa + 2.f); f += (double)(fa + 3.f);
      fa += 1.0f;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + d + e + f;
}

__global__ void l2_stream(const float4* __restrict__ p, int n, int reps, float* out) {
  float acc = 0.f;
  for (int r = 0; r < reps; ++r)
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      float4 v = __ldg(&p[i]);
      acc += v.x + v.y + v.z + v.w;
    }
  if (acc == 12345.f) out[blockIdx.x] = acc;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  printf("device %s sms %d clock %d kHz\n", prop.name, sms, prop.clockRate);
  unsigned long long* dout; CK(cudaMalloc(&dout, 1 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[] = {"u32 add", "u64 add", "u64 CAS", "f64 add (CAS loop)", "LDS.64 random"};
  for (int mode = 0; mode < 5; ++mode) {
    int iters = 4096, threads = 1024, blocks = sms * 2;
    void (*k)(unsigned long long*, int) = mode == 0 ? smem_atomics<0> : mode == 1 ? smem_atomics<1> : mode == 2 ? smem_atomics<2> : mode == 3 ? smem_atomics<3> : smem_atomics<4>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    k<<<blocks, threads, 65536>>>(dout, 16); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); k<<<blocks, threads, 65536>>>(dout, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * iters;
    printf("smem %-20s: %.3f Gop/s chip, %.3f lane-ops/clk/SM (at %.0f MHz)\n", names[mode], ops / ms / 1e6,
           ops / (ms * 1e-3) / sms / (prop.clockRate * 1e3), prop.clockRate / 1e3);
  }
  const char* fn[] = {"DFMA", "DADD.RM", "F2F.F64.F32+DADD"};
  double* dd; CK(cudaMalloc(&dd, sizeof(double) * sms * 8 * 1024));
  for (int mode = 0; mode < 3; ++mode) {
    int iters = 1 << 14, threads = 1024, blocks = sms * 2;
    fp64_rate<<<blocks, threads>>>(dd, 16, mode); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); fp64_rate<<<blocks, threads>>>(dd, iters, mode); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * iters * 4;
    printf("%-18s: %.2f Gop/s, %.2f lane-ops/clk/SM\n", fn[mode], ops / ms / 1e6, ops / (ms * 1e-3) / sms / (prop.clockRate * 1e3));
  }
  int n = 120000; float4* pts; CK(cudaMalloc(&pts, n * 16)); CK(cudaMemset(pts, 0, n * 16));
  float* fo; CK(cudaMalloc(&fo, 4096 * 4));
  for (int bpsm = 1; bpsm <= 4; bpsm *= 2) {
    int blocks = sms * bpsm, reps = 20;
    l2_stream<<<blocks, 1024 / bpsm>>>(pts, n, 2, fo); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); l2_stream<<<blocks, 1024 / bpsm>>>(pts, n, reps, fo); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double bytes = (double)blocks * reps * n * 16;
    printf("L2 stream 1.92MB x %d CTAs: %.1f GB/s (%.2f B/clk/SM)\n", blocks, bytes / ms / 1e6, bytes / (ms * 1e-3) / sms / (prop.clockRate * 1e3));
  }
  return 0;
}
