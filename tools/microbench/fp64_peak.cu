// FP64 pipe microbenchmark for B200 (sm_100a): DFMA and DMMA throughput, DFMA latency.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

template<int CH>
__global__ void dfma_tput(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dfma_lat(double* out, int iters, double a, double b, long long* cyc) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void dmma884_tput(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[4][2];
#pragma unroll
  for (int t = 0; t < 4; ++t) { c[t][0] = 0; c[t][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 4; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma16816_tput(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int t = 0; t < 8; ++t) a[t] = threadIdx.x * 1e-3 + t;
#pragma unroll
  for (int t = 0; t < 4; ++t) b[t] = 1.0 + t * 1e-4;
  double c[2][4];
#pragma unroll
  for (int t = 0; t < 2; ++t) for (int q = 0; q < 4; ++q) c[t][q] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 2; ++t)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 2; ++t) for (int q = 0; q < 4; ++q) s += c[t][q];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void smem_lat(double* out, int iters, long long* cyc) {
  __shared__ int idx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i + 1) & 1023;
  __syncthreads();
  int p = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) p = idx[p];
  long long t1 = clock64();
  out[threadIdx.x] = p;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int clk; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  printf("SMs %d clock(kHz) %d\n", sms, clk);
  double* out; CK(cudaMalloc(&out, sizeof(double) * 148 * 64 * 1024));
  long long* cyc; CK(cudaMalloc(&cyc, sizeof(long long)));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // DFMA throughput
  for (int threads : {256, 512, 1024}) {
    int blocks = sms * (2048 / threads);
    int iters = 4096;
    dfma_tput<8><<<blocks, threads>>>(out, 16, 1.000001, 1e-7);
    cudaEventRecord(e0);
    dfma_tput<8><<<blocks, threads>>>(out, iters, 1.000001, 1e-7);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * iters * (double)blocks * threads;
    printf("DFMA tput threads=%d: %.2f TFLOP/s\n", threads, flops / ms / 1e9);
  }
  {
    int blocks = sms * 8, threads = 256, iters = 4096;
    dmma884_tput<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0);
    dmma884_tput<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 4 * (double)iters * blocks * (threads / 32);
    printf("DMMA m8n8k4 tput: %.2f TFLOP/s\n", flops / ms / 1e9);
  }
  {
    int blocks = sms * 8, threads = 256, iters = 1024;
    dmma16816_tput<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0);
    dmma16816_tput<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * 8 * 16 * 2 * (double)iters * blocks * (threads / 32);
    printf("DMMA m16n8k16 tput: %.2f TFLOP/s\n", flops / ms / 1e9);
  }
  {
    long long h;
    dfma_lat<<<1, 32>>>(out, 1024, 1.000001, 1e-7, cyc);
    CK(cudaDeviceSynchronize());
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DFMA latency: %.2f cycles\n", h / 1024.0);
    smem_lat<<<1, 32>>>(out, 1024, cyc);
    CK(cudaDeviceSynchronize());
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("LDS (int) dependent latency: %.2f cycles\n", h / 1024.0);
  }
  return 0;
}
