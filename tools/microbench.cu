// tools/microbench.cu -- B200 latency / throughput probes for the operations
// the simulate kernel is built from (fp64 add / max, warp shuffles, int64
// add).  Not part of the product; the numbers feed DESIGN.md's cost model
// and the ALU roofline peak.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb tools/microbench.cu && ./mb
#include <cstdio>
#include <cuda_runtime.h>

#define N_CHAIN 4096

__global__ void lat_dadd(double* out, long long* cyc, double a) {
  double x = threadIdx.x * 1e-3;
  long long t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N_CHAIN; i++) x = __dadd_rn(x, a);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void lat_dmax(double* out, long long* cyc, double a) {
  double x = threadIdx.x * 1e-3, y = a;
  long long t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N_CHAIN; i++) { x = fmax(x, y); y = y + 0.0; x = -x; }
  long long t1 = clock64();
  out[threadIdx.x] = x + y;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void lat_fadd(float* out, long long* cyc, float a) {
  float x = threadIdx.x * 1e-3f;
  long long t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N_CHAIN; i++) x = __fadd_rn(x, a);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void lat_i64(long long* out, long long* cyc, long long a) {
  long long x = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N_CHAIN; i++) x = x + a;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void lat_shfl(double* out, long long* cyc) {
  double x = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N_CHAIN / 8; i++) x = __shfl_xor_sync(0xffffffffu, x, 1);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void lat_frnd(double* out, long long* cyc, double a) {
  double x = threadIdx.x * 1e-3 + a;
  long long t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N_CHAIN; i++) x = floor(x) + 0.75;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

// throughput: 8 independent chains per thread, many warps
__global__ void tput_dadd(double* out, double a, int iters) {
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; j++) x[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++) x[j] = __dadd_rn(x[j], a);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; j++) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void tput_iadd(int* out, int a, int iters) {
  int x[8];
#pragma unroll
  for (int j = 0; j < 8; j++) x[j] = threadIdx.x + j;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++) x[j] = x[j] * 3 + a;
  }
  int s = 0;
#pragma unroll
  for (int j = 0; j < 8; j++) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double *d;
  float* f;
  long long *c, *l;
  int* iv;
  cudaMalloc(&d, 1 << 26);
  cudaMalloc(&f, 1 << 20);
  cudaMalloc(&l, 1 << 20);
  cudaMalloc(&c, 8);
  cudaMalloc(&iv, 1 << 26);
  long long h;
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"device\": \"%s\", \"sms\": %d, \"clock_mhz\": %.0f", prop.name, prop.multiProcessorCount,
         clk_khz / 1e3);
  auto lat = [&](const char* name, double per) { printf(", \"%s_cycles\": %.2f", name, per); };
  for (int rep = 0; rep < 2; rep++) {
    lat_dadd<<<1, 32>>>(d, c, 1e-9); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (rep) lat("dadd_latency", (double)h / N_CHAIN);
    lat_fadd<<<1, 32>>>(f, c, 1e-9f); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (rep) lat("fadd_latency", (double)h / N_CHAIN);
    lat_i64<<<1, 32>>>(l, c, 3); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (rep) lat("iadd64_latency", (double)h / N_CHAIN);
    lat_shfl<<<1, 32>>>(d, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (rep) lat("shfl_f64_latency", (double)h / (N_CHAIN / 8));
    lat_dmax<<<1, 32>>>(d, c, 0.5); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (rep) lat("dmax_neg_dadd_chain", (double)h / N_CHAIN);
    lat_frnd<<<1, 32>>>(d, c, 0.5); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (rep) lat("floor_dadd_chain", (double)h / N_CHAIN);
  }
  // throughput
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = prop.multiProcessorCount * 8, threads = 256, iters = 4096;
  tput_dadd<<<blocks, threads>>>(d, 1e-9, 16);
  cudaEventRecord(e0);
  tput_dadd<<<blocks, threads>>>(d, 1e-9, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double dadds = (double)blocks * threads * iters * 8;
  printf(", \"dadd_per_s\": %.4g", dadds / (ms * 1e-3));
  tput_iadd<<<blocks, threads>>>(iv, 1, 16);
  cudaEventRecord(e0);
  tput_iadd<<<blocks, threads>>>(iv, 1, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf(", \"imad_per_s\": %.4g", dadds / (ms * 1e-3));
  printf("}\n");
  return 0;
}
