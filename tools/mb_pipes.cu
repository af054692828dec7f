// Pipe-throughput microbenchmark (B200): FP64 add / compare, 64-bit integer
// max via ISETP+SEL vs predicated moves, int32 ALU vs IMAD.  Used to choose
// the arithmetic of the schedule kernel.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define N_ITER 4096
__global__ void k_dadd(double *out, double a) {
  double x[8];
  for (int j = 0; j < 8; j++) x[j] = threadIdx.x + j;
  for (int i = 0; i < N_ITER; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) x[j] = x[j] + a;
  double s = 0; for (int j = 0; j < 8; j++) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dmax(double *out, double a) {   // DSETP + select
  double x[8], y = a;
  for (int j = 0; j < 8; j++) x[j] = threadIdx.x + j;
  for (int i = 0; i < N_ITER; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++) x[j] = (y > x[j]) ? y : x[j];
    y = y + 1.0;
  }
  double s = 0; for (int j = 0; j < 8; j++) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_u64max_sel(uint64_t *out, uint64_t a) {
  uint64_t x[8], y = a;
  for (int j = 0; j < 8; j++) x[j] = threadIdx.x + j;
  for (int i = 0; i < N_ITER; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++) x[j] = (y > x[j]) ? y : x[j];
    y += 3;
  }
  uint64_t s = 0; for (int j = 0; j < 8; j++) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__device__ __forceinline__ uint64_t max_pred(uint64_t x, uint64_t y) {
  uint64_t r;
  asm("{\n .reg .pred p;\n .reg .b32 xl, xh, yl, yh;\n mov.b64 {xl, xh}, %1;\n mov.b64 {yl, yh}, %2;\n"
      " setp.gt.u64 p, %2, %1;\n @p mov.b32 xl, yl;\n @p mov.b32 xh, yh;\n mov.b64 %0, {xl, xh};\n}"
      : "=l"(r) : "l"(x), "l"(y));
  return r;
}
__global__ void k_u64max_pred(uint64_t *out, uint64_t a) {
  uint64_t x[8], y = a;
  for (int j = 0; j < 8; j++) x[j] = threadIdx.x + j;
  for (int i = 0; i < N_ITER; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++) x[j] = max_pred(x[j], y);
    y += 3;
  }
  uint64_t s = 0; for (int j = 0; j < 8; j++) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__device__ __forceinline__ uint64_t max_fsel(uint64_t x, uint64_t y) {
  uint64_t r;
  asm("{\n .reg .pred p;\n .reg .f32 xl, xh, yl, yh;\n mov.b64 {xl, xh}, %1;\n mov.b64 {yl, yh}, %2;\n"
      " setp.gt.u64 p, %2, %1;\n selp.f32 xl, yl, xl, p;\n selp.f32 xh, yh, xh, p;\n mov.b64 %0, {xl, xh};\n}"
      : "=l"(r) : "l"(x), "l"(y));
  return r;
}
__global__ void k_u64max_fsel(uint64_t *out, uint64_t a) {
  uint64_t x[8], y = a;
  for (int j = 0; j < 8; j++) x[j] = threadIdx.x + j;
  for (int i = 0; i < N_ITER; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++) x[j] = max_fsel(x[j], y);
    y += 3;
  }
  uint64_t s = 0; for (int j = 0; j < 8; j++) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_i2f64(double *out, uint32_t a) {   // I2F.F64.U32
  double x[8];
  uint32_t u[8];
  for (int j = 0; j < 8; j++) { x[j] = 0; u[j] = threadIdx.x + j; }
  for (int i = 0; i < N_ITER; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) { x[j] += (double)(u[j] & 1u); u[j] += a; }
  double s = 0; for (int j = 0; j < 8; j++) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dfma(double *out, double a) {
  double x[8];
  for (int j = 0; j < 8; j++) x[j] = threadIdx.x + j;
  for (int i = 0; i < N_ITER; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) x[j] = __fma_rn(x[j], a, 1.0);
  double s = 0; for (int j = 0; j < 8; j++) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_alu(uint32_t *out, uint32_t a) {   // LOP3/IADD3 only
  uint32_t x[8];
  for (int j = 0; j < 8; j++) x[j] = threadIdx.x + j;
  for (int i = 0; i < N_ITER; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) x[j] = (x[j] ^ a) + (x[j] >> 3);
  uint32_t s = 0; for (int j = 0; j < 8; j++) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_imad(uint32_t *out, uint32_t a) {  // IMAD only
  uint32_t x[8];
  for (int j = 0; j < 8; j++) x[j] = threadIdx.x + j;
  for (int i = 0; i < N_ITER; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) x[j] = x[j] * 3u + a;
  uint32_t s = 0; for (int j = 0; j < 8; j++) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class F>
static void run(const char *name, F launch, double ops_per_thread, int blocks, int thr) {
  cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
  launch(); cudaDeviceSynchronize();
  cudaEventRecord(s); launch(); cudaEventRecord(e); cudaEventSynchronize(e);
  float ms; cudaEventElapsedTime(&ms, s, e);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double per_s = ops_per_thread * blocks * thr / (ms * 1e-3);
  printf("%-28s %8.3f ms  %7.2f Gop/s  %6.1f ops/clk/SM (at %d MHz)\n", name, ms, per_s / 1e9,
         per_s / sms / (clk * 1e3), clk / 1000);
}

int main() {
  void *d; cudaMalloc(&d, 1 << 26);
  int blocks = 148 * 8, thr = 256;
  double n = (double)N_ITER * 8;
  run("DADD", [&] { k_dadd<<<blocks, thr>>>((double *)d, 1.0); }, n, blocks, thr);
  run("double max (DSETP+sel)", [&] { k_dmax<<<blocks, thr>>>((double *)d, 1.0); }, n, blocks, thr);
  run("u64 max (ISETP+SEL)", [&] { k_u64max_sel<<<blocks, thr>>>((uint64_t *)d, 1); }, n, blocks, thr);
  run("u64 max (ISETP+@P MOV)", [&] { k_u64max_pred<<<blocks, thr>>>((uint64_t *)d, 1); }, n, blocks, thr);
  run("u64 max (ISETP+FSEL)", [&] { k_u64max_fsel<<<blocks, thr>>>((uint64_t *)d, 1); }, n, blocks, thr);
  run("I2F.F64.U32 + DADD + IADD", [&] { k_i2f64<<<blocks, thr>>>((double *)d, 3); }, n, blocks, thr);
  run("DFMA", [&] { k_dfma<<<blocks, thr>>>((double *)d, 0.5); }, n, blocks, thr);
  run("int32 xor+shift+add (ALU)", [&] { k_alu<<<blocks, thr>>>((uint32_t *)d, 7); }, n, blocks, thr);
  run("int32 IMAD (FMA pipe)", [&] { k_imad<<<blocks, thr>>>((uint32_t *)d, 7); }, n, blocks, thr);
  return 0;
}
