// Microbenchmark: FP32 FFMA / FFMA2 / FADD2 / mixed FADD2+FFMA2 and FP64 DFMA issue rates on sm_100a.
// Used to derive the "alu" roofline peak for DESIGN.md. Run: ./fp_rates
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
__global__ void k_ffma(float* out, float a, float b) {
  float c[8]; for (int i = 0; i < 8; ++i) c[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fmaf(c[i], a, b);
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += c[i]; out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma2(float* out, float a, float b) {
  float2 c[8]; for (int i = 0; i < 8; ++i) c[i] = make_float2(threadIdx.x * 1e-3f + i, i);
  float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = __ffma2_rn(c[i], a2, b2);
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += c[i].x + c[i].y; out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// the distance inner step: d = y - s (FADD2), acc = d*d + acc (FFMA2)
__global__ void k_dist2(float* out, float a, float b) {
  float2 y[8], acc[8]; for (int i = 0; i < 8; ++i) { y[i] = make_float2(threadIdx.x * 1e-3f + i, i); acc[i] = make_float2(0.f, 0.f); }
  float2 s2 = make_float2(a, b);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { float2 d = __fadd2_rn(y[i], s2); acc[i] = __ffma2_rn(d, d, acc[i]); }
    s2.x += 1e-7f;
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += acc[i].x + acc[i].y; out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dist1(float* out, float a, float b) {
  float y[8], acc[8]; for (int i = 0; i < 8; ++i) { y[i] = threadIdx.x * 1e-3f + i; acc[i] = 0.f; }
  float s1 = a;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { float d = y[i] - s1; acc[i] = fmaf(d, d, acc[i]); }
    s1 += 1e-7f;
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += acc[i]; out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dfma(double* out, double a, double b) {
  double c[8]; for (int i = 0; i < 8; ++i) c[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITERS / 8; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += c[i]; out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_clock(long long* out) {
  long long t0 = clock64(); 
  float c = threadIdx.x; for (int i = 0; i < 1 << 20; ++i) c = fmaf(c, 0.999f, 0.001f);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0 + (c > 1e30f);
}
template <class F> float timeit(F f) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(e0); for (int r = 0; r < 5; ++r) f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); return ms / 5;
}
int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("device %s SMs %d clockRate %d kHz\n", p.name, p.multiProcessorCount, clk_khz);
  int sms = p.multiProcessorCount, threads = 512, blocks = sms * 4;
  float* of; double* od; long long* oc;
  cudaMalloc(&of, sizeof(float) * blocks * threads); cudaMalloc(&od, sizeof(double) * blocks * threads);
  cudaMalloc(&oc, sizeof(long long) * sms);
  // measure effective SM clock: one block per SM, clock64 delta vs event time
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k_clock<<<sms, 32>>>(oc); cudaDeviceSynchronize();
  cudaEventRecord(e0); k_clock<<<sms, 32>>>(oc); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float msc; cudaEventElapsedTime(&msc, e0, e1); long long cyc; cudaMemcpy(&cyc, oc, 8, cudaMemcpyDeviceToHost);
  double ghz = cyc / (msc * 1e6);
  printf("effective SM clock (single-warp loop) %.3f GHz\n", ghz);
  double n_thr = (double)blocks * threads;
  float t;
  t = timeit([&] { k_ffma<<<blocks, threads>>>(of, 0.999f, 0.001f); });
  double ops = n_thr * ITERS * 8;  // FFMA lane-instructions
  printf("FFMA   : %.3f ms  %.2f T lane-FMA/s  (%.1f lane-FMA/clk/SM @%.3fGHz)\n", t, ops / t / 1e9, ops / t / 1e9 * 1e12 / (ghz * 1e9) / sms / 1e12 * 1e0 * 1, ghz);
  t = timeit([&] { k_ffma2<<<blocks, threads>>>(of, 0.999f, 0.001f); });
  ops = n_thr * ITERS * 8 * 2;
  printf("FFMA2  : %.3f ms  %.2f T lane-FMA/s  (%.1f lane-FMA/clk/SM)\n", t, ops / t / 1e9, ops / (t * 1e-3) / (ghz * 1e9) / sms);
  t = timeit([&] { k_dist2<<<blocks, threads>>>(of, 0.5f, 0.25f); });
  ops = n_thr * ITERS * 8 * 4;  // 2 FADD + 2 FFMA per float2 step = 4 lane ops
  printf("FADD2+FFMA2 dist: %.3f ms  %.2f T lane-op/s  (%.1f lane-op/clk/SM)  frame-updates %.2f T/s\n", t, ops / t / 1e9, ops / (t * 1e-3) / (ghz * 1e9) / sms, ops / 2 / t / 1e9);
  t = timeit([&] { k_dist1<<<blocks, threads>>>(of, 0.5f, 0.25f); });
  ops = n_thr * ITERS * 8 * 2;
  printf("FADD+FFMA dist : %.3f ms  %.2f T lane-op/s  (%.1f lane-op/clk/SM)  frame-updates %.2f T/s\n", t, ops / t / 1e9, ops / (t * 1e-3) / (ghz * 1e9) / sms, ops / 2 / t / 1e9);
  t = timeit([&] { k_dfma<<<blocks, threads>>>(od, 0.999, 0.001); });
  ops = n_thr * (ITERS / 8) * 8;
  printf("DFMA   : %.3f ms  %.3f T lane-DFMA/s (%.2f /clk/SM)\n", t, ops / t / 1e9, ops / (t * 1e-3) / (ghz * 1e9) / sms);
  // re-measure the clock after the load
  cudaEventRecord(e0); k_clock<<<sms, 32>>>(oc); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&msc, e0, e1); cudaMemcpy(&cyc, oc, 8, cudaMemcpyDeviceToHost);
  printf("effective SM clock after %.3f GHz\n", cyc / (msc * 1e6));
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
