// Microbenchmark: FP32 pipe throughput on sm_100a for FFMA (3-reg), FFMA2
// (packed f32x2), FMUL and FADD, full chip, many warps.  Prints lane-ops/clk/SM.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void kern(float* out, float s, int iters) {
  float a0 = threadIdx.x * 1e-3f, a1 = a0 + 1.f, a2 = a0 + 2.f, a3 = a0 + 3.f;
  float a4 = a0 + 4.f, a5 = a0 + 5.f, a6 = a0 + 6.f, a7 = a0 + 7.f;
  float b = s, c = s * 0.5f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (MODE == 0) {  // FFMA 3-reg: 8 independent chains
        a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c);
        a4 = fmaf(a4, b, c); a5 = fmaf(a5, b, c); a6 = fmaf(a6, b, c); a7 = fmaf(a7, b, c);
      } else if (MODE == 1) {  // FFMA2: 4 packed chains == 8 lanes of work
        unsigned long long x0, x1, x2, x3, bb, cc;
        asm("mov.b64 %0, {%1,%2};" : "=l"(x0) : "f"(a0), "f"(a1));
        asm("mov.b64 %0, {%1,%2};" : "=l"(x1) : "f"(a2), "f"(a3));
        asm("mov.b64 %0, {%1,%2};" : "=l"(x2) : "f"(a4), "f"(a5));
        asm("mov.b64 %0, {%1,%2};" : "=l"(x3) : "f"(a6), "f"(a7));
        asm("mov.b64 %0, {%1,%2};" : "=l"(bb) : "f"(b), "f"(b));
        asm("mov.b64 %0, {%1,%2};" : "=l"(cc) : "f"(c), "f"(c));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x0) : "l"(bb), "l"(cc));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x1) : "l"(bb), "l"(cc));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x2) : "l"(bb), "l"(cc));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x3) : "l"(bb), "l"(cc));
        asm("mov.b64 {%0,%1}, %2;" : "=f"(a0), "=f"(a1) : "l"(x0));
        asm("mov.b64 {%0,%1}, %2;" : "=f"(a2), "=f"(a3) : "l"(x1));
        asm("mov.b64 {%0,%1}, %2;" : "=f"(a4), "=f"(a5) : "l"(x2));
        asm("mov.b64 {%0,%1}, %2;" : "=f"(a6), "=f"(a7) : "l"(x3));
      } else if (MODE == 4 || MODE == 5) {
        // mixed: packed chains (a0..a3 as 2 pairs) and scalar chains (a4..a7);
        // MODE 4: 1 FFMA2 : 1 FFMA per pair of chains, MODE 5: 1 FFMA2 : 2 FFMA
        unsigned long long x0, x1, bb, cc;
        asm("mov.b64 %0, {%1,%2};" : "=l"(x0) : "f"(a0), "f"(a1));
        asm("mov.b64 %0, {%1,%2};" : "=l"(x1) : "f"(a2), "f"(a3));
        asm("mov.b64 %0, {%1,%2};" : "=l"(bb) : "f"(b), "f"(b));
        asm("mov.b64 %0, {%1,%2};" : "=l"(cc) : "f"(c), "f"(c));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x0) : "l"(bb), "l"(cc));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x1) : "l"(bb), "l"(cc));
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a4) : "f"(b), "f"(c));
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a5) : "f"(b), "f"(c));
        if (MODE == 5) {
          asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a6) : "f"(b), "f"(c));
          asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a7) : "f"(b), "f"(c));
        }
        asm("mov.b64 {%0,%1}, %2;" : "=f"(a0), "=f"(a1) : "l"(x0));
        asm("mov.b64 {%0,%1}, %2;" : "=f"(a2), "=f"(a3) : "l"(x1));
      } else if (MODE == 2) {  // FMUL
        a0 = a0 * b; a1 = a1 * b; a2 = a2 * b; a3 = a3 * b;
        a4 = a4 * b; a5 = a5 * b; a6 = a6 * b; a7 = a7 * b;
      } else {  // FADD
        a0 = a0 + b; a1 = a1 + b; a2 = a2 + b; a3 = a3 + b;
        a4 = a4 + b; a5 = a5 + b; a6 = a6 + b; a7 = a7 + b;
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

template <int MODE>
void run(const char* name, float* out, int sms, int clk_khz) {
  const int iters = 4096, blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<MODE><<<blocks, threads>>>(out, 0.999f, 16);
  cudaEventRecord(e0);
  kern<MODE><<<blocks, threads>>>(out, 0.999f, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  // lane-ops per inner step: 8 chains (modes 0-3), 4 packed + 2 scalar
  // (mode 4), 4 packed + 4 scalar (mode 5)
  const double per = MODE == 4 ? 6.0 : 8.0;
  const double lane_ops = (double)blocks * threads * iters * 16 * per;
  const double warp_instr = (double)blocks * threads * iters * 16 / 32 *
                            (MODE == 1 ? 4.0 : MODE == 4 ? 4.0 : MODE == 5 ? 6.0 : 8.0);
  const double clks = ms * 1e-3 * clk_khz * 1e3;
  printf("%-6s %8.3f ms  lane-ops/s %7.2f T  lane-ops/clk/SM %6.1f  warp-instr/clk/SMSP %5.2f\n",
         name, ms, lane_ops / (ms * 1e-3) / 1e12, lane_ops / clks / sms, warp_instr / clks / sms / 4);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, (size_t)p.multiProcessorCount * 8 * 256 * 4);
  printf("%s SMs=%d clk=%d kHz (nominal max; actual may differ)\n", p.name, p.multiProcessorCount, clk);
  run<0>("FFMA", out, p.multiProcessorCount, clk);
  run<1>("FFMA2", out, p.multiProcessorCount, clk);
  run<2>("FMUL", out, p.multiProcessorCount, clk);
  run<3>("FADD", out, p.multiProcessorCount, clk);
  run<4>("MIX11", out, p.multiProcessorCount, clk);
  run<5>("MIX12", out, p.multiProcessorCount, clk);
  return 0;
}
