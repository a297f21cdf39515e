// Measures sustained throughput of integer instruction classes on the GPU
// (development microbenchmark for the RNG: which pipe bounds mix64?).
#include <cstdio>
#include <cstdint>
#define N_ITER 4096
template <int OP>
__global__ void k(uint32_t* out, uint32_t seed) {
  uint32_t a0 = seed ^ threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, a4 = a0 * 11, a5 = a0 * 13, a6 = a0 * 17, a7 = a0 * 19;
  uint32_t c = seed | 1;
#pragma unroll 1
  for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (OP == 0) {  // LOP3 xor
        asm volatile("xor.b32 %0, %0, %1;" : "+r"(a0) : "r"(a1)); asm volatile("xor.b32 %0, %0, %1;" : "+r"(a1) : "r"(a2));
        asm volatile("xor.b32 %0, %0, %1;" : "+r"(a2) : "r"(a3)); asm volatile("xor.b32 %0, %0, %1;" : "+r"(a3) : "r"(a4));
        asm volatile("xor.b32 %0, %0, %1;" : "+r"(a4) : "r"(a5)); asm volatile("xor.b32 %0, %0, %1;" : "+r"(a5) : "r"(a6));
        asm volatile("xor.b32 %0, %0, %1;" : "+r"(a6) : "r"(a7)); asm volatile("xor.b32 %0, %0, %1;" : "+r"(a7) : "r"(a0));
      } else if (OP == 1) {  // SHF funnel
        asm volatile("shf.r.wrap.b32 %0, %0, %1, 7;" : "+r"(a0) : "r"(a1)); asm volatile("shf.r.wrap.b32 %0, %0, %1, 7;" : "+r"(a1) : "r"(a2));
        asm volatile("shf.r.wrap.b32 %0, %0, %1, 7;" : "+r"(a2) : "r"(a3)); asm volatile("shf.r.wrap.b32 %0, %0, %1, 7;" : "+r"(a3) : "r"(a4));
        asm volatile("shf.r.wrap.b32 %0, %0, %1, 7;" : "+r"(a4) : "r"(a5)); asm volatile("shf.r.wrap.b32 %0, %0, %1, 7;" : "+r"(a5) : "r"(a6));
        asm volatile("shf.r.wrap.b32 %0, %0, %1, 7;" : "+r"(a6) : "r"(a7)); asm volatile("shf.r.wrap.b32 %0, %0, %1, 7;" : "+r"(a7) : "r"(a0));
      } else if (OP == 2) {  // IMAD lo
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a0) : "r"(c), "r"(a1)); asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a1) : "r"(c), "r"(a2));
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a2) : "r"(c), "r"(a3)); asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a3) : "r"(c), "r"(a4));
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a4) : "r"(c), "r"(a5)); asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a5) : "r"(c), "r"(a6));
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a6) : "r"(c), "r"(a7)); asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a7) : "r"(c), "r"(a0));
      } else if (OP == 3) {  // IMAD.HI
        asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a0) : "r"(c), "r"(a1)); asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a1) : "r"(c), "r"(a2));
        asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a2) : "r"(c), "r"(a3)); asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a3) : "r"(c), "r"(a4));
        asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a4) : "r"(c), "r"(a5)); asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a5) : "r"(c), "r"(a6));
        asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a6) : "r"(c), "r"(a7)); asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a7) : "r"(c), "r"(a0));
      } else if (OP == 4) {  // IMAD.WIDE
        uint64_t w0, w1, w2, w3;
        asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(w0) : "r"(a0), "r"(c)); asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(w1) : "r"(a2), "r"(c));
        asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(w2) : "r"(a4), "r"(c)); asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(w3) : "r"(a6), "r"(c));
        a0 = uint32_t(w0 >> 32) ^ a1; a2 = uint32_t(w1 >> 32) ^ a3; a4 = uint32_t(w2 >> 32) ^ a5; a6 = uint32_t(w3 >> 32) ^ a7;
        a1 = uint32_t(w0); a3 = uint32_t(w1); a5 = uint32_t(w2); a7 = uint32_t(w3);
      } else if (OP == 6) {  // LEA.HI: b + (a >> 30) via lea.hi-friendly pattern
        a0 = (a1 >> 30) + a0; a1 = (a2 >> 30) + a1; a2 = (a3 >> 30) + a2; a3 = (a4 >> 30) + a3;
        a4 = (a5 >> 30) + a4; a5 = (a6 >> 30) + a5; a6 = (a7 >> 30) + a6; a7 = (a0 >> 30) + a7;
      } else if (OP == 7) {  // LEA: (a << 5) + b
        a0 = (a1 << 5) + a0; a1 = (a2 << 5) + a1; a2 = (a3 << 5) + a2; a3 = (a4 << 5) + a3;
        a4 = (a5 << 5) + a4; a5 = (a6 << 5) + a5; a6 = (a7 << 5) + a6; a7 = (a0 << 5) + a7;
      } else if (OP == 8) {  // DFMA throughput
        double d0 = a0, d1 = a1;
        asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d0) : "d"(d1));
        asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d1) : "d"(d0));
        a0 = uint32_t(__double_as_longlong(d0)); a1 = uint32_t(__double_as_longlong(d1));
      } else if (OP == 5) {  // IADD3 carry chain pairs (64-bit adds)
        asm volatile("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, %3;" : "+r"(a0), "+r"(a1) : "r"(a2), "r"(a3));
        asm volatile("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, %3;" : "+r"(a2), "+r"(a3) : "r"(a4), "r"(a5));
        asm volatile("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, %3;" : "+r"(a4), "+r"(a5) : "r"(a6), "r"(a7));
        asm volatile("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, %3;" : "+r"(a6), "+r"(a7) : "r"(a0), "r"(a1));
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7;
}
template <int OP>
void run(const char* name, int sms, uint32_t* out, int instr_per_iter) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256;
  k<OP><<<blocks, threads>>>(out, 1); cudaDeviceSynchronize();
  cudaEventRecord(e0);
  k<OP><<<blocks, threads>>>(out, 2);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double warp_instr = double(blocks) * threads / 32 * N_ITER * instr_per_iter;
  double cycles = ms * 1e-3 * clk * 1e3;
  printf("%-10s %8.3f ms  %.3f warp-instr/clk/SMSP\n", name, ms, warp_instr / (sms * 4) / cycles);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out; cudaMalloc(&out, sms * 8 * 256 * 4);
  run<0>("LOP3", sms, out, 32); run<1>("SHF", sms, out, 32); run<2>("IMAD", sms, out, 32);
  run<3>("IMAD.HI", sms, out, 32); run<4>("IMAD.WIDE", sms, out, 16 + 16); run<5>("IADD3x2", sms, out, 32);
  run<6>("LEA.HI?", sms, out, 32); run<7>("LEA?", sms, out, 32);
  return 0;
}
