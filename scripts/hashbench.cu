// Development microbenchmark: cost of the reference RNG key
// mix64(seed ^ mix64(b ^ mix64(i))) (util.hpp:14-29) under several sm_100a
// formulations, to pick K1's inline form.  Each variant writes an xor
// checksum so the work cannot be dead-code eliminated; all variants must
// print the same checksum.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hashbench hashbench.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t mix64_ref(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// 3-op 64x64 multiply by a constant: X = lo*ch + hi*cl, then
// (lo*cl) + (X << 32) with one IMAD.WIDE carrying a 64-bit addend
__device__ __forceinline__ void mul3(uint32_t& lo, uint32_t& hi, uint32_t cl, uint32_t ch) {
  uint32_t x;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(x) : "r"(hi), "r"(cl), "r"(lo * ch));
  uint64_t w;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(w) : "r"(lo), "r"(cl), "l"((uint64_t)x << 32));
  lo = uint32_t(w);
  hi = uint32_t(w >> 32);
}

template <int SHIFTMODE>
__device__ __forceinline__ void xs(uint32_t& lo, uint32_t& hi, uint32_t k) {
  const uint32_t f = __funnelshift_r(lo, hi, k);
  const uint32_t t = hi >> k;
  lo ^= f;
  hi ^= t;
}

__device__ __forceinline__ void mix_split(uint32_t& lo, uint32_t& hi) {
  asm("add.cc.u32 %0, %0, 0x7f4a7c15;\n\taddc.u32 %1, %1, 0x9e3779b9;" : "+r"(lo), "+r"(hi));
  xs<0>(lo, hi, 30);
  mul3(lo, hi, 0x1ce4e5b9u, 0xbf58476du);
  xs<0>(lo, hi, 27);
  mul3(lo, hi, 0x133111ebu, 0x94d049bbu);
  xs<0>(lo, hi, 31);
}

// hi word only of the final finalizer (lo of the last multiply unused)
__device__ __forceinline__ uint32_t mix_split_hi(uint32_t lo, uint32_t hi) {
  asm("add.cc.u32 %0, %0, 0x7f4a7c15;\n\taddc.u32 %1, %1, 0x9e3779b9;" : "+r"(lo), "+r"(hi));
  xs<0>(lo, hi, 30);
  mul3(lo, hi, 0x1ce4e5b9u, 0xbf58476du);
  xs<0>(lo, hi, 27);
  uint32_t x = lo * 0x94d049bbu;
  x = hi * 0x133111ebu + x;
  const uint32_t h = __umulhi(lo, 0x133111ebu) + x;
  return h ^ (h >> 31);
}

template <int V>
__global__ void k(uint64_t n, uint64_t seed, uint32_t B, unsigned long long* sink,
                  const unsigned long long* __restrict__ pre) {
  uint64_t acc = 0;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  const uint32_t sl = uint32_t(seed), sh = uint32_t(seed >> 32);
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += stride) {
    const uint32_t b = uint32_t(i) / B;
    if (V == 0) {
      acc ^= mix64_ref(seed ^ mix64_ref(b ^ mix64_ref(i))) >> 11;
    } else if (V == 1) {
      uint32_t lo = uint32_t(i), hi = 0;
      mix_split(lo, hi);
      lo ^= b;
      mix_split(lo, hi);
      lo ^= sl;
      hi ^= sh;
      mix_split(lo, hi);
      acc ^= ((uint64_t(hi) << 32) | lo) >> 11;
    } else if (V == 2) {  // hi word only (what the fast path needs)
      uint32_t lo = uint32_t(i), hi = 0;
      mix_split(lo, hi);
      lo ^= b;
      mix_split(lo, hi);
      acc ^= mix_split_hi(lo ^ sl, hi ^ sh) >> 9;
    } else if (V == 3) {  // prefix table + one finalizer (hi only)
      const unsigned long long K = __ldcs(pre + i);
      acc ^= mix_split_hi(uint32_t(K) ^ sl, uint32_t(K >> 32) ^ sh) >> 9;
    } else if (V == 4) {  // build the prefix table
      uint32_t lo = uint32_t(i), hi = 0;
      mix_split(lo, hi);
      lo ^= b;
      mix_split(lo, hi);
      reinterpret_cast<unsigned long long*>(const_cast<unsigned long long*>(pre))[i] =
          (uint64_t(hi) << 32) | lo;
    }
  }
  for (int o = 16; o > 0; o >>= 1) acc ^= __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicXor(sink, (unsigned long long)acc);
}

template <int V>
void run(const char* name, uint64_t n, unsigned long long* sink, unsigned long long* pre, int sms) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaMemset(sink, 0, 8);
  k<V><<<sms * 8, 256>>>(n, 42, 128, sink, pre);
  cudaDeviceSynchronize();
  cudaMemset(sink, 0, 8);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<V><<<sms * 8, 256>>>(n, 42, 128, sink, pre);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h;
  cudaMemcpy(&h, sink, 8, cudaMemcpyDeviceToHost);
  printf("%-28s %8.1f us   checksum %016llx\n", name, ms * 1e3 / 5, h);
}

int main() {
  const uint64_t n = 25557032;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long *sink, *pre;
  cudaMalloc(&sink, 8);
  cudaMalloc(&pre, n * 8);
  run<4>("build prefix table", n, sink, pre, sms);
  run<0>("v0 reference u64", n, sink, pre, sms);
  run<1>("v1 split, 3-op mul, SHF", n, sink, pre, sms);
  run<2>("v2 split, hi-only final", n, sink, pre, sms);
  run<3>("v3 prefix table + 1 final", n, sink, pre, sms);
  return 0;
}
