// gcx_stats.cu — K4: device statistics for the layer-wise adaptive bit-width
// selector (/root/reference/proj/src/adaptive.cpp:21-97, :390-415).
//
//   gcx_stats_accumulate  sum[i] += (double)v[i]  (StatsCollector::add; the
//                         per-element add order is the step order, so the
//                         window sums are bit-identical to the reference)
//   gcx_stats_reduce      l2^2 = sum sum[i]^2 and the top-q sum of squares
//                         (StatsCollector::stats; keep = max(1, ceil(q n)))
//   gcx_stats_snapshot    (float)sum[i]           (StatsCollector::snapshots)
//   gcx_sq_error          sum (double(a)-double(b))^2   (plan_error)
// The reductions use a fixed-shape tree, so they are deterministic run to run
// but not in the reference's sequential order: tolerance parity (the
// reference's own top-q order is implementation-defined, nth_element).
#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "gcx.h"

namespace {

constexpr int kThreads = 256;
constexpr int kBlocks = 592;  // 148 SMs x 4

thread_local std::string g_err2;

__global__ void k_accumulate(double* __restrict__ sum, const float* __restrict__ v, uint64_t n,
                             unsigned int* __restrict__ nonfinite) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  const uint64_t t0 = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  uint64_t head = 0;
  if (((reinterpret_cast<uintptr_t>(v) | reinterpret_cast<uintptr_t>(sum)) & 15u) == 0) {
    // 16-byte accesses: one float4 of the gradient, two double2 of the sums
    const uint64_t n4 = n >> 2;
    const float4* v4 = reinterpret_cast<const float4*>(v);
    double2* s2 = reinterpret_cast<double2*>(sum);
    for (uint64_t q = t0; q < n4; q += stride) {
      const float4 x = __ldcs(v4 + q);
      double2 a = s2[2 * q], b = s2[2 * q + 1];
      if (!(isfinite(x.x) && isfinite(x.y) && isfinite(x.z) && isfinite(x.w)))
        atomicOr(nonfinite, 1u);
      a.x = __dadd_rn(a.x, double(x.x));
      a.y = __dadd_rn(a.y, double(x.y));
      b.x = __dadd_rn(b.x, double(x.z));
      b.y = __dadd_rn(b.y, double(x.w));
      s2[2 * q] = a;
      s2[2 * q + 1] = b;
    }
    head = n4 << 2;
  }
  for (uint64_t i = head + t0; i < n; i += stride) {
    const float x = v[i];
    if (!isfinite(x)) atomicOr(nonfinite, 1u);
    sum[i] = __dadd_rn(sum[i], double(x));
  }
}

__global__ void k_snapshot(const double* __restrict__ sum, float* __restrict__ out, uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = __double2float_rn(sum[i]);
}

// squares as order-preserving u64 keys (non-negative doubles)
__global__ void k_square_keys(const double* __restrict__ sum, unsigned long long* __restrict__ keys,
                              uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const double s = sum[i];
    keys[i] = __double_as_longlong(__dmul_rn(s, s));
  }
}

__device__ __forceinline__ double block_reduce(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  v = threadIdx.x < blockDim.x / 32 ? sh[threadIdx.x] : 0.0;
  if (wid == 0) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  }
  return v;
}

// partial[block] = sum over its grid-stride range of keys-as-doubles
// (first `count` keys) or of sum^2 (when keys == nullptr)
__global__ void k_sum_squares(const double* __restrict__ sum, const unsigned long long* keys,
                              uint64_t count, double* __restrict__ partial) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
       i += uint64_t(gridDim.x) * blockDim.x) {
    if (keys) {
      acc += __longlong_as_double(keys[i]);
    } else {
      const double s = sum[i];
      acc = __dadd_rn(acc, __dmul_rn(s, s));  // squared[i], then total += (adaptive.cpp:64-67)
    }
  }
  acc = block_reduce(acc, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

__global__ void k_sq_error(const float* __restrict__ a, const float* __restrict__ b, uint64_t n,
                           double* __restrict__ partial) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const double e = __dsub_rn(double(a[i]), double(b[i]));
    acc = __fma_rn(e, e, acc);
  }
  acc = block_reduce(acc, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

// mean over nodes in node order (engine.cpp:270-278): stack holds nodes rows
__global__ void k_mean_nodes(const float* __restrict__ stack, uint32_t nodes, uint64_t n,
                             float* __restrict__ out) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    float m = stack[i];
    for (uint32_t k = 1; k < nodes; ++k) m = __fadd_rn(m, stack[uint64_t(k) * n + i]);
    out[i] = __fdiv_rn(m, float(nodes));
  }
}

__global__ void k_final_sum(const double* __restrict__ partial, int n, double* out) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += partial[i];
  acc = block_reduce(acc, sh);
  if (threadIdx.x == 0) *out = acc;
}

int launch_check(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_err2 = std::string(where) + ": " + cudaGetErrorString(e);
    return GCX_E_CUDA;
  }
  return GCX_OK;
}

uint32_t grid(uint64_t n) {
  const uint64_t g = (n + kThreads - 1) / kThreads;
  return uint32_t(g < 4096 ? (g ? g : 1) : 4096);
}

// ---------------------------------------------------------------------------
// TopK + error feedback (codec.cpp:158-214): acc = v + residual; keep the k
// largest |acc| (ties to the lower index) in increasing index order; residual
// = acc with the kept entries zeroed.  The selection order is a total order on
// the 64-bit key (|acc| bits << 32) | (2^32 - 1 - i): |acc| as unsigned bits
// is monotone for non-negative floats, and the complemented index makes the
// lower index win a tie; a descending radix sort of the keys gives exactly the
// reference's nth_element partition.
// ---------------------------------------------------------------------------
__global__ void k_topk_acc(const float* __restrict__ v, float* __restrict__ residual, uint64_t n,
                           unsigned long long* __restrict__ keys,
                           unsigned long long* __restrict__ bad) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const float x = v[i];
    if (!isfinite(x)) atomicMin(bad, (unsigned long long)i);
    const float a = __fadd_rn(x, residual[i]);
    residual[i] = a;
    const uint32_t mag = __float_as_uint(a) & 0x7FFFFFFFu;
    keys[i] = (unsigned long long)mag << 32 | (0xFFFFFFFFu - uint32_t(i));
  }
}

// the k winners' indices (from the sorted keys), for the index sort
__global__ void k_topk_idx(const unsigned long long* __restrict__ sorted, uint64_t k,
                           uint32_t* __restrict__ idx) {
  for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < k;
       j += uint64_t(gridDim.x) * blockDim.x)
    idx[j] = 0xFFFFFFFFu - uint32_t(sorted[j]);
}

__global__ void k_topk_take(const uint32_t* __restrict__ idx, uint64_t k, float* __restrict__ residual,
                            float* __restrict__ val) {
  for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < k;
       j += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t i = idx[j];
    val[j] = residual[i];
    residual[i] = 0.0f;
  }
}

// dense[i] = 0, then dense[idx[j]] = val[j] (topk_decompress)
__global__ void k_zero(float* __restrict__ x, uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    x[i] = 0.0f;
}

__global__ void k_scatter(const uint32_t* __restrict__ idx, const float* __restrict__ val,
                          uint64_t k, float* __restrict__ dense) {
  for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < k;
       j += uint64_t(gridDim.x) * blockDim.x)
    dense[idx[j]] = val[j];
}

}  // namespace

extern "C" {

uint64_t gcx_topk_scratch_bytes(uint64_t n) {
  size_t t1 = 0, t2 = 0;
  const int m = int(n > 0 ? n : 1);
  cub::DeviceRadixSort::SortKeysDescending(nullptr, t1, (unsigned long long*)nullptr,
                                           (unsigned long long*)nullptr, m);
  cub::DeviceRadixSort::SortKeys(nullptr, t2, (uint32_t*)nullptr, (uint32_t*)nullptr, m);
  return 2 * 8 * n + 2 * 4 * n + (t1 > t2 ? t1 : t2) + 512;
}

int gcx_topk_compress(const float* v, uint64_t n, uint64_t k, float* residual, uint32_t* idx_out,
                      float* val_out, void* scratch, uint64_t scratch_bytes,
                      unsigned long long* bad, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (k < 1 || k > n) {
    g_err2 = "topk k must be in [1, length], got " + std::to_string(k);
    return GCX_E_INVALID;
  }
  if (n >= (1ull << 31)) {
    g_err2 = "gcx_topk_compress: length must be below 2^31";
    return GCX_E_INVALID;
  }
  if (scratch_bytes < gcx_topk_scratch_bytes(n)) {
    g_err2 = "gcx_topk_compress: scratch too small";
    return GCX_E_INVALID;
  }
  auto* keys = static_cast<unsigned long long*>(scratch);
  auto* sorted = keys + n;
  auto* idx = reinterpret_cast<uint32_t*>(sorted + n);
  const uintptr_t t0 = (reinterpret_cast<uintptr_t>(idx + 2 * n) + 255) & ~uintptr_t(255);
  void* temp = reinterpret_cast<void*>(t0);
  size_t temp_bytes = scratch_bytes - (t0 - reinterpret_cast<uintptr_t>(scratch));
  k_topk_acc<<<grid(n), kThreads, 0, st>>>(v, residual, n, keys, bad);
  cub::DeviceRadixSort::SortKeysDescending(temp, temp_bytes, keys, sorted, int(n), 0, 64, st);
  k_topk_idx<<<grid(k), kThreads, 0, st>>>(sorted, k, idx);
  cub::DeviceRadixSort::SortKeys(temp, temp_bytes, idx, idx_out, int(k), 0, 32, st);
  k_topk_take<<<grid(k), kThreads, 0, st>>>(idx_out, k, residual, val_out);
  return launch_check("gcx_topk_compress");
}

int gcx_topk_densify(const uint32_t* idx, const float* val, uint64_t k, uint64_t n, float* dense,
                     void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n) k_zero<<<grid(n), kThreads, 0, st>>>(dense, n);
  if (k) k_scatter<<<grid(k), kThreads, 0, st>>>(idx, val, k, dense);
  return launch_check("gcx_topk_densify");
}

const char* gcx_stats_last_error(void) { return g_err2.c_str(); }

int gcx_stats_accumulate(double* sum, const float* v, uint64_t n, unsigned int* nonfinite,
                         void* stream) {
  if (n == 0) return GCX_OK;
  k_accumulate<<<grid(n), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(sum, v, n, nonfinite);
  return launch_check("gcx_stats_accumulate");
}

int gcx_stats_snapshot(const double* sum, float* out, uint64_t n, void* stream) {
  if (n == 0) return GCX_OK;
  k_snapshot<<<grid(n), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(sum, out, n);
  return launch_check("gcx_stats_snapshot");
}

uint64_t gcx_stats_scratch_bytes(uint64_t n) {
  size_t temp = 0;
  cub::DeviceRadixSort::SortKeysDescending(nullptr, temp, (unsigned long long*)nullptr,
                                           (unsigned long long*)nullptr, int(n > 0 ? n : 1));
  return 2 * 8 * n + temp + 8 * kBlocks + 256;
}

// out[0] = sum of squares (l2^2), out[1] = sum of the keep largest squares
int gcx_stats_reduce(const double* sum, uint64_t n, uint64_t keep, void* scratch,
                     uint64_t scratch_bytes, double* out, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n == 0 || n >= (1ull << 31)) {
    g_err2 = "gcx_stats_reduce: layer size must be in [1, 2^31)";
    return GCX_E_INVALID;
  }
  if (scratch_bytes < gcx_stats_scratch_bytes(n)) {
    g_err2 = "gcx_stats_reduce: scratch too small";
    return GCX_E_INVALID;
  }
  auto* keys_in = static_cast<unsigned long long*>(scratch);
  auto* keys_out = keys_in + n;
  auto* partial = reinterpret_cast<double*>(keys_out + n);
  // CUB wants 256-byte aligned temp storage
  const uintptr_t t0 = (reinterpret_cast<uintptr_t>(partial + kBlocks) + 255) & ~uintptr_t(255);
  void* temp = reinterpret_cast<void*>(t0);
  size_t temp_bytes = scratch_bytes - (t0 - reinterpret_cast<uintptr_t>(scratch));
  k_sum_squares<<<kBlocks, kThreads, 0, st>>>(sum, nullptr, n, partial);
  k_final_sum<<<1, kThreads, 0, st>>>(partial, kBlocks, out);
  k_square_keys<<<grid(n), kThreads, 0, st>>>(sum, keys_in, n);
  cub::DeviceRadixSort::SortKeysDescending(temp, temp_bytes, keys_in, keys_out, int(n), 0, 64, st);
  k_sum_squares<<<kBlocks, kThreads, 0, st>>>(nullptr, keys_out, keep < n ? keep : n, partial);
  k_final_sum<<<1, kThreads, 0, st>>>(partial, kBlocks, out + 1);
  return launch_check("gcx_stats_reduce");
}

int gcx_mean_nodes(const float* stack, uint32_t nodes, uint64_t n, float* out, void* stream) {
  if (n == 0) return GCX_OK;
  k_mean_nodes<<<grid(n), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(stack, nodes, n, out);
  return launch_check("gcx_mean_nodes");
}

// out = sum (double(a_i) - double(b_i))^2 ; scratch >= 8*592 bytes
int gcx_sq_error(const float* a, const float* b, uint64_t n, double* scratch, double* out,
                 void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  k_sq_error<<<kBlocks, kThreads, 0, st>>>(a, b, n, scratch);
  k_final_sum<<<1, kThreads, 0, st>>>(scratch, kBlocks, out);
  return launch_check("gcx_sq_error");
}

}  // extern "C"
