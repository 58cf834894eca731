// Offline side of the path: the component scores of a layer,
// the choice of its r SVD components and the sqrt(sigma) factor split, on the
// GPU in fp64 -- the step that produces a_r / b_r for rsp_linear_create.
//
//   scores[i][j] = (1/T) * sum_t |sigma_i * x_tj * Vt_ij|    scores.cpp:15-71
//     (per-token |.| terms summed over the tokens in the reference's fixed
//     pairwise tree: split at lo + (hi - lo) / 2, so the result is
//     bit-identical to aggregate_scores for any worker count)
//   mass[i]   = sum_j scores[i][j] (ascending j, one thread per row: the
//               reference's sequential order)                  scores.cpp:73-85
//   comps     = the r largest |mass| (ties to the lower index), ascending
//               (top_k_by_magnitude, matrix.cpp:100-117)
//   a_r(i,c)  = U(i, comps_c) * sqrt(sigma_c),  b_r(c,j) = sqrt(sigma_c) * Vt(comps_c, j)
//                                                              layer.cpp:58-66
// fp64 throughout (the reference's type): every value matches the reference
// bit for bit.  Not on the decode path; no effort spent on its speed beyond
// coalesced access.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "rsp_internal.h"

namespace rsp {
namespace {

constexpr int kOffThreads = 256;

// The reference's pairwise tree over tokens [lo, hi) (scores.cpp:33-58).
__device__ double token_tree(const double* __restrict__ x, uint32_t n, uint32_t j, double sig, double v, uint32_t lo,
                             uint32_t hi) {
  if (hi - lo == 1) return fabs(sig * x[static_cast<size_t>(lo) * n + j] * v);
  const uint32_t mid = lo + (hi - lo) / 2;
  const double left = token_tree(x, n, j, sig, v, lo, mid);
  return left + token_tree(x, n, j, sig, v, mid, hi);
}

__global__ void __launch_bounds__(kOffThreads) score_kernel(const double* __restrict__ x, uint32_t T, uint32_t n,
                                                            const double* __restrict__ sigma,
                                                            const double* __restrict__ vt, uint32_t k,
                                                            double* __restrict__ out) {
  const uint32_t j = blockIdx.x * kOffThreads + threadIdx.x, i = blockIdx.y;
  if (j >= n || i >= k) return;
  const size_t e = static_cast<size_t>(i) * n + j;
  const double inv = 1.0 / static_cast<double>(T);
  out[e] = token_tree(x, n, j, sigma[i], vt[e], 0, T) * inv;
}

__global__ void __launch_bounds__(kOffThreads) mass_kernel(const double* __restrict__ s, uint32_t k, uint32_t n,
                                                           double* __restrict__ mass) {
  const uint32_t i = blockIdx.x * kOffThreads + threadIdx.x;
  if (i >= k) return;
  const double* row = s + static_cast<size_t>(i) * n;
  double acc = 0.0;
  for (uint32_t j = 0; j < n; ++j) acc += row[j];
  mass[i] = acc;
}

// One CTA: rank of every |mass| (ties to the lower index) by comparison with
// all others, then the selected indices written in ascending order (chunked
// block prefix over the flags).
__global__ void __launch_bounds__(1024) select_kernel_f64(const double* __restrict__ mass, uint32_t k, uint32_t r,
                                                          uint32_t* __restrict__ comps) {
  __shared__ uint32_t warp_sums[32];
  __shared__ uint32_t base_s;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) base_s = 0;
  __syncthreads();
  for (uint32_t c0 = 0; c0 < k; c0 += blockDim.x) {
    const uint32_t i = c0 + tid;
    uint32_t sel = 0;
    if (i < k) {
      const double a = fabs(mass[i]);
      uint32_t rank = 0;
      for (uint32_t q = 0; q < k; ++q) {
        const double b = fabs(mass[q]);
        rank += (b > a) || (b == a && q < i);
      }
      sel = rank < r;
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, sel);
    if (lane == 0) warp_sums[warp] = __popc(bal);
    __syncthreads();
    uint32_t before = base_s;
    for (uint32_t w = 0; w < warp; ++w) before += warp_sums[w];
    before += __popc(bal & ((1u << lane) - 1u));
    if (sel) comps[before] = i;
    __syncthreads();
    if (tid == 0) {
      uint32_t tot = 0;
      for (uint32_t w = 0; w < blockDim.x / 32; ++w) tot += warp_sums[w];
      base_s += tot;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kOffThreads) split_kernel(const double* __restrict__ u, uint32_t m, uint32_t ucols,
                                                            const double* __restrict__ sigma,
                                                            const double* __restrict__ vt, uint32_t n,
                                                            const uint32_t* __restrict__ comps, uint32_t r,
                                                            double* __restrict__ a_r, double* __restrict__ b_r) {
  const uint32_t c = blockIdx.y;
  const uint32_t comp = comps[c];
  const double root = sqrt(sigma[comp]);
  for (uint32_t i = blockIdx.x * kOffThreads + threadIdx.x; i < m; i += gridDim.x * kOffThreads)
    a_r[static_cast<size_t>(i) * r + c] = u[static_cast<size_t>(i) * ucols + comp] * root;
  for (uint32_t j = blockIdx.x * kOffThreads + threadIdx.x; j < n; j += gridDim.x * kOffThreads)
    b_r[static_cast<size_t>(c) * n + j] = root * vt[static_cast<size_t>(comp) * n + j];
}

}  // namespace

cudaError_t launch_scores(const double* x, uint32_t T, uint32_t n, const double* sigma, const double* vt, uint32_t k,
                          double* out, cudaStream_t s) {
  score_kernel<<<dim3((n + kOffThreads - 1) / kOffThreads, k), kOffThreads, 0, s>>>(x, T, n, sigma, vt, k, out);
  return cudaGetLastError();
}

cudaError_t launch_select_components(const double* scores, uint32_t k, uint32_t n, uint32_t r, uint32_t* comps,
                                     double* mass, cudaStream_t s) {
  mass_kernel<<<(k + kOffThreads - 1) / kOffThreads, kOffThreads, 0, s>>>(scores, k, n, mass);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || r == 0) return e;
  select_kernel_f64<<<1, 1024, 0, s>>>(mass, k, r, comps);
  return cudaGetLastError();
}

cudaError_t launch_split_factors(const double* u, uint32_t m, uint32_t ucols, const double* sigma, const double* vt,
                                 uint32_t n, const uint32_t* comps, uint32_t r, double* a_r, double* b_r,
                                 cudaStream_t s) {
  if (r == 0) return cudaSuccess;
  const uint32_t mx = m > n ? m : n;
  const uint32_t gx = (mx + kOffThreads - 1) / kOffThreads < 64 ? (mx + kOffThreads - 1) / kOffThreads : 64;
  split_kernel<<<dim3(gx, r), kOffThreads, 0, s>>>(u, m, ucols, sigma, vt, n, comps, r, a_r, b_r);
  return cudaGetLastError();
}

}  // namespace rsp
