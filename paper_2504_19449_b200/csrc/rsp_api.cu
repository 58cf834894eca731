// rsp_api.cu -- the C ABI (include/rsparse_b200.h) over the sm_100a kernels.
//
// Host-side responsibilities: validate arguments exactly where the reference
// throws (layer.cpp:96-99, sparsity.cpp:22-25, matrix.cpp:101-104,
// layer.cpp:83-86, layer.cpp:40-49), upload the operator in the B200 layout,
// plan the fused kernel's decomposition for this GPU, and capture stacks of
// forwards into CUDA graphs.  There is no CPU compute fallback: every
// numeric result comes from a kernel in rsp_kernels.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/rsparse_b200.h"
#include "rsp_internal.h"

using rsp::LinDesc;
using rsp::BatchParams;
using rsp::StackParams;
using rsp::WsLayout;

namespace {

thread_local std::string g_last_error;

rsp_status fail(rsp_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

#define RSP_CUDA(call)                                                                    \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(RSP_E_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                    \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

struct DevProps {
  int sms = 0;
  int smem_optin = 0;
};

DevProps device_props(int dev) {
  static std::mutex mu;
  static std::vector<DevProps> cache;
  std::lock_guard<std::mutex> lk(mu);
  if (dev >= static_cast<int>(cache.size())) cache.resize(dev + 1);
  if (cache[dev].sms == 0) {
    cudaDeviceGetAttribute(&cache[dev].sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&cache[dev].smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  }
  return cache[dev];
}

size_t dtype_size(rsp_dtype d) { return d == RSP_F64 ? 8 : (d == RSP_F32 ? 4 : 2); }

uint32_t round_up(uint32_t v, uint32_t a) { return (v + a - 1) / a * a; }

constexpr int kMaxN = 32768;  // selection keeps x in shared memory
constexpr int kMaxKSplits = 40;  // channel splits per column tile (o / down use all 148 SMs)

std::atomic<int> g_batch_trace{0};  // rsp_debug_set_batch_trace

// k = ceil(s * n) in double (sparsity.cpp:26-27).
uint32_t keep_count(double s, uint32_t n) {
  return static_cast<uint32_t>(std::ceil(s * static_cast<double>(n)));
}

// How one linear is decomposed over the GPU (see make_plan).
struct LaunchPlan {
  int col_tiles = 1, k_splits = 1, grid = 1;
  int cap_w = 1, cap_u = 1, cap_a = 1;
  int nb_pad = 4;
  size_t smem = 0;
  size_t ws_bytes = 0;  // single-linear workspace
  bool bf16_x_only = false;  // m_in too wide for fp32 activations on chip
};

}  // namespace

struct rsp_linear {
  int device = 0;
  uint32_t m_in = 0, m_out = 0, rank = 0, k = 0;
  double keep_fraction = 1.0;
  uint32_t row_begin = 0, row_end = 0, m = 0, m_pad = 0, r_pad = 0;
  rsp_dtype wdt = RSP_BF16;
  int es = 2;
  void* Wt = nullptr;
  void* At = nullptr;
  void* Bt = nullptr;
  LaunchPlan plan;
  bool pdl = true;
  bool deterministic = false;  // RSP_FLAG_DETERMINISTIC: fixed-order split-K combine
  bool batch_tc = false;       // RSP_FLAG_BATCH_TCGEN05: batched products on tcgen05 (TMEM accumulators)
  // forward_host staging (lazily created)
  cudaStream_t stream = nullptr;
  void* x_dev = nullptr;
  float* y_dev = nullptr;
  void* ws = nullptr;
  void* x_pin = nullptr;
  float* y_pin = nullptr;
  uint32_t host_batch = 0;
  std::mutex host_mu;  // concurrent forward_host calls on one handle take turns on the staging
  std::vector<uint32_t> comps;  // DecomposedLayer::selected_components
};

struct rsp_stack {
  int device = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  void* ws = nullptr;
  LinDesc* descs = nullptr;  // device array
  float** ypeer = nullptr;   // device [count][kMaxPeers] y destinations (npeer > 1)
  unsigned long long** xctr = nullptr;  // device [xrank] every rank's exchange words (cross-process)
  std::vector<uint32_t> grids;          // per-linear CTA counts
  rsp::LinCtl* ctl = nullptr;  // device control table
  void* plans = nullptr;     // device plan table [count][grid]
  StackParams params = {};   // the captured launch (re-launched by the debug trace)
  int es = 2, grid = 1;
  bool x_bf16 = false;
  bool pdl = true;
  size_t smem = 0;
  // contiguous device spans covering every x / y of the stack (host-buffer path)
  uint8_t* x_lo = nullptr;
  uint8_t* y_lo = nullptr;
  size_t x_span = 0, y_span = 0;
};

namespace {

// Decompose one forward over the GPU: col_tiles column tiles x k_splits
// channel splits, at most one CTA per SM (a second slot per SM is left for
// the next linear's CTAs under PDL).  A column tile is C2 whole 512-byte warp
// columns of a row (C2 in {1,2,4,8,16}); per-CTA time ~ k*C2/(16*k_splits),
// and the split-K combine costs k_splits*m float reductions, so the cheapest
// C2/k_splits wins with k_splits <= kMaxKSplits.
rsp_status make_plan(const rsp_linear& L, const DevProps& dp, LaunchPlan* out, int budget = 0) {
  LaunchPlan p;
  const uint32_t n = L.m_in;
  const int vrow = static_cast<int>(L.m_pad * L.es / 16);  // 16-B units per W^T row
  const int wcols = (vrow + 31) / 32;                       // 512-B warp columns per row
  if (L.r_pad > rsp::kTAccCap || L.r_pad * L.es > 4096u)
    return fail(RSP_E_UNSUPPORTED, "rank %u too large (B_r^T rows limited to 4 KB, r_pad <= %u)", L.rank,
                rsp::kTAccCap);
  const int sms = std::max(1, budget > 0 ? std::min(budget, dp.sms) : dp.sms);  // CTAs this linear may use
  const int ks_cap = kMaxKSplits;
  int best_nt = 1, best_ks = 1;
  double best = 1e30;
  // with a low-rank term, prefer tiles of at most 4 warp columns: that leaves
  // room for a stage-1 warp group beside the W warps (warp-specialised path)
  const int c2_pref = (L.rank > 0 && L.k < n) ? 4 : 8;
  for (int c2 = 1; c2 <= 8; c2 *= 2) {  // <= one row of warps (kThreads / 32 = 8)
    const int nt = (wcols + c2 - 1) / c2;
    if (nt > sms || nt > static_cast<int>(rsp::kMaxTickets)) continue;
    const int ks = std::min(sms / nt, ks_cap);
    const double cost = static_cast<double>(c2) / ks * (c2 > c2_pref ? 1.25 : 1.0);
    if (cost < best * 0.99 || (cost <= best * 1.01 && ks <= 24)) {
      best = std::min(best, cost);
      best_nt = nt;
      best_ks = ks;
    }
  }
  if (best > 1e29 || (wcols + best_nt - 1) / best_nt > 8)
    return fail(RSP_E_UNSUPPORTED, "no column tiling for m_out %u (%d warp columns)", L.m, wcols);
  int nt = best_nt, ks = best_ks;
  // Small layers: keep >= ~32 KB of streamed bytes per CTA.
  const double bytes = static_cast<double>(L.k + L.rank) * vrow * 16.0 +
                       static_cast<double>(n - std::min(n, L.k)) * (L.r_pad * L.es);
  const int want = std::max(1, static_cast<int>(std::ceil(bytes / 32768.0)));
  ks = std::min(ks, std::max(1, (want + nt - 1) / nt));
  ks = std::min(ks, static_cast<int>(std::max(1u, n)));
  ks = std::max(1, std::min(ks, sms / nt));
  p.col_tiles = nt;
  p.k_splits = ks;
  p.grid = nt * ks;
  p.nb_pad = static_cast<int>(round_up(static_cast<uint32_t>(p.grid), 4u));
  p.cap_w = static_cast<int>((n + ks - 1) / ks) + 1;          // W channel range of one CTA
  p.cap_u = static_cast<int>((n + p.grid - 1) / p.grid) + 1;  // stage-1 channel range of one CTA
  p.cap_a = static_cast<int>((L.rank + ks - 1) / ks) + 1;     // A_r^T rows of one CTA
  p.smem = rsp::stack_smem_bytes(static_cast<int>(n), false, p.cap_w, p.cap_u, p.cap_a);  // fp32 x: the larger
  if (p.smem > static_cast<size_t>(dp.smem_optin)) {
    // wide inputs: x kept on chip as bf16 only (fp32 activations refused at forward)
    p.smem = rsp::stack_smem_bytes(static_cast<int>(n), true, p.cap_w, p.cap_u, p.cap_a);
    p.bf16_x_only = true;
    if (p.smem > static_cast<size_t>(dp.smem_optin))
      return fail(RSP_E_UNSUPPORTED, "fused kernel needs %zu B shared memory (> %d)", p.smem, dp.smem_optin);
  }
  p.ws_bytes = WsLayout::make(1, p.nb_pad, static_cast<int>(L.r_pad), ks, static_cast<int>(L.m_pad)).bytes;
  *out = p;
  return RSP_OK;
}

LinDesc lin_desc(const rsp_linear* h, const void* x, float* y, bool dense, int slot, int flags,
                 const LaunchPlan* plan = nullptr, int cta0 = 0) {
  const LaunchPlan& pl = plan ? *plan : h->plan;
  LinDesc d = {};
  d.Wt = h->Wt;
  d.At = h->At;
  d.Bt = h->Bt;
  d.x = x;
  d.y = y;
  d.n = static_cast<int>(h->m_in);
  d.m = static_cast<int>(h->m);
  d.m_pad = static_cast<int>(h->m_pad);
  d.r = static_cast<int>(h->rank);
  d.r_pad = static_cast<int>(h->r_pad);
  d.k = dense ? static_cast<int>(h->m_in) : static_cast<int>(h->k);
  d.col_tiles = pl.col_tiles;
  d.k_splits = pl.k_splits;
  d.grid = pl.grid;
  d.flags = flags | (dense ? rsp::kLinDense : 0);
  d.slot = slot;
  d.cta0 = cta0;
  return d;
}

void bind_workspace(StackParams* p, void* ws, const WsLayout& w) {
  uint8_t* b = static_cast<uint8_t*>(ws);
  p->hdr = reinterpret_cast<unsigned*>(b);
  p->slots = reinterpret_cast<unsigned*>(b + w.slots_off);
  p->t_acc = reinterpret_cast<float*>(b + w.tacc_off);
  p->t_part = reinterpret_cast<float*>(b + w.tpart_off);
  p->y_part = reinterpret_cast<float*>(b + w.ypart_off);
}

rsp_status check_x_dtype(rsp_dtype d) {
  if (d != RSP_F32 && d != RSP_BF16)
    return fail(RSP_E_USAGE, "activation dtype must be RSP_F32 or RSP_BF16");
  return RSP_OK;
}

rsp_status upload(const rsp_linear_desc* d, rsp_linear* h) {
  const size_t sz = dtype_size(d->src_dtype);
  const int sdt = d->src_dtype == RSP_F32 ? 0 : (d->src_dtype == RSP_BF16 ? 1 : 2);
  const size_t n = h->m_in, mo = h->m_out, r = h->rank, m = h->m;
  // Stage host sources on the device (in their own dtype) and convert there.
  auto stage = [&](const void* src, size_t count, void** tmp) -> rsp_status {
    *tmp = nullptr;
    if (d->src_memory == RSP_MEM_DEVICE) return RSP_OK;
    RSP_CUDA(cudaMalloc(tmp, std::max<size_t>(count * sz, 16)));
    RSP_CUDA(cudaMemcpy(*tmp, src, count * sz, cudaMemcpyHostToDevice));
    return RSP_OK;
  };
  auto src_of = [&](const void* host_or_dev, void* tmp) -> const uint8_t* {
    return static_cast<const uint8_t*>(tmp ? tmp : host_or_dev);
  };
  const int de = h->es;
  void* tmp = nullptr;
  rsp_status st;
  // W -> Wt[n][m_pad]
  if ((st = stage(d->w, n * mo, &tmp))) return st;
  {
    const uint8_t* w = src_of(d->w, tmp);
    cudaError_t e;
    if (d->w_layout == RSP_W_ROW_MAJOR)
      e = rsp::launch_convert(w + h->row_begin * n * sz, sdt, m, n, n, h->Wt, de, h->m_pad, true,
                              nullptr);
    else
      e = rsp::launch_convert(w + h->row_begin * sz, sdt, n, m, mo, h->Wt, de, h->m_pad, false,
                              nullptr);
    cudaDeviceSynchronize();
    if (tmp) cudaFree(tmp);
    if (e != cudaSuccess) return fail(RSP_E_CUDA, "convert W: %s", cudaGetErrorString(e));
  }
  if (r > 0) {
    // a_r (m_out x r) -> At[r][m_pad]
    if ((st = stage(d->a_r, mo * r, &tmp))) return st;
    cudaError_t e = rsp::launch_convert(src_of(d->a_r, tmp) + h->row_begin * r * sz, sdt, m, r, r,
                                        h->At, de, h->m_pad, true, nullptr);
    cudaDeviceSynchronize();
    if (tmp) cudaFree(tmp);
    if (e != cudaSuccess) return fail(RSP_E_CUDA, "convert a_r: %s", cudaGetErrorString(e));
    // b_r (r x n) -> Bt[n][r_pad]
    if ((st = stage(d->b_r, r * n, &tmp))) return st;
    e = rsp::launch_convert(src_of(d->b_r, tmp), sdt, r, n, n, h->Bt, de, h->r_pad, true, nullptr);
    cudaDeviceSynchronize();
    if (tmp) cudaFree(tmp);
    if (e != cudaSuccess) return fail(RSP_E_CUDA, "convert b_r: %s", cudaGetErrorString(e));
  }
  RSP_CUDA(cudaGetLastError());
  return RSP_OK;
}

void free_linear(rsp_linear* h) {
  if (!h) return;
  DeviceGuard g(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  cudaFree(h->Wt);
  cudaFree(h->At);
  cudaFree(h->Bt);
  cudaFree(h->x_dev);
  cudaFree(h->y_dev);
  cudaFree(h->ws);
  cudaFreeHost(h->x_pin);
  cudaFreeHost(h->y_pin);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

rsp_status launch_forward(const rsp_linear* h, const void* x, rsp_dtype xdt, float* y, void* ws,
                          size_t ws_bytes, cudaStream_t stream, bool dense, long long* trace = nullptr) {
  if (!ws || ws_bytes < h->plan.ws_bytes)
    return fail(RSP_E_USAGE, "workspace of %zu bytes is smaller than the %zu required", ws_bytes,
                h->plan.ws_bytes);
  if (xdt != RSP_BF16 && h->plan.bf16_x_only)
    return fail(RSP_E_UNSUPPORTED, "m_in %u: fp32 activations do not fit in shared memory; pass bf16 activations",
                h->m_in);
  StackParams p = {};
  p.descs = nullptr;
  p.one = lin_desc(h, x, y, dense, 0, 0);
  p.count = 1;
  p.n_max = static_cast<int>(h->m_in);
  p.cap_w = h->plan.cap_w;
  p.cap_u = h->plan.cap_u;
  p.cap_a = h->plan.cap_a;
  p.nb_pad = h->plan.nb_pad;
  p.deterministic = h->deterministic ? 1 : 0;
  p.zero = 0u;
  p.trace = trace;
  bind_workspace(&p, ws, WsLayout::make(1, h->plan.nb_pad, static_cast<int>(h->r_pad), h->plan.k_splits,
                                         static_cast<int>(h->m_pad)));
  cudaError_t e = rsp::launch_stack(p, h->es, xdt == RSP_BF16, h->plan.grid, h->plan.smem, stream, h->pdl);
  if (e != cudaSuccess) return fail(RSP_E_CUDA, "fused forward launch: %s", cudaGetErrorString(e));
  return RSP_OK;
}

// Device operand [rows][ld] (first `cols` valid) -> host float, element (i, j)
// stored at out[j * rows + i] (the reference's row-major transpose).
rsp_status device_to_host_t(const rsp_linear* h, const void* src, size_t rows, size_t cols, size_t ld,
                            std::vector<float>* out) {
  out->assign(rows * cols, 0.f);
  if (rows * cols == 0) return RSP_OK;
  std::vector<uint8_t> buf(rows * ld * h->es);
  RSP_CUDA(cudaMemcpy(buf.data(), src, buf.size(), cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < rows; ++i)
    for (size_t j = 0; j < cols; ++j) {
      const size_t idx = i * ld + j;
      float f;
      if (h->es == 4) {
        std::memcpy(&f, buf.data() + idx * 4, 4);
      } else {
        uint16_t b;
        std::memcpy(&b, buf.data() + idx * 2, 2);
        const uint32_t u = static_cast<uint32_t>(b) << 16;
        std::memcpy(&f, &u, 4);
      }
      (*out)[j * rows + i] = f;
    }
  return RSP_OK;
}

// RSPL parse (layer.cpp:269-301) over an in-memory copy of the file.
struct RsplReader {
  const std::string& path;
  const std::vector<char>& buf;
  size_t pos = 0;
  bool take(void* dst, size_t bytes) {
    if (buf.size() - pos < bytes) return false;
    if (dst) std::memcpy(dst, buf.data() + pos, bytes);
    pos += bytes;
    return true;
  }
};

rsp_status rspl_parse(const char* path, rsp_rspl_header* hdr, float* w, float* a, float* b, uint32_t* comps) {
  if (!path || !hdr) return fail(RSP_E_USAGE, "null path or header");
  const std::string p(path);
  std::ifstream in(p, std::ios::binary);
  if (!in) return fail(RSP_E_IO, "cannot open layer file: %s", path);
  const std::vector<char> buf((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  RsplReader r{p, buf};
  char magic[4];
  if (!r.take(magic, 4) || std::memcmp(magic, "RSPL", 4) != 0)
    return fail(RSP_E_IO, "bad magic in %s (expected RSPL)", path);
  uint8_t version = 0;
  if (!r.take(&version, 1)) return fail(RSP_E_IO, "truncated file: %s", path);
  if (version != 1) return fail(RSP_E_IO, "unsupported RSPL version %u in %s", version, path);
  uint32_t dims[4];
  if (!r.take(dims, sizeof(dims))) return fail(RSP_E_IO, "truncated file: %s", path);
  const uint64_t n = dims[0], m = dims[1], rk = dims[2];
  if (!r.take(w, 4 * n * m) || !r.take(a, 4 * m * rk) || !r.take(b, 4 * rk * n) ||
      !r.take(comps, 4 * rk))
    return fail(RSP_E_IO, "truncated file: %s", path);
  double plan[2];
  if (!r.take(plan, sizeof(plan))) return fail(RSP_E_IO, "truncated file: %s", path);
  if (static_cast<uint64_t>(plan[1]) != rk) return fail(RSP_E_IO, "inconsistent rank fields in %s", path);
  hdr->m_in = dims[0];
  hdr->m_out = dims[1];
  hdr->rank = dims[2];
  hdr->kept_width = dims[3];
  hdr->keep_fraction = plan[0];
  return RSP_OK;
}

}  // namespace

extern "C" {

int rsp_abi_version(void) { return RSP_ABI_VERSION; }

const char* rsp_last_error(void) { return g_last_error.c_str(); }

int rsp_device_sm_count(int device) { return device_props(device).sms; }

rsp_status rsp_keep_count(double keep_fraction, uint32_t n, uint32_t* k_out) {
  if (!(keep_fraction >= 0.0 && keep_fraction <= 1.0))
    return fail(RSP_E_USAGE, "keep_fraction must lie in [0, 1], got %f", keep_fraction);
  *k_out = keep_count(keep_fraction, n);
  return RSP_OK;
}

rsp_status rsp_plan_for(double rho, double budget, uint32_t m_in, uint32_t m_out,
                        double* keep_fraction, uint32_t* rank) {
  // search.cpp:14-25, search.hpp:24
  const double m = static_cast<double>(m_out), n = static_cast<double>(m_in);
  const double raw = (1.0 - rho) * budget * (m * n) / (m + n);
  long long r = std::llround(raw);
  const long long cap = static_cast<long long>(std::min(m_in, m_out));
  r = std::clamp(r, 0LL, cap);
  *keep_fraction = rho * budget;
  *rank = static_cast<uint32_t>(r);
  return RSP_OK;
}

rsp_status rsp_shard_rows(uint32_t m_out, uint32_t shard_rank, uint32_t shard_count, uint32_t* begin,
                          uint32_t* end) {
  const uint32_t sc = shard_count ? shard_count : 1;
  if (shard_rank >= sc) return fail(RSP_E_USAGE, "shard_rank %u >= shard_count %u", shard_rank, sc);
  *begin = static_cast<uint32_t>(static_cast<uint64_t>(m_out) * shard_rank / sc);
  *end = static_cast<uint32_t>(static_cast<uint64_t>(m_out) * (shard_rank + 1) / sc);
  return RSP_OK;
}

rsp_status rsp_linear_create(const rsp_linear_desc* d, rsp_linear** out) {
  if (!d || !out) return fail(RSP_E_USAGE, "null descriptor or output");
  *out = nullptr;
  if (d->m_in == 0 || d->m_out == 0) return fail(RSP_E_USAGE, "m_in and m_out must be positive");
  if (d->m_in > static_cast<uint32_t>(kMaxN))
    return fail(RSP_E_UNSUPPORTED, "m_in %u exceeds %d", d->m_in, kMaxN);
  if (d->rank > std::min(d->m_in, d->m_out))  // layer.cpp:40-44
    return fail(RSP_E_USAGE, "decompose: rank %u exceeds min(m_in, m_out) = %u", d->rank,
                std::min(d->m_in, d->m_out));
  if (!(d->keep_fraction >= 0.0 && d->keep_fraction <= 1.0))  // sparsity.cpp:22-25
    return fail(RSP_E_USAGE, "keep_fraction must lie in [0, 1], got %f", d->keep_fraction);
  if (d->k_override > static_cast<int64_t>(d->m_in))  // matrix.cpp:101-104
    return fail(RSP_E_USAGE, "top_k_by_magnitude: k=%lld exceeds vector length %u",
                static_cast<long long>(d->k_override), d->m_in);
  if (d->weight_dtype != RSP_F32 && d->weight_dtype != RSP_BF16)
    return fail(RSP_E_USAGE, "weight_dtype must be RSP_F32 or RSP_BF16");
  if (d->src_dtype != RSP_F32 && d->src_dtype != RSP_BF16 && d->src_dtype != RSP_F64)
    return fail(RSP_E_USAGE, "src_dtype must be F32, BF16 or F64");
  if (!d->w || (d->rank > 0 && (!d->a_r || !d->b_r)))
    return fail(RSP_E_USAGE, "missing weight or factor pointer");
  const uint32_t sc = d->shard_count ? d->shard_count : 1;
  if (d->shard_rank >= sc) return fail(RSP_E_USAGE, "shard_rank %u >= shard_count %u", d->shard_rank, sc);

  DeviceGuard g(d->device);
  auto* h = new rsp_linear();
  h->device = d->device;
  h->m_in = d->m_in;
  h->m_out = d->m_out;
  h->rank = d->rank;
  h->keep_fraction = d->keep_fraction;
  h->k = d->k_override >= 0 ? static_cast<uint32_t>(d->k_override) : keep_count(d->keep_fraction, d->m_in);
  rsp_shard_rows(d->m_out, d->shard_rank, sc, &h->row_begin, &h->row_end);
  h->m = h->row_end - h->row_begin;
  if (h->m == 0) {
    delete h;
    return fail(RSP_E_USAGE, "shard %u of %u owns no output rows", d->shard_rank, sc);
  }
  h->m_pad = round_up(h->m, 8);
  h->r_pad = d->rank ? round_up(d->rank, 8) : 0;
  h->wdt = d->weight_dtype;
  h->es = d->weight_dtype == RSP_F32 ? 4 : 2;
  h->pdl = true;
  h->deterministic = (d->flags & RSP_FLAG_DETERMINISTIC) != 0;
  h->batch_tc = (d->flags & RSP_FLAG_BATCH_TCGEN05) != 0;
  const DevProps dp = device_props(d->device);
  if (dp.sms == 0) {
    delete h;
    return fail(RSP_E_CUDA, "no CUDA device %d", d->device);
  }
  rsp_status st = make_plan(*h, dp, &h->plan);
  if (st) {
    delete h;
    return st;
  }
  const size_t wbytes = static_cast<size_t>(h->m_in) * h->m_pad * h->es;
  const size_t abytes = static_cast<size_t>(h->rank) * h->m_pad * h->es;
  const size_t bbytes = static_cast<size_t>(h->m_in) * h->r_pad * h->es;
  cudaError_t e = cudaMalloc(&h->Wt, wbytes);
  if (e == cudaSuccess && abytes) e = cudaMalloc(&h->At, abytes);
  if (e == cudaSuccess && bbytes) e = cudaMalloc(&h->Bt, bbytes);
  if (e == cudaSuccess) e = cudaMemset(h->Wt, 0, wbytes);
  if (e == cudaSuccess && abytes) e = cudaMemset(h->At, 0, abytes);
  if (e == cudaSuccess && bbytes) e = cudaMemset(h->Bt, 0, bbytes);
  if (e != cudaSuccess) {
    free_linear(h);
    return fail(RSP_E_CUDA, "allocating %zu B of operator storage: %s", wbytes + abytes + bbytes,
                cudaGetErrorString(e));
  }
  st = upload(d, h);
  if (st) {
    free_linear(h);
    return st;
  }
  // The attribute is per kernel, not per launch: raise it to the opt-in
  // maximum once so every handle's plan fits regardless of creation order.
  e = rsp::stack_set_smem(static_cast<size_t>(dp.smem_optin));
  if (e != cudaSuccess) {
    free_linear(h);
    return fail(RSP_E_CUDA, "cudaFuncSetAttribute(smem=%zu): %s", h->plan.smem, cudaGetErrorString(e));
  }
  h->comps.resize(h->rank);
  for (uint32_t c = 0; c < h->rank; ++c) h->comps[c] = c;
  *out = h;
  return RSP_OK;
}

void rsp_linear_destroy(rsp_linear* h) { free_linear(h); }

rsp_status rsp_linear_info_get(const rsp_linear* h, rsp_linear_info* o) {
  if (!h || !o) return fail(RSP_E_USAGE, "null handle");
  o->m_in = h->m_in;
  o->m_out = h->m_out;
  o->rank = h->rank;
  o->k = h->k;
  o->row_begin = h->row_begin;
  o->row_end = h->row_end;
  o->m_pad = h->m_pad;
  o->r_pad = h->r_pad;
  o->col_tiles = static_cast<uint32_t>(h->plan.col_tiles);
  o->k_splits = static_cast<uint32_t>(h->plan.k_splits);
  o->grid = static_cast<uint32_t>(h->plan.grid);
  o->smem_bytes = static_cast<uint32_t>(h->plan.smem);
  o->weight_dtype = h->wdt;
  o->device_bytes = (static_cast<uint64_t>(h->m_in) * h->m_pad + static_cast<uint64_t>(h->rank) * h->m_pad +
                     static_cast<uint64_t>(h->m_in) * h->r_pad) * h->es;
  o->path = RSP_PATH_PERSISTENT | (h->deterministic ? RSP_PATH_DETERMINISTIC : 0u) |
            (h->deterministic || h->es != 2 ? 0u : (h->batch_tc ? RSP_PATH_BATCH_TCGEN05 : RSP_PATH_BATCH_MMA));
  return RSP_OK;
}

size_t rsp_linear_workspace_size(const rsp_linear* h, uint32_t /*batch*/) {
  // single-token area, then the batch > 1 area (counters, cuts, t accumulator)
  return h ? h->plan.ws_bytes + rsp::kBatchWsBytes(static_cast<int>(h->r_pad)) : 0;
}

rsp_status rsp_workspace_init(void* ws, size_t bytes, void* stream) {
  RSP_CUDA(cudaMemsetAsync(ws, 0, bytes, static_cast<cudaStream_t>(stream)));
  return RSP_OK;
}

namespace {

// Decomposition of a batched forward: 64 x cw output columns per CTA, ks
// channel splits, the most CTAs (<= #SMs) whose per-CTA activation slab
// (B x n/ks bf16) and shared-memory carve-up fit.
bool batch_plan(const rsp_linear* h, int B, const DevProps& dp, BatchParams* out) {
  const int n = static_cast<int>(h->m_in), m = static_cast<int>(h->m), sms = std::max(1, dp.sms);
  bool found = false;
  BatchParams best = {};
  for (int cw = 1; cw <= 8; cw *= 2) {
    const int tiles = (m + 64 * cw - 1) / (64 * cw);
    if (tiles > sms) continue;
    const int ks = std::max(1, std::min({sms / tiles, 32, n}));
    BatchParams p = {};
    p.n = n;
    p.m = m;
    p.m_pad = static_cast<int>(h->m_pad);
    p.r = static_cast<int>(h->rank);
    p.r_pad = static_cast<int>(h->r_pad);
    p.k = static_cast<int>(h->k);
    p.B = B;
    p.cw = cw;
    p.ks = ks;
    p.tc = cw == 8 && h->batch_tc;
    p.grid = tiles * ks;
    // CTA b < B computes token b's cut and every CTA waits for all B cuts:
    // fewer CTAs than tokens would never publish some cuts (small n / m)
    if (p.grid < B) continue;
    p.range_max = ((n + ks - 1) / ks + 16 + 7) / 8 * 8;  // 8-aligned rows around [wc0, wc1)
    p.slice_max = ((n + p.grid - 1) / p.grid + 16 + 7) / 8 * 8;
    p.na_max = (p.r + ks - 1) / ks + 1;
    if (2 * B * p.range_max > 96 * 1024) continue;
    if (rsp::batch_smem_bytes(p) > static_cast<size_t>(dp.smem_optin)) continue;
    if (!found || p.grid >= best.grid) {  // ties: the wider column tile (cw = 8 stages whole rows)
      best = p;
      found = true;
    }
  }
  if (found) *out = best;
  return found;
}

}  // namespace

rsp_status rsp_linear_forward(const rsp_linear* h, const void* x, rsp_dtype xdt, float* y,
                              uint32_t batch, void* ws, size_t ws_bytes, void* stream) {
  if (!h || !x || !y) return fail(RSP_E_USAGE, "null handle or buffer");
  if (rsp_status st = check_x_dtype(xdt)) return st;
  if (batch == 0) return RSP_OK;
  DeviceGuard g(h->device);
  // batch > 1, bf16 weights and activations: one pass over the union of the
  // tokens' selected rows on the tensor cores (rsp_batch.cu)
  BatchParams bp;
  if (batch > 1 && batch <= static_cast<uint32_t>(rsp::kBatchMax) && h->es == 2 && xdt == RSP_BF16 &&
      !h->deterministic &&
      batch_plan(h, static_cast<int>(batch), device_props(h->device), &bp)) {
    if (!ws || ws_bytes < rsp_linear_workspace_size(h, batch))
      return fail(RSP_E_USAGE, "workspace of %zu bytes is smaller than the %zu required", ws_bytes,
                  rsp_linear_workspace_size(h, batch));
    uint8_t* area = static_cast<uint8_t*>(ws) + h->plan.ws_bytes;
    bp.Wt = h->Wt;
    bp.At = h->At;
    bp.Bt = h->Bt;
    bp.x = x;
    bp.y = y;
    bp.ctr = reinterpret_cast<unsigned*>(area);
    bp.cuts = reinterpret_cast<int2*>(area + 256);
    bp.t_acc = reinterpret_cast<float*>(area + 512);
    bp.trace = g_batch_trace.load() ? 1 : 0;
    const cudaStream_t cs = static_cast<cudaStream_t>(stream);
    const bool has_lr = bp.r > 0 && bp.k < bp.n;
    bp.zero_y = bp.ks > 1 && has_lr;  // zeroed inside, ahead of the t barrier
    bp.pdl = 1;
    bp.zero = 0u;
    if (bp.ks > 1 && !has_lr) RSP_CUDA(cudaMemsetAsync(y, 0, sizeof(float) * h->m * batch, cs));
    cudaError_t e = rsp::launch_batch(bp, true, cs);
    if (e != cudaSuccess) return fail(RSP_E_CUDA, "batched forward launch: %s", cudaGetErrorString(e));
    return RSP_OK;
  }
  const size_t xs = static_cast<size_t>(h->m_in) * (xdt == RSP_BF16 ? 2 : 4);
  for (uint32_t t = 0; t < batch; ++t) {
    rsp_status st = launch_forward(h, static_cast<const uint8_t*>(x) + t * xs, xdt, y + static_cast<size_t>(t) * h->m,
                                   ws, ws_bytes, static_cast<cudaStream_t>(stream), false);
    if (st) return st;
  }
  return RSP_OK;
}

extern "C" rsp_status rsp_debug_set_batch_trace(int on) {
  g_batch_trace.store(on ? 1 : 0);
  return RSP_OK;
}

extern "C" rsp_status rsp_debug_batch_trace(int64_t* host, uint32_t ctas) {
  if (!host || ctas > 160) return fail(RSP_E_USAGE, "bad trace buffer");
  RSP_CUDA(rsp::batch_trace_copy(reinterpret_cast<long long*>(host), static_cast<int>(ctas)));
  return RSP_OK;
}

rsp_status rsp_linear_dense_forward(const rsp_linear* h, const void* x, rsp_dtype xdt, float* y,
                                    void* ws, size_t ws_bytes, void* stream) {
  if (!h || !x || !y) return fail(RSP_E_USAGE, "null handle or buffer");
  if (rsp_status st = check_x_dtype(xdt)) return st;
  DeviceGuard g(h->device);
  return launch_forward(h, x, xdt, y, ws, ws_bytes, static_cast<cudaStream_t>(stream), true);
}

rsp_status rsp_debug_forward_trace(const rsp_linear* h, const void* x, rsp_dtype xdt, float* y, void* ws,
                                   size_t ws_bytes, int64_t* trace, int dense, void* stream) {
  if (!h || !x || !y || !trace) return fail(RSP_E_USAGE, "null handle or buffer");
  if (rsp_status st = check_x_dtype(xdt)) return st;
  DeviceGuard g(h->device);
  return launch_forward(h, x, xdt, y, ws, ws_bytes, static_cast<cudaStream_t>(stream), dense != 0,
                        reinterpret_cast<long long*>(trace));
}

rsp_status rsp_linear_forward_host(rsp_linear* h, const void* x_host, rsp_dtype xdt, void* y_host,
                                   rsp_dtype ydt, uint32_t batch) {
  if (!h || !x_host || !y_host) return fail(RSP_E_USAGE, "null handle or buffer");
  if (rsp_status st = check_x_dtype(xdt)) return st;
  if (ydt != RSP_F32 && ydt != RSP_F64) return fail(RSP_E_USAGE, "y dtype must be F32 or F64");
  if (batch == 0) return RSP_OK;
  std::lock_guard<std::mutex> lock(h->host_mu);
  DeviceGuard g(h->device);
  const size_t xs = static_cast<size_t>(h->m_in) * 4;  // room for fp32
  if (!h->stream) RSP_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  if (h->host_batch < batch) {
    cudaFree(h->x_dev);
    cudaFree(h->y_dev);
    cudaFreeHost(h->x_pin);
    cudaFreeHost(h->y_pin);
    h->x_dev = h->x_pin = nullptr;
    h->y_dev = h->y_pin = nullptr;
    RSP_CUDA(cudaMalloc(&h->x_dev, xs * batch));
    RSP_CUDA(cudaMalloc(&h->y_dev, sizeof(float) * h->m * batch));
    RSP_CUDA(cudaMallocHost(&h->x_pin, xs * batch));
    RSP_CUDA(cudaMallocHost(&h->y_pin, sizeof(float) * h->m * batch));
    h->host_batch = batch;
  }
  // the workspace of the largest path forward() may take (batch > 1 adds the
  // batched-kernel area after the single-token one)
  const size_t ws_bytes = rsp_linear_workspace_size(h, batch);
  if (!h->ws) {
    RSP_CUDA(cudaMalloc(&h->ws, ws_bytes));
    RSP_CUDA(cudaMemsetAsync(h->ws, 0, ws_bytes, h->stream));
  }
  const size_t xbytes = static_cast<size_t>(h->m_in) * (xdt == RSP_BF16 ? 2 : 4) * batch;
  std::memcpy(h->x_pin, x_host, xbytes);
  RSP_CUDA(cudaMemcpyAsync(h->x_dev, h->x_pin, xbytes, cudaMemcpyHostToDevice, h->stream));
  rsp_status st = rsp_linear_forward(h, h->x_dev, xdt, h->y_dev, batch, h->ws, ws_bytes, h->stream);
  if (st) return st;
  const size_t ycount = static_cast<size_t>(h->m) * batch;
  RSP_CUDA(cudaMemcpyAsync(h->y_pin, h->y_dev, ycount * sizeof(float), cudaMemcpyDeviceToHost, h->stream));
  RSP_CUDA(cudaStreamSynchronize(h->stream));
  if (ydt == RSP_F32) {
    std::memcpy(y_host, h->y_pin, ycount * sizeof(float));
  } else {
    double* yd = static_cast<double*>(y_host);
    for (size_t i = 0; i < ycount; ++i) yd[i] = h->y_pin[i];
  }
  return RSP_OK;
}

rsp_status rsp_gather_matvec(const rsp_linear* h, const void* x, rsp_dtype xdt, const int64_t* kept,
                             uint32_t nkept, float* y, uint64_t* touched_bytes, void* stream) {
  if (!h || !x || !y || (nkept && !kept)) return fail(RSP_E_USAGE, "null handle or buffer");
  if (rsp_status st = check_x_dtype(xdt)) return st;
  std::vector<int32_t> k32(nkept);
  for (uint32_t t = 0; t < nkept; ++t) {
    if (kept[t] < 0 || kept[t] >= static_cast<int64_t>(h->m_in))  // layer.cpp:83-86
      return fail(RSP_E_USAGE, "gather_matvec: kept index %lld out of range for %u columns",
                  static_cast<long long>(kept[t]), h->m_in);
    k32[t] = static_cast<int32_t>(kept[t]);
  }
  DeviceGuard g(h->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int32_t* kd = nullptr;
  if (nkept) {
    RSP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&kd), nkept * sizeof(int32_t), s));
    RSP_CUDA(cudaMemcpyAsync(kd, k32.data(), nkept * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  }
  cudaError_t e = rsp::launch_gather(h->Wt, h->es, static_cast<int>(h->m), static_cast<int>(h->m_pad), x,
                                     xdt == RSP_BF16, kd, static_cast<int>(nkept), y, s);
  if (kd) cudaFreeAsync(kd, s);
  RSP_CUDA(cudaStreamSynchronize(s));  // k32 must outlive the async copy
  if (e != cudaSuccess) return fail(RSP_E_CUDA, "gather launch: %s", cudaGetErrorString(e));
  if (touched_bytes) *touched_bytes += static_cast<uint64_t>(nkept) * h->m_out * 4u;  // layer.cpp:91
  return RSP_OK;
}

rsp_status rsp_rspl_read(const char* path, rsp_rspl_header* hdr, float* w_cols, float* a_r, float* b_r,
                         uint32_t* comps) {
  return rspl_parse(path, hdr, w_cols, a_r, b_r, comps);
}

rsp_status rsp_linear_load_rspl(const char* path, const rsp_linear_desc* opts, rsp_linear** out) {
  if (!out) return fail(RSP_E_USAGE, "null output");
  *out = nullptr;
  rsp_rspl_header hd;
  if (rsp_status st = rspl_parse(path, &hd, nullptr, nullptr, nullptr, nullptr)) return st;
  std::vector<float> w(static_cast<size_t>(hd.m_in) * hd.m_out), a(static_cast<size_t>(hd.m_out) * hd.rank),
      b(static_cast<size_t>(hd.rank) * hd.m_in);
  std::vector<uint32_t> comps(hd.rank);
  if (rsp_status st = rspl_parse(path, &hd, w.data(), a.data(), b.data(), comps.data())) return st;
  rsp_linear_desc d = {};
  if (opts) d = *opts;
  else d.weight_dtype = RSP_F32;
  if (!opts) d.k_override = -1;
  d.m_in = hd.m_in;
  d.m_out = hd.m_out;
  d.rank = hd.rank;
  d.keep_fraction = hd.keep_fraction;
  d.src_dtype = RSP_F32;
  d.src_memory = RSP_MEM_HOST;
  d.w_layout = RSP_W_COL_MAJOR;
  d.w = w.data();
  d.a_r = hd.rank ? a.data() : nullptr;
  d.b_r = hd.rank ? b.data() : nullptr;
  if (rsp_status st = rsp_linear_create(&d, out)) return st;
  (*out)->comps = comps;
  return RSP_OK;
}

rsp_status rsp_linear_save_rspl(const rsp_linear* h, const char* path) {
  if (!h || !path) return fail(RSP_E_USAGE, "null handle or path");
  if (h->m != h->m_out) return fail(RSP_E_USAGE, "save_rspl: handle is a row shard (%u of %u rows)", h->m, h->m_out);
  DeviceGuard g(h->device);
  std::vector<float> w, a, b;
  // Wt[n][m_pad] -> w_cols data[j*m+i]: row j of Wt is column j of W
  if (rsp_status st = device_to_host_t(h, h->Wt, h->m_in, h->m, h->m_pad, &w)) return st;
  std::vector<float> wc(w.size());
  for (size_t j = 0; j < h->m_in; ++j)
    for (size_t i = 0; i < h->m; ++i) wc[j * h->m + i] = w[i * h->m_in + j];
  if (rsp_status st = device_to_host_t(h, h->At, h->rank, h->m, h->m_pad, &a)) return st;  // -> m x r
  if (rsp_status st = device_to_host_t(h, h->Bt, h->m_in, h->rank, h->r_pad, &b)) return st;  // -> r x n
  std::ofstream f(path, std::ios::binary);
  if (!f) return fail(RSP_E_IO, "cannot open layer file for writing: %s", path);
  const uint8_t version = 1;
  const uint32_t dims[4] = {h->m_in, h->m_out, h->rank,
                            static_cast<uint32_t>(std::ceil(h->keep_fraction * static_cast<double>(h->m_in)))};
  const double plan[2] = {h->keep_fraction, static_cast<double>(h->rank)};
  f.write("RSPL", 4);
  f.write(reinterpret_cast<const char*>(&version), 1);
  f.write(reinterpret_cast<const char*>(dims), sizeof(dims));
  f.write(reinterpret_cast<const char*>(wc.data()), static_cast<std::streamsize>(wc.size() * 4));
  f.write(reinterpret_cast<const char*>(a.data()), static_cast<std::streamsize>(a.size() * 4));
  f.write(reinterpret_cast<const char*>(b.data()), static_cast<std::streamsize>(b.size() * 4));
  f.write(reinterpret_cast<const char*>(h->comps.data()), static_cast<std::streamsize>(h->comps.size() * 4));
  f.write(reinterpret_cast<const char*>(plan), sizeof(plan));
  if (!f) return fail(RSP_E_IO, "write failed: %s", path);
  return RSP_OK;
}

rsp_status rsp_linear_components(const rsp_linear* h, uint32_t* comps) {
  if (!h || (h->rank && !comps)) return fail(RSP_E_USAGE, "null handle or buffer");
  std::copy(h->comps.begin(), h->comps.end(), comps);
  return RSP_OK;
}

rsp_status rsp_linear_set_components(rsp_linear* h, const uint32_t* comps, uint32_t r) {
  if (!h || (r && !comps)) return fail(RSP_E_USAGE, "null handle or buffer");
  if (r != h->rank) return fail(RSP_E_USAGE, "%u components for a rank-%u layer", r, h->rank);
  h->comps.assign(comps, comps + r);
  return RSP_OK;
}

rsp_status rsp_aggregate_scores(const double* tokens, uint32_t T, uint32_t n, const double* sigma,
                                const double* vt, uint32_t k, double* scores, void* stream) {
  if (T == 0) return fail(RSP_E_USAGE, "aggregate_scores requires at least one token");  // scores.cpp:55
  if (n == 0 || k == 0) return RSP_OK;
  if (!tokens || !sigma || !vt || !scores) return fail(RSP_E_USAGE, "null buffer");
  const cudaError_t e = rsp::launch_scores(tokens, T, n, sigma, vt, k, scores, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? RSP_OK : fail(RSP_E_CUDA, "aggregate_scores: %s", cudaGetErrorString(e));
}

rsp_status rsp_select_components(const double* scores, uint32_t k, uint32_t n, uint32_t r, uint32_t* comps,
                                 double* mass, void* stream) {
  if (r > k)  // scores.cpp:74-77
    return fail(RSP_E_USAGE, "select_components: r=%u exceeds component count %u", r, k);
  if (k == 0) return RSP_OK;
  if (!scores || !mass || (r && !comps)) return fail(RSP_E_USAGE, "null buffer");
  const cudaError_t e = rsp::launch_select_components(scores, k, n, r, comps, mass, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? RSP_OK : fail(RSP_E_CUDA, "select_components: %s", cudaGetErrorString(e));
}

rsp_status rsp_split_factors(const double* u, uint32_t m, uint32_t ucols, const double* sigma, const double* vt,
                             uint32_t n, const uint32_t* comps, uint32_t r, double* a_r, double* b_r, void* stream) {
  if (r == 0) return RSP_OK;
  if (!u || !sigma || !vt || !comps || !a_r || !b_r) return fail(RSP_E_USAGE, "null buffer");
  const cudaError_t e =
      rsp::launch_split_factors(u, m, ucols, sigma, vt, n, comps, r, a_r, b_r, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? RSP_OK : fail(RSP_E_CUDA, "split_factors: %s", cudaGetErrorString(e));
}

namespace {
// The stand-alone selector keeps x and its histograms in one CTA's shared
// memory: refuse (RSP_E_UNSUPPORTED) before touching CUDA when this device's
// opt-in limit cannot hold them.
rsp_status selector_fits(uint32_t n, bool x_bf16) {
  int dev = 0;
  cudaGetDevice(&dev);
  const size_t need = rsp::select_smem_bytes(static_cast<int>(n), x_bf16);
  const int cap = device_props(dev).smem_optin;
  if (need > static_cast<size_t>(cap))
    return fail(RSP_E_UNSUPPORTED, "selector: n=%u needs %zu B of shared memory (device limit %d B)", n, need, cap);
  return RSP_OK;
}
}  // namespace

extern "C" rsp_status rsp_top_k_by_magnitude(const void* x, rsp_dtype xdt, uint32_t n, uint32_t k,
                                  int32_t* kept, int32_t* rest, void* stream) {
  if (k > n)  // matrix.cpp:101-104
    return fail(RSP_E_USAGE, "top_k_by_magnitude: k=%u exceeds vector length %u", k, n);
  if (rsp_status st = check_x_dtype(xdt)) return st;
  if (n == 0) return RSP_OK;
  if (!x) return fail(RSP_E_USAGE, "null x");
  if (rsp_status st = selector_fits(n, xdt == RSP_BF16)) return st;
  cudaError_t e = rsp::launch_select(x, xdt == RSP_BF16, static_cast<int>(n), static_cast<int>(k), kept, rest,
                                     nullptr, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(RSP_E_CUDA, "selector launch: %s", cudaGetErrorString(e));
  return RSP_OK;
}

rsp_status rsp_threshold_sparsify(const void* x, rsp_dtype xdt, uint32_t n, double s,
                                  float* sparse_x, int32_t* kept, uint32_t* k_out, void* stream) {
  uint32_t k = 0;
  if (rsp_status st = rsp_keep_count(s, n, &k)) return st;  // sparsity.cpp:22-27
  if (rsp_status st = check_x_dtype(xdt)) return st;
  if (k_out) *k_out = k;
  if (n == 0) return RSP_OK;
  if (rsp_status st = selector_fits(n, xdt == RSP_BF16)) return st;
  cudaError_t e = rsp::launch_select(x, xdt == RSP_BF16, static_cast<int>(n), static_cast<int>(k), kept, nullptr,
                                     sparse_x, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(RSP_E_CUDA, "selector launch: %s", cudaGetErrorString(e));
  return RSP_OK;
}

rsp_status rsp_linear_selected(const rsp_linear* h, const void* x, rsp_dtype xdt, int32_t* S_host,
                               uint32_t* k_out) {
  if (!h || !x || !S_host) return fail(RSP_E_USAGE, "null handle or buffer");
  if (rsp_status st = check_x_dtype(xdt)) return st;
  DeviceGuard g(h->device);
  int32_t* kd = nullptr;
  RSP_CUDA(cudaMalloc(&kd, sizeof(int32_t) * std::max<uint32_t>(h->k, 1)));
  cudaError_t e = rsp::launch_select(x, xdt == RSP_BF16, static_cast<int>(h->m_in), static_cast<int>(h->k), kd,
                                     nullptr, nullptr, nullptr);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(S_host, kd, sizeof(int32_t) * h->k, cudaMemcpyDeviceToHost);
  cudaFree(kd);
  if (e != cudaSuccess) return fail(RSP_E_CUDA, "selected: %s", cudaGetErrorString(e));
  if (k_out) *k_out = h->k;
  return RSP_OK;
}

rsp_status rsp_linear_io_cost(const rsp_linear* h, rsp_io_report* o) {
  if (!h || !o) return fail(RSP_E_USAGE, "null handle");
  // layer.cpp:125-140, evaluated on the whole layer
  const double m = h->m_out, n = h->m_in, r = h->rank;
  const uint64_t kept_cols = static_cast<uint64_t>(std::ceil(h->keep_fraction * n));
  o->dense_bytes = static_cast<uint64_t>(h->m_in) * h->m_out * 4u;
  o->touched_bytes = (kept_cols * h->m_out + static_cast<uint64_t>(h->rank) * (h->m_in + h->m_out)) * 4u;
  o->relative_cost = r * (m + n) / (m * n) + h->keep_fraction;
  // what the fused kernel streams for this shard (padded widths)
  const uint64_t k = h->k, nn = h->m_in;
  const bool lr = h->rank > 0 && k < nn;
  o->kernel_weight_bytes = static_cast<uint64_t>(h->es) *
                           (k * h->m_pad + (lr ? (nn - k) * h->r_pad + static_cast<uint64_t>(h->rank) * h->m_pad : 0));
  o->kernel_total_bytes = o->kernel_weight_bytes + 4u * nn + 4u * static_cast<uint64_t>(h->m);
  o->dense_weight_bytes = static_cast<uint64_t>(h->es) * nn * h->m_pad;
  return RSP_OK;
}

rsp_status rsp_linear_export(const rsp_linear* h, int which, double* out) {
  if (!h || !out) return fail(RSP_E_USAGE, "null handle or buffer");
  DeviceGuard g(h->device);
  const size_t n = h->m_in, m = h->m, r = h->rank;
  size_t rows, cols;  // device array shape
  const void* src;
  size_t ld;
  if (which == 0) {
    rows = n; cols = m; src = h->Wt; ld = h->m_pad;
  } else if (which == 1) {
    rows = r; cols = m; src = h->At; ld = h->m_pad;
  } else if (which == 2) {
    rows = n; cols = r; src = h->Bt; ld = h->r_pad;
  } else {
    return fail(RSP_E_USAGE, "export: which must be 0, 1 or 2");
  }
  if (rows * cols == 0) return RSP_OK;
  std::vector<uint8_t> buf(rows * ld * h->es);
  RSP_CUDA(cudaMemcpy(buf.data(), src, buf.size(), cudaMemcpyDeviceToHost));
  auto val = [&](size_t i, size_t j) -> double {
    const size_t idx = i * ld + j;
    if (h->es == 4) {
      float f;
      std::memcpy(&f, buf.data() + idx * 4, 4);
      return f;
    }
    uint16_t b;
    std::memcpy(&b, buf.data() + idx * 2, 2);
    const uint32_t u = static_cast<uint32_t>(b) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
  };
  // device [rows][cols] -> reference row-major transpose
  for (size_t i = 0; i < rows; ++i)
    for (size_t j = 0; j < cols; ++j) out[j * rows + i] = val(i, j);
  return RSP_OK;
}

rsp_status rsp_stack_create_ex(const rsp_linear* const* layers, uint32_t count, const void* const* x_devs,
                               rsp_dtype xdt, float* const* y_devs, int dense, const uint8_t* wait_prev,
                               rsp_stack** out) {
  return rsp_stack_create_ops(layers, count, x_devs, xdt, y_devs, dense, wait_prev, nullptr, out);
}

rsp_status rsp_stack_create_ops(const rsp_linear* const* layers, uint32_t count, const void* const* x_devs,
                                rsp_dtype xdt, float* const* y_devs, int dense, const uint8_t* wait_prev,
                                const uint8_t* x_ops, rsp_stack** out) {
  rsp_stack_spec sp = {};
  sp.layers = layers;
  sp.count = count;
  sp.x_devs = x_devs;
  sp.x_dtype = xdt;
  sp.y_devs = y_devs;
  sp.dense = dense;
  sp.wait_prev = wait_prev;
  sp.x_ops = x_ops;
  sp.npeer = 1;
  return rsp_stack_create_spec(&sp, out);
}

rsp_status rsp_stack_create_spec(const rsp_stack_spec* spec, rsp_stack** out) {
  if (!spec || !out) return fail(RSP_E_USAGE, "bad stack arguments");
  const rsp_linear* const* layers = spec->layers;
  const uint32_t count = spec->count;
  const void* const* x_devs = spec->x_devs;
  const rsp_dtype xdt = spec->x_dtype;
  float* const* y_devs = spec->y_devs;
  const int dense = spec->dense;
  const uint8_t* wait_prev = spec->wait_prev;
  const uint8_t* x_ops = spec->x_ops;
  const uint32_t npeer = spec->npeer ? spec->npeer : 1;
  if (npeer > static_cast<uint32_t>(rsp::kMaxPeers))
    return fail(RSP_E_USAGE, "npeer %u exceeds %d y destinations", npeer, rsp::kMaxPeers);
  if (npeer > 1 && !spec->y_peers) return fail(RSP_E_USAGE, "npeer > 1 needs y_peers");
  for (uint32_t i = 0; npeer > 1 && i < count * npeer; ++i)
    if (!spec->y_peers[i]) return fail(RSP_E_USAGE, "null y_peers[%u]", i);
  if (!layers || !x_devs || !y_devs || !out || count == 0) return fail(RSP_E_USAGE, "bad stack arguments");
  if (rsp_status st = check_x_dtype(xdt)) return st;
  const uint32_t xrank = spec->xrank;
  if (xrank > 0) {
    if (xrank > static_cast<uint32_t>(rsp::kMaxPeers)) return fail(RSP_E_USAGE, "xrank %u exceeds %d", xrank, rsp::kMaxPeers);
    if (npeer != xrank && !(xrank == 1 && npeer == 1))
      return fail(RSP_E_USAGE, "xrank %u needs npeer == xrank y destinations (got %u)", xrank, npeer);
    if (!spec->xctr || spec->xself >= xrank) return fail(RSP_E_USAGE, "xrank needs xctr[xrank] and xself < xrank");
    for (uint32_t p = 0; p < xrank; ++p)
      if (!spec->xctr[p]) return fail(RSP_E_USAGE, "null xctr[%u]", p);
    if (layers[0] && layers[0]->deterministic)
      return fail(RSP_E_UNSUPPORTED, "cross-process stacks do not support RSP_FLAG_DETERMINISTIC");
  }
  for (uint32_t i = 0; x_ops && i < count; ++i) {
    if (x_ops[i] > RSP_XOP_SILU_GATE) return fail(RSP_E_USAGE, "x_ops[%u] = %u is not an RSP_XOP_*", i, x_ops[i]);
    if (x_ops[i] == RSP_XOP_SILU_GATE && xdt != RSP_F32)
      return fail(RSP_E_USAGE, "RSP_XOP_SILU_GATE needs fp32 activations (the gated input is formed in fp32)");
  }
  *out = nullptr;
  const rsp_linear* h0 = layers[0];
  const int dev = h0->device;
  DeviceGuard g(dev);
  std::vector<LinDesc> descs(count);
  int grid = 1, n_max = 1, cap_w = 1, cap_u = 1, cap_a = 1, nb_pad = 4, r_pad_max = 8, ks_max = 1, m_pad_max = 8;
  size_t smem = 0;
  const bool det = h0->deterministic;
  const DevProps dpx = device_props(dev);
  for (uint32_t i = 0; i < count; ++i) {
    const rsp_linear* h = layers[i];
    if (!h) return fail(RSP_E_USAGE, "null layer %u", i);
    if (h->device != dev) return fail(RSP_E_USAGE, "stack layers must share one device");
    if (h->es != h0->es) return fail(RSP_E_USAGE, "stack layers must share one weight dtype");
    if (h->deterministic != det) return fail(RSP_E_USAGE, "stack layers must share the deterministic flag");
  }
  // Groups: a linear that does not wait for its predecessor shares its
  // input and runs beside it on a disjoint partition of the CTAs, sized by
  // its share of the group's bytes.  Deterministic mode shares one
  // partial-sum scratch, so there every linear waits for the previous one.
  std::vector<LaunchPlan> plans(count);
  std::vector<uint32_t> gstart(count);  // first linear of each linear's group
  uint32_t pg0 = 0, pg1 = 0;  // the previous group
  // CTA budget of the whole launch: the device's SMs, or fewer (spec.max_ctas)
  // so that several stacks -- e.g. the tokens of a small batch -- run side
  // by side on disjoint SMs
  const int sms = std::max(1, spec->max_ctas ? std::min(dpx.sms, static_cast<int>(spec->max_ctas)) : dpx.sms);
  // fewest CTAs a linear's column tiling accepts (tiles of <= 8 warp columns)
  auto min_ctas = [](const rsp_linear* h) {
    const int wcols = (static_cast<int>(h->m_pad * h->es / 16) + 31) / 32;
    return std::max(1, (wcols + 7) / 8);
  };
  for (uint32_t g0 = 0; g0 < count;) {
    uint32_t g1 = g0 + 1;
    // a group whose members cannot all get their minimum partition at once
    // is split; the later part then waits for the earlier (stricter order,
    // same results)
    int need = min_ctas(layers[g0]);
    while (g1 < count && !det && wait_prev && !wait_prev[g1] && need + min_ctas(layers[g1]) <= sms)
      need += min_ctas(layers[g1++]);
    for (uint32_t i = g0; i < g1; ++i) gstart[i] = g0;
    double tot = 0.0;
    std::vector<double> bytes(g1 - g0);
    for (uint32_t i = g0; i < g1; ++i) {
      const rsp_linear* h = layers[i];
      const uint32_t kk = dense ? h->m_in : h->k;
      const bool lr = !dense && h->rank > 0 && kk < h->m_in;
      // bytes of the linear (W rows of S, stage-1 rows of S^c, A_r rows);
      // weighting the stage-1 rows 0.7x / 1.5x / 2x in this split measured
      // within 0.2% of 1x
      bytes[i - g0] = static_cast<double>(h->es) *
                      (static_cast<double>(kk) * h->m_pad +
                       (lr ? static_cast<double>(h->m_in - kk) * h->r_pad + static_cast<double>(h->rank) * h->m_pad
                           : 0.0));
      tot += bytes[i - g0];
    }
    int cta0 = 0;
    for (uint32_t i = g0; i < g1; ++i) {
      int budget = g1 - g0 == 1 ? sms
                                : std::max(min_ctas(layers[i]),
                                           static_cast<int>(std::floor(sms * bytes[i - g0] / std::max(tot, 1.0))));
      int later = 0;  // leave every later member its minimum partition
      for (uint32_t j = i + 1; j < g1; ++j) later += min_ctas(layers[j]);
      budget = std::min(budget, sms - cta0 - later);
      if (rsp_status st = make_plan(*layers[i], dpx, &plans[i], std::max(1, budget))) return st;
      const bool wp = i > 0 && (i == g0);
      const int xop = (x_ops && x_ops[i] == RSP_XOP_SILU_GATE) ? rsp::kLinSiluGate : 0;
      descs[i] = lin_desc(layers[i], x_devs[i], y_devs[i], dense != 0, static_cast<int>(i),
                          (wp ? rsp::kLinWaitPrev : 0) | xop, &plans[i], cta0);
      if (wp) {
        descs[i].dep0 = static_cast<int>(pg0);
        descs[i].ndep = static_cast<int>(pg1 - pg0);
      }
      cta0 += plans[i].grid;
      grid = std::max(grid, cta0);
    }
    pg0 = g0;
    pg1 = g1;
    g0 = g1;
  }
  for (uint32_t i = 0; i < count; ++i) {
    const rsp_linear* h = layers[i];
    n_max = std::max(n_max, static_cast<int>(h->m_in));
    cap_w = std::max(cap_w, plans[i].cap_w);
    cap_u = std::max(cap_u, plans[i].cap_u);
    cap_a = std::max(cap_a, plans[i].cap_a);
    nb_pad = std::max(nb_pad, plans[i].nb_pad);
    r_pad_max = std::max(r_pad_max, static_cast<int>(h->r_pad));
    ks_max = std::max(ks_max, plans[i].k_splits);
    m_pad_max = std::max(m_pad_max, static_cast<int>(h->m_pad));
  }
  smem = rsp::stack_smem_bytes(n_max, xdt == RSP_BF16, cap_w, cap_u, cap_a, static_cast<int>(count));
  const DevProps& dp = dpx;
  if (smem > static_cast<size_t>(dp.smem_optin))
    return fail(RSP_E_UNSUPPORTED, "stack needs %zu B shared memory (> %d)", smem, dp.smem_optin);
  const WsLayout wl = WsLayout::make(static_cast<int>(count), nb_pad, r_pad_max, ks_max, m_pad_max);
  auto* s = new rsp_stack();
  s->device = dev;
  {
    const size_t xe = xdt == RSP_BF16 ? 2 : 4;
    uintptr_t xl = UINTPTR_MAX, xh = 0, yl = UINTPTR_MAX, yh = 0;
    for (uint32_t i = 0; i < count; ++i) {
      const uintptr_t xa = reinterpret_cast<uintptr_t>(x_devs[i]), ya = reinterpret_cast<uintptr_t>(y_devs[i]);
      xl = std::min(xl, xa);
      xh = std::max(xh, xa + xe * layers[i]->m_in * ((x_ops && x_ops[i] == RSP_XOP_SILU_GATE) ? 2 : 1));
      yl = std::min(yl, ya);
      yh = std::max(yh, ya + sizeof(float) * layers[i]->m);
    }
    s->x_lo = reinterpret_cast<uint8_t*>(xl);
    s->y_lo = reinterpret_cast<uint8_t*>(yl);
    s->x_span = xh - xl;
    s->y_span = yh - yl;
  }
  cudaStream_t cs = nullptr;
  cudaError_t e = cudaMalloc(&s->ws, wl.bytes);
  if (e == cudaSuccess) e = cudaMemset(s->ws, 0, wl.bytes);
  if (e == cudaSuccess) e = cudaMalloc(&s->descs, sizeof(LinDesc) * count);
  if (e == cudaSuccess) e = cudaMemcpy(s->descs, descs.data(), sizeof(LinDesc) * count, cudaMemcpyHostToDevice);
  // Completion arrivals go to one counter per group (the slot of its first
  // linear): a dependent group polls one counter, not one per linear (each
  // poll is an L2 round trip).
  // (garr = the arrivals its group's counter collects per launch: the CTA
  // that completes it publishes the group to the other ranks)
  std::vector<int> garr(count, 0);
  for (uint32_t i = 0; i < count; ++i) garr[gstart[i]] += descs[i].grid;
  std::vector<rsp::LinCtl> ctl(count);
  for (uint32_t i = 0; i < count; ++i)
    ctl[i] = rsp::LinCtl{descs[i].flags, descs[i].dep0, descs[i].ndep, descs[i].cta0, descs[i].grid, descs[i].slot,
                         descs[gstart[i]].slot, garr[gstart[i]]};
  if (e == cudaSuccess && npeer > 1) {
    std::vector<float*> tab(static_cast<size_t>(count) * rsp::kMaxPeers, nullptr);
    for (uint32_t i = 0; i < count; ++i)
      for (uint32_t p = 0; p < npeer; ++p) tab[static_cast<size_t>(i) * rsp::kMaxPeers + p] = spec->y_peers[i * npeer + p];
    e = cudaMalloc(&s->ypeer, sizeof(float*) * tab.size());
    if (e == cudaSuccess) e = cudaMemcpy(s->ypeer, tab.data(), sizeof(float*) * tab.size(), cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess && xrank > 0) {
    e = cudaMalloc(&s->xctr, sizeof(unsigned long long*) * xrank);
    if (e == cudaSuccess)
      e = cudaMemcpy(s->xctr, spec->xctr, sizeof(unsigned long long*) * xrank, cudaMemcpyHostToDevice);
  }
  s->grids.resize(count);
  for (uint32_t i = 0; i < count; ++i) s->grids[i] = static_cast<uint32_t>(descs[i].grid);
  if (e == cudaSuccess) e = cudaMalloc(&s->ctl, sizeof(rsp::LinCtl) * count);
  if (e == cudaSuccess) e = cudaMemcpy(s->ctl, ctl.data(), sizeof(rsp::LinCtl) * count, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&s->plans, static_cast<size_t>(count) * grid * rsp::kPlanBytes);
  if (e == cudaSuccess)
    e = rsp::launch_plans(s->descs, static_cast<int>(count), grid,
                          rsp::stack_acopy_bytes(n_max, xdt == RSP_BF16, cap_w, cap_u, cap_a, static_cast<int>(count)),
                          h0->es, s->plans, cs);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
  if (e == cudaSuccess) e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
  if (e == cudaSuccess) {
    StackParams p = {};
    p.descs = s->descs;
    p.one = descs[0];
    p.count = static_cast<int>(count);
    p.n_max = n_max;
    p.cap_w = cap_w;
    p.cap_u = cap_u;
    p.cap_a = cap_a;
    p.nb_pad = nb_pad;
    p.deterministic = det ? 1 : 0;
    p.zero = 0u;
    p.ypeer = s->ypeer;
    p.npeer = static_cast<int>(npeer);
    p.xctr = s->xctr;
    p.xlocal = xrank > 0 ? spec->xctr[spec->xself] : nullptr;
    p.xrank = static_cast<int>(xrank);
    p.xslots = static_cast<int>(count);  // arrival words [0, count) (group slots), then the start fence
    p.plans = s->plans;
    p.ctl = s->ctl;
    bind_workspace(&p, s->ws, wl);
    s->params = p;
    s->es = h0->es;
    s->grid = grid;
    s->x_bf16 = xdt == RSP_BF16;
    s->smem = smem;
    s->pdl = h0->pdl;
    const cudaError_t el = rsp::launch_stack(p, h0->es, xdt == RSP_BF16, grid, smem, cs, h0->pdl);
    cudaGraph_t graph = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(cs, &graph);
    s->graph = graph;
    e = el != cudaSuccess ? el : ec;
  }
  if (e == cudaSuccess) e = cudaGraphInstantiate(&s->exec, s->graph, 0);
  if (cs) cudaStreamDestroy(cs);
  if (e != cudaSuccess) {
    rsp_stack_destroy(s);
    return fail(RSP_E_CUDA, "stack graph: %s", cudaGetErrorString(e));
  }
  *out = s;
  return RSP_OK;
}

rsp_status rsp_stack_create(const rsp_linear* const* layers, uint32_t count, const void* const* x_devs,
                            rsp_dtype xdt, float* const* y_devs, int dense, rsp_stack** out) {
  return rsp_stack_create_ex(layers, count, x_devs, xdt, y_devs, dense, nullptr, out);
}

rsp_status rsp_stack_launch(rsp_stack* s, void* stream) {
  if (!s) return fail(RSP_E_USAGE, "null stack");
  DeviceGuard g(s->device);
  RSP_CUDA(cudaGraphLaunch(s->exec, static_cast<cudaStream_t>(stream)));
  return RSP_OK;
}

rsp_status rsp_stack_launch_direct(rsp_stack* s, void* stream) {
  if (!s) return fail(RSP_E_USAGE, "null stack");
  DeviceGuard g(s->device);
  cudaError_t e = rsp::launch_stack(s->params, s->es, s->x_bf16, s->grid, s->smem, static_cast<cudaStream_t>(stream),
                                    s->pdl);
  if (e != cudaSuccess) return fail(RSP_E_CUDA, "stack launch: %s", cudaGetErrorString(e));
  return RSP_OK;
}

rsp_status rsp_stack_io_spans(const rsp_stack* s, size_t* x_bytes, size_t* y_bytes) {
  if (!s) return fail(RSP_E_USAGE, "null stack");
  if (x_bytes) *x_bytes = s->x_span;
  if (y_bytes) *y_bytes = s->y_span;
  return RSP_OK;
}

rsp_status rsp_stack_launch_host(rsp_stack* s, const void* x_host, size_t x_bytes, void* y_host, size_t y_bytes,
                                 void* stream) {
  if (!s || !x_host || !y_host) return fail(RSP_E_USAGE, "null stack or buffer");
  if (x_bytes != s->x_span || y_bytes != s->y_span)
    return fail(RSP_E_USAGE, "host buffers of %zu / %zu bytes do not match the stack's x / y spans (%zu / %zu)",
                x_bytes, y_bytes, s->x_span, s->y_span);
  DeviceGuard g(s->device);
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  RSP_CUDA(cudaMemcpyAsync(s->x_lo, x_host, x_bytes, cudaMemcpyHostToDevice, cs));
  RSP_CUDA(cudaGraphLaunch(s->exec, cs));
  RSP_CUDA(cudaMemcpyAsync(y_host, s->y_lo, y_bytes, cudaMemcpyDeviceToHost, cs));
  RSP_CUDA(cudaStreamSynchronize(cs));
  return RSP_OK;
}

rsp_status rsp_debug_stack_trace(rsp_stack* s, int64_t* trace_dev, uint32_t* grid_out, void* stream) {
  if (!s || !trace_dev) return fail(RSP_E_USAGE, "null stack or trace buffer");
  DeviceGuard g(s->device);
  StackParams p = s->params;
  p.trace = reinterpret_cast<long long*>(trace_dev);
  cudaError_t e = rsp::launch_stack(p, s->es, s->x_bf16, s->grid, s->smem, static_cast<cudaStream_t>(stream), false);
  if (e != cudaSuccess) return fail(RSP_E_CUDA, "stack trace launch: %s", cudaGetErrorString(e));
  if (grid_out) *grid_out = static_cast<uint32_t>(s->grid);
  return RSP_OK;
}

size_t rsp_stack_exchange_words(uint32_t count) { return static_cast<size_t>(count) + 1; }

rsp_status rsp_stack_grids(const rsp_stack* s, uint32_t* grids, uint32_t count) {
  if (!s || !grids || count != s->grids.size()) return fail(RSP_E_USAGE, "rsp_stack_grids: null or count mismatch");
  std::copy(s->grids.begin(), s->grids.end(), grids);
  return RSP_OK;
}

rsp_status rsp_ipc_alloc(int device, size_t bytes, void** dev_ptr) {
  if (!dev_ptr || bytes == 0) return fail(RSP_E_USAGE, "rsp_ipc_alloc: null pointer or zero bytes");
  DeviceGuard g(device);
  RSP_CUDA(cudaMalloc(dev_ptr, bytes));  // its own allocation: an IPC handle maps exactly this block
  RSP_CUDA(cudaMemset(*dev_ptr, 0, bytes));
  return RSP_OK;
}

rsp_status rsp_ipc_free(void* dev_ptr) {
  RSP_CUDA(cudaFree(dev_ptr));
  return RSP_OK;
}

rsp_status rsp_ipc_export(const void* dev_ptr, void* handle_out) {
  static_assert(sizeof(cudaIpcMemHandle_t) <= RSP_IPC_HANDLE_BYTES, "IPC handle size");
  if (!dev_ptr || !handle_out) return fail(RSP_E_USAGE, "rsp_ipc_export: null pointer");
  cudaIpcMemHandle_t h;
  RSP_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)));
  std::memset(handle_out, 0, RSP_IPC_HANDLE_BYTES);
  std::memcpy(handle_out, &h, sizeof(h));
  return RSP_OK;
}

rsp_status rsp_ipc_open(int device, const void* handle, void** dev_ptr) {
  if (!handle || !dev_ptr) return fail(RSP_E_USAGE, "rsp_ipc_open: null pointer");
  DeviceGuard g(device);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  RSP_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return RSP_OK;
}

rsp_status rsp_ipc_close(void* dev_ptr) {
  RSP_CUDA(cudaIpcCloseMemHandle(dev_ptr));
  return RSP_OK;
}

void rsp_stack_destroy(rsp_stack* s) {
  if (!s) return;
  DeviceGuard g(s->device);
  if (s->exec) cudaGraphExecDestroy(s->exec);
  if (s->graph) cudaGraphDestroy(s->graph);
  cudaFree(s->ws);
  cudaFree(s->descs);
  cudaFree(s->plans);
  cudaFree(s->ctl);
  cudaFree(s->ypeer);
  cudaFree(s->xctr);
  delete s;
}

}  // extern "C"
