// mm_api.cpp -- the C ABI of include/mm.h: argument validation, plan geometry,
// fingerprints, the host half of calibration (thresholds, counts, argsort), and
// dispatch to the sm_100a kernels.  Citations: include/mm.h and DESIGN.md.
#include "../../include/mm.h"

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <sys/syscall.h>
#include <unistd.h>
#include <map>
#include <mutex>
#include <tuple>
#include <numeric>
#include <string>
#include <vector>

#include "internal.h"

namespace mmx {


namespace {

thread_local std::string g_err;
thread_local int64_t g_launches = 0;
GemmConfig g_gemm_cfg;
std::mutex g_cfg_mu;

mm_status fail(mm_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

mm_status cuda_fail(cudaError_t e, const char* what) {
  return fail(MM_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

mm_status check_device() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  int major = 0, minor = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0)
    return fail(MM_ERR_UNSUPPORTED_DEVICE, "device %d is sm_%d%d; this library is built for sm_100a (B200)", dev,
                major, minor);
  return MM_OK;
}

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

int64_t roundup(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

int bits_of(int g) { return g == 0 ? 4 : (g == 1 ? 6 : 8); }

int emax_of(int fmt) {
  switch (fmt) {
    case F_E2M1: return 2;
    case F_E3M2: return 4;
    case F_E2M3: return 2;
    case F_E4M3: return 8;
    default: return 15;  // E5M2
  }
}
int bias_of(int fmt) {
  switch (fmt) {
    case F_E2M1: return 1;
    case F_E3M2: return 3;
    case F_E2M3: return 1;
    case F_E4M3: return 7;
    default: return 15;
  }
}
double qmax_of(int fmt) {
  switch (fmt) {
    case F_E2M1: return 6.0;
    case F_E3M2: return 28.0;
    case F_E2M3: return 7.5;
    case F_E4M3: return 448.0;
    default: return 57344.0;
  }
}

mm_status validate_plan_fields(int32_t K, const int32_t n[3], int32_t fmt6, int32_t fmt8, int32_t rule) {
  if (K < 32 || K % 32 != 0 || K > 65536) return fail(MM_ERR_SHAPE, "K=%d must be a multiple of 32 in [32, 65536]", K);
  int64_t s = 0;
  for (int g = 0; g < 3; ++g) {
    if (n[g] < 0 || n[g] % 32 != 0) return fail(MM_ERR_SHAPE, "n[%d]=%d must be a non-negative multiple of 32", g, n[g]);
    s += n[g];
  }
  if (s != K) return fail(MM_ERR_SHAPE, "n4+n6+n8=%lld != K=%d", (long long)s, K);
  if (fmt6 != MM_E3M2 && fmt6 != MM_E2M3) return fail(MM_ERR_INVALID_ARGUMENT, "fmt6 must be E3M2 or E2M3");
  if (fmt8 != MM_E4M3 && fmt8 != MM_E5M2) return fail(MM_ERR_INVALID_ARGUMENT, "fmt8 must be E4M3 or E5M2");
  if (rule != MM_SCALE_OCP && rule != MM_SCALE_PAPER_EQ1) return fail(MM_ERR_INVALID_ARGUMENT, "bad scale rule");
  return MM_OK;
}

mm_status validate_plan(const mm_plan* p) {
  if (!p) return fail(MM_ERR_INVALID_ARGUMENT, "plan is NULL");
  mm_status st = validate_plan_fields(p->K, p->n, p->fmt6, p->fmt8, p->rule);
  if (st != MM_OK) return st;
  if (!p->d_perm) return fail(MM_ERR_INVALID_ARGUMENT, "plan.d_perm is NULL");
  return MM_OK;
}

SegGeom geom_of(const mm_plan* p) {
  SegGeom G{};
  const int fmts[3] = {F_E2M1, p->fmt6, p->fmt8};
  int off = 0;
  for (int g = 0; g < 3; ++g) {
    G.n[g] = p->n[g];
    G.kp[g] = (int)roundup(p->n[g], 128);
    G.off[g] = off;
    off += p->n[g];
    G.fmt[g] = fmts[g];
    G.sc_off[g] = p->rule == MM_SCALE_OCP ? emax_of(fmts[g]) : bias_of(fmts[g]);
    G.pitch[g] = (int64_t)G.kp[g] * bits_of(g) / 8;
  }
  return G;
}

uint64_t fingerprint(int32_t K, const int32_t n[3], int32_t fmt6, int32_t fmt8, int32_t rule, const int32_t* perm) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](uint32_t v) {
    for (int i = 0; i < 4; ++i) {
      h ^= (v >> (8 * i)) & 0xFF;
      h *= 1099511628211ull;
    }
  };
  mix((uint32_t)K);
  for (int g = 0; g < 3; ++g) mix((uint32_t)n[g]);
  mix((uint32_t)fmt6);
  mix((uint32_t)fmt8);
  mix((uint32_t)rule);
  for (int32_t k = 0; k < K; ++k) mix((uint32_t)perm[k]);
  return h | 1ull;  // never 0 (0 = "no plan")
}

// Shared memory the reorder-quantize kernel needs for this K (R = 1 layout).
bool rq_fits(int32_t K) { return (size_t)((K + 255) / 256) * 512 * 2 <= kRqSmemBudget; }   // >= 2 one-row stages

mm_status check_mx_out(const mm_plan* p, const mm_mx_tensor* t, int64_t rows, const char* what) {
  if (!t) return fail(MM_ERR_INVALID_ARGUMENT, "%s is NULL", what);
  for (int g = 0; g < 3; ++g) {
    if (p->n[g] == 0) continue;
    if (!t->codes[g] || !t->sf[g]) return fail(MM_ERR_INVALID_ARGUMENT, "%s segment %d buffers are NULL", what, g);
    if (!aligned(t->codes[g], 256) || !aligned(t->sf[g], 256))
      return fail(MM_ERR_ALIGNMENT, "%s segment %d buffers must be 256-byte aligned", what, g);
  }
  (void)rows;
  return MM_OK;
}

mm_status run_rq(const void* d_x, int64_t rows, int64_t ldx, const mm_plan* plan, mm_mx_tensor* out,
                 mm_stream_t stream, const char* what, const void* d_gamma = nullptr, double eps = 0.0) {
  mm_status st = check_device();
  if (st != MM_OK) return st;
  if ((st = validate_plan(plan)) != MM_OK) return st;
  if (rows < 0) return fail(MM_ERR_SHAPE, "rows < 0");
  if (!d_x && rows > 0) return fail(MM_ERR_INVALID_ARGUMENT, "input is NULL");
  if (ldx < plan->K) return fail(MM_ERR_SHAPE, "ld=%lld < K=%d", (long long)ldx, plan->K);
  if (ldx % 8 != 0 || !aligned(d_x, 16)) return fail(MM_ERR_ALIGNMENT, "input rows must be 16-byte aligned");
  if (!rq_fits(plan->K)) return fail(MM_ERR_SHAPE, "K=%d exceeds the shared-memory capacity of the RQ kernel", plan->K);
  if ((st = check_mx_out(plan, out, rows, what)) != MM_OK) return st;
  out->rows = rows;
  out->fingerprint = plan->fingerprint;
  if (rows == 0) return MM_OK;
  RqArgs a{};
  a.x = static_cast<const uint16_t*>(d_x);
  a.rows = rows;
  a.ldx = ldx;
  a.K = plan->K;
  a.perm = plan->d_perm;
  a.layout = plan->d_layout;
  a.geom = geom_of(plan);
  a.gamma = static_cast<const uint16_t*>(d_gamma);
  a.eps = eps;
  for (int g = 0; g < 3; ++g) {
    a.codes[g] = static_cast<uint8_t*>(out->codes[g]);
    a.sf[g] = static_cast<uint8_t*>(out->sf[g]);
  }
  cudaError_t e = launch_reorder_quantize(a, reinterpret_cast<cudaStream_t>(stream), &g_launches);
  if (e != cudaSuccess) return cuda_fail(e, "reorder-quantize launch");
  return MM_OK;
}

}  // namespace

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = v > 0 ? v : 1;
  }
  return cached[dev];
}

namespace {
std::mutex g_cache_mu;
std::map<std::pair<const void*, int>, size_t> g_smem_attr;
std::map<std::tuple<const void*, int, int, size_t>, int> g_occ;
}  // namespace

cudaError_t ensure_smem_attr(const void* func, size_t smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_cache_mu);
  size_t& cur = g_smem_attr[{func, dev}];
  if (smem <= cur) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) cur = smem;
  return e;
}

cudaError_t cached_occupancy(const void* func, int threads, size_t smem, int* per_sm) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_cache_mu);
  auto key = std::make_tuple(func, dev, threads, smem);
  auto it = g_occ.find(key);
  if (it != g_occ.end()) { *per_sm = it->second; return cudaSuccess; }
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, func, threads, smem);
  if (e == cudaSuccess) g_occ[key] = *per_sm;
  return e;
}

}  // namespace mmx

using namespace mmx;

extern "C" {

int32_t mm_abi_version(void) { return 3; }   // 2: caller GEMM workspace, N-shard stage bytes, peer timeout; 3: plan gather layout
const char* mm_last_error(void) { return g_err.c_str(); }
int64_t mm_launch_count(void) { return g_launches; }
void mm_reset_launch_count(void) { g_launches = 0; }

int64_t mm_padded_cols(const mm_plan* p, int seg) {
  if (!p || seg < 0 || seg > 2 || p->n[seg] < 0) return -1;
  return roundup(p->n[seg], 128);
}
int64_t mm_code_pitch_bytes(const mm_plan* p, int seg) {
  int64_t kp = mm_padded_cols(p, seg);
  return kp < 0 ? -1 : kp * bits_of(seg) / 8;
}
int64_t mm_codes_bytes(const mm_plan* p, int64_t rows, int seg) {
  int64_t pitch = mm_code_pitch_bytes(p, seg);
  return (pitch < 0 || rows < 0) ? -1 : rows * pitch;
}
int64_t mm_sf_bytes(const mm_plan* p, int64_t rows, int seg) {
  int64_t kp = mm_padded_cols(p, seg);
  return (kp < 0 || rows < 0) ? -1 : roundup(rows, 128) * kp / 32;
}
int64_t mm_calib_workspace_bytes(int64_t L, int32_t K) {
  if (L < 0 || K <= 0) return -1;
  return (int64_t)roundup((int64_t)calib_workspace_bytes(L, K), 256) + 2 * (int64_t)roundup((int64_t)K * 8, 256);
}

mm_status mm_set_gemm_config(int32_t block_n, int32_t num_stages, int32_t max_ctas) {
  if (block_n != 0 && block_n != 1 && block_n != 128 && block_n != 256 && block_n != 512)
    return fail(MM_ERR_INVALID_ARGUMENT,
                "block_n must be 0 (auto), 1 (small-M swap-AB kernel, M <= 128), 128, 256 (one CTA) or 512 (CTA pair)");
  std::lock_guard<std::mutex> lk(g_cfg_mu);
  g_gemm_cfg.block_n = block_n;
  g_gemm_cfg.num_stages = num_stages;
  g_gemm_cfg.max_ctas = max_ctas;
  return MM_OK;
}

mm_status mm_plan_init(mm_plan* out, int32_t K, const int32_t n[3], int32_t fmt6, int32_t fmt8, int32_t rule,
                       const int32_t* h_perm, int32_t* d_perm_storage, mm_stream_t stream) {
  if (!out || !n || !h_perm || !d_perm_storage) return fail(MM_ERR_INVALID_ARGUMENT, "NULL argument");
  mm_status st = validate_plan_fields(K, n, fmt6, fmt8, rule);
  if (st != MM_OK) return st;
  std::vector<char> seen(K, 0);
  for (int32_t j = 0; j < K; ++j) {
    if (h_perm[j] < 0 || h_perm[j] >= K || seen[h_perm[j]])
      return fail(MM_ERR_INVALID_ARGUMENT, "permutation is not a bijection on [0, K) (position %d)", j);
    seen[h_perm[j]] = 1;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(d_perm_storage, h_perm, (size_t)K * 4, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "copy permutation");
  std::memset(out, 0, sizeof(*out));
  out->K = K;
  for (int g = 0; g < 3; ++g) out->n[g] = n[g];
  out->fmt6 = fmt6;
  out->fmt8 = fmt8;
  out->rule = rule;
  out->d_perm = d_perm_storage;
  out->fingerprint = fingerprint(K, n, fmt6, fmt8, rule, h_perm);
  return MM_OK;
}

int64_t mm_gather_layout_words(int32_t K) { return (K > 0 && K % 32 == 0) ? K / 32 : -1; }

static bool layout_args_ok(int32_t K, const int32_t n[3], const int32_t* h_perm) {
  if (!n || !h_perm || K <= 0 || K % 32 != 0 || K > 65536) return false;
  int64_t sum = 0;
  for (int g = 0; g < 3; ++g) {
    if (n[g] < 0 || n[g] % 32 != 0) return false;
    sum += n[g];
  }
  if (sum != K) return false;
  for (int32_t j = 0; j < K; ++j)
    if (h_perm[j] < 0 || h_perm[j] >= K) return false;
  return true;
}

mm_status mm_gather_layout_host(int32_t K, const int32_t n[3], const int32_t* h_perm, uint32_t* h_layout_out) {
  if (!h_layout_out || !layout_args_ok(K, n, h_perm)) return fail(MM_ERR_INVALID_ARGUMENT, "bad K / n / permutation");
  const std::vector<uint32_t> lay = gather_layout(K, n, h_perm);
  std::memcpy(h_layout_out, lay.data(), lay.size() * 4);
  return MM_OK;
}

int64_t mm_gather_wavefronts(int32_t K, const int32_t n[3], const int32_t* h_perm, const uint32_t* h_layout) {
  if (!layout_args_ok(K, n, h_perm)) return -1;
  return gather_wavefronts(K, n, h_perm, h_layout);
}

mm_status mm_plan_set_gather_layout(mm_plan* plan, uint32_t* d_layout_storage, mm_stream_t stream) {
  mm_status st = validate_plan(plan);
  if (st != MM_OK) return st;
  if (!d_layout_storage || !aligned(d_layout_storage, 16))
    return fail(MM_ERR_ALIGNMENT, "layout storage must be non-NULL and 16-byte aligned");
  const int K = plan->K;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  std::vector<int32_t> perm(K);
  cudaError_t e = cudaMemcpyAsync(perm.data(), plan->d_perm, (size_t)K * 4, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "read the permutation");
  const std::vector<uint32_t> lay = gather_layout(K, plan->n, perm.data());
  e = cudaMemcpyAsync(d_layout_storage, lay.data(), lay.size() * 4, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "upload the layout");
  plan->d_layout = d_layout_storage;
  return MM_OK;
}

// Host half of calibration, shared by the one-shot and the streaming paths.
static mm_status plan_from_stats(const std::vector<double>& chmax, const std::vector<double>& chmean, int32_t K,
                                 int32_t fmt6, int32_t fmt8, int32_t rule, int32_t* d_perm_out, mm_plan* plan_out,
                                 mm_stream_t stream) {
  // Eq. 5: T(n) = 2^(b+n-1) max|X| / (254 q_max), one correctly rounded division.
  double tmax = 0.0;
  for (double v : chmax) tmax = std::max(tmax, v);
  if (!(tmax > 0.0)) return fail(MM_ERR_DEGENERATE, "calibration data has max|X| == 0");
  const double t4 = (std::ldexp(1.0, bias_of(F_E2M1) + 4 - 1) * tmax) / (254.0 * qmax_of(F_E2M1));
  const double t6 = (std::ldexp(1.0, bias_of(fmt6) + 6 - 1) * tmax) / (254.0 * qmax_of(fmt6));
  // Eq. 6 / Eq. 17: channel counts by channel max.
  int32_t c4 = 0, c6 = 0;
  for (double v : chmax) {
    if (v <= t4) ++c4;
    else if (v <= t6) ++c6;
  }
  const int32_t c8 = K - c4 - c6;
  // Rounding to whole 32-blocks: n8 up, then n6 up (capped), n4 the remainder.
  int32_t n[3];
  n[2] = (int32_t)roundup(c8, 32);
  n[1] = std::min((int32_t)roundup(c6, 32), K - n[2]);
  n[0] = K - n[2] - n[1];
  // Eq. 7 + Q3: stable ascending argsort of the channel means.
  std::vector<int32_t> perm(K);
  std::iota(perm.begin(), perm.end(), 0);
  std::stable_sort(perm.begin(), perm.end(), [&](int32_t a, int32_t b) { return chmean[a] < chmean[b]; });
  mm_status st = mm_plan_init(plan_out, K, n, fmt6, fmt8, rule, perm.data(), d_perm_out, stream);
  if (st != MM_OK) return st;
  plan_out->tensor_max = tmax;
  plan_out->t4 = t4;
  plan_out->t6 = t6;
  plan_out->c[0] = c4;
  plan_out->c[1] = c6;
  plan_out->c[2] = c8;
  return MM_OK;
}

mm_status mm_calibrate_thresholds(const void* d_x, int64_t L, int32_t K, int64_t ldx, int32_t fmt6, int32_t fmt8,
                                  int32_t rule, int32_t* d_perm_out, mm_plan* plan_out, void* d_ws, size_t ws_bytes,
                                  double* h_chmax, double* h_chmean, mm_stream_t stream) {
  mm_status st = check_device();
  if (st != MM_OK) return st;
  const int32_t nz[3] = {K, 0, 0};
  if ((st = validate_plan_fields(K, nz, fmt6, fmt8, rule)) != MM_OK) return st;
  if (!d_x || !d_perm_out || !plan_out || !d_ws) return fail(MM_ERR_INVALID_ARGUMENT, "NULL argument");
  if (L <= 0) return fail(MM_ERR_SHAPE, "L must be positive");
  if (ldx < K) return fail(MM_ERR_SHAPE, "ldx < K");
  if (ldx % 8 != 0 || !aligned(d_x, 16)) return fail(MM_ERR_ALIGNMENT, "input rows must be 16-byte aligned");
  if ((int64_t)ws_bytes < mm_calib_workspace_bytes(L, K) || !aligned(d_ws, 256))
    return fail(MM_ERR_WORKSPACE, "workspace too small or unaligned (need %lld bytes)",
                (long long)mm_calib_workspace_bytes(L, K));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  uint8_t* ws = static_cast<uint8_t*>(d_ws);
  const int64_t part_bytes = roundup((int64_t)calib_workspace_bytes(L, K), 256);
  double* d_chmax = reinterpret_cast<double*>(ws + part_bytes);
  double* d_chmean = reinterpret_cast<double*>(ws + part_bytes + roundup((int64_t)K * 8, 256));
  cudaError_t e = launch_calib_stats(static_cast<const uint16_t*>(d_x), L, ldx, K, ws, d_chmax, d_chmean, s,
                                     &g_launches);
  if (e != cudaSuccess) return cuda_fail(e, "calibration launch");
  std::vector<double> chmax(K), chmean(K);
  e = cudaMemcpyAsync(chmax.data(), d_chmax, (size_t)K * 8, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(chmean.data(), d_chmean, (size_t)K * 8, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "calibration statistics");
  if ((st = plan_from_stats(chmax, chmean, K, fmt6, fmt8, rule, d_perm_out, plan_out, stream)) != MM_OK) return st;
  if (h_chmax) std::memcpy(h_chmax, chmax.data(), (size_t)K * 8);
  if (h_chmean) std::memcpy(h_chmean, chmean.data(), (size_t)K * 8);
  return MM_OK;
}

int64_t mm_calib_state_bytes(int32_t K) { return K <= 0 ? -1 : (int64_t)calib_state_bytes(K); }

mm_status mm_calib_accumulate(const void* d_x, int64_t L, int32_t K, int64_t ldx, void* d_ws, size_t ws_bytes,
                              void* d_state, mm_stream_t stream) {
  mm_status st = check_device();
  if (st != MM_OK) return st;
  if (K < 32 || K % 32 != 0 || K > 65536) return fail(MM_ERR_SHAPE, "K=%d must be a multiple of 32 in [32, 65536]", K);
  if (!d_x || !d_ws || !d_state) return fail(MM_ERR_INVALID_ARGUMENT, "NULL argument");
  if (L <= 0) return fail(MM_ERR_SHAPE, "L must be positive");
  if (ldx < K) return fail(MM_ERR_SHAPE, "ldx < K");
  if (ldx % 8 != 0 || !aligned(d_x, 16)) return fail(MM_ERR_ALIGNMENT, "input rows must be 16-byte aligned");
  if (!aligned(d_state, 256)) return fail(MM_ERR_ALIGNMENT, "state must be 256-byte aligned");
  if ((int64_t)ws_bytes < mm_calib_workspace_bytes(L, K) || !aligned(d_ws, 256))
    return fail(MM_ERR_WORKSPACE, "workspace too small or unaligned (need %lld bytes)",
                (long long)mm_calib_workspace_bytes(L, K));
  cudaError_t e = launch_calib_accumulate(static_cast<const uint16_t*>(d_x), L, ldx, K, d_ws, d_state,
                                          reinterpret_cast<cudaStream_t>(stream), &g_launches);
  if (e != cudaSuccess) return cuda_fail(e, "calibration accumulate launch");
  return MM_OK;
}

mm_status mm_calib_finalize(const void* d_state, int32_t K, int32_t fmt6, int32_t fmt8, int32_t rule,
                            int32_t* d_perm_out, mm_plan* plan_out, double* h_chmax, double* h_chmean,
                            int64_t* h_rows, mm_stream_t stream) {
  mm_status st = check_device();
  if (st != MM_OK) return st;
  const int32_t nz[3] = {K, 0, 0};
  if ((st = validate_plan_fields(K, nz, fmt6, fmt8, rule)) != MM_OK) return st;
  if (!d_state || !d_perm_out || !plan_out) return fail(MM_ERR_INVALID_ARGUMENT, "NULL argument");
  std::vector<uint8_t> h(calib_state_bytes(K));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(h.data(), d_state, h.size(), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "calibration state");
  std::vector<double> chmax(K), chmean(K);
  int64_t rows = 0;
  calib_state_to_stats(h.data(), K, chmax.data(), chmean.data(), &rows);
  if (rows <= 0) return fail(MM_ERR_DEGENERATE, "no calibration rows accumulated");
  if ((st = plan_from_stats(chmax, chmean, K, fmt6, fmt8, rule, d_perm_out, plan_out, stream)) != MM_OK) return st;
  if (h_chmax) std::memcpy(h_chmax, chmax.data(), (size_t)K * 8);
  if (h_chmean) std::memcpy(h_chmean, chmean.data(), (size_t)K * 8);
  if (h_rows) *h_rows = rows;
  return MM_OK;
}

mm_status mm_plan_diagnostics(const mm_plan* plan, const double* h_chmax, const int32_t* h_perm,
                              mm_plan_diag* out) {
  if (!plan || !out) return fail(MM_ERR_INVALID_ARGUMENT, "NULL argument");
  mm_status st = validate_plan_fields(plan->K, plan->n, plan->fmt6, plan->fmt8, plan->rule);
  if (st != MM_OK) return st;
  const int32_t K = plan->K;
  std::memset(out, 0, sizeof(*out));
  for (int g = 0; g < 3; ++g) out->p[g] = (double)plan->n[g] / K;
  // Table 1 accounting: element bits + 8-bit E8M0 scale per 32 elements
  out->avg_bits = (4.0 * plan->n[0] + 6.0 * plan->n[1] + 8.0 * plan->n[2]) / K + 8.0 / 32.0;
  out->stored_bytes_per_row = 0;
  for (int g = 0; g < 3; ++g) out->stored_bytes_per_row += mm_code_pitch_bytes(plan, g) + roundup(plan->n[g], 128) / 32;
  if (h_chmax && h_perm && plan->t4 > 0.0) {
    // Eq. 6 violations: channels ordered by mean (Eq. 7) into a group whose threshold
    // their maximum exceeds (a diagnostic, never "fixed": DESIGN.md R13)
    for (int32_t j = 0; j < plan->n[0]; ++j) out->eq6_violations[0] += h_chmax[h_perm[j]] > plan->t4;
    for (int32_t j = plan->n[0]; j < plan->n[0] + plan->n[1]; ++j)
      out->eq6_violations[1] += h_chmax[h_perm[j]] > plan->t6;
  }
  return MM_OK;
}

mm_status mm_quantize_weight_offline(const void* d_w, int64_t N, int64_t ldw, const mm_plan* plan,
                                     mm_mx_tensor* w_out, mm_stream_t stream) {
  return run_rq(d_w, N, ldw, plan, w_out, stream, "w_out");
}

mm_status mm_reorder_quantize_act(const void* d_x, int64_t M, int64_t ldx, const mm_plan* plan, mm_mx_tensor* a_out,
                                  mm_stream_t stream) {
  return run_rq(d_x, M, ldx, plan, a_out, stream, "a_out");
}

mm_status mm_rmsnorm_reorder_quantize_act(const void* d_x, int64_t M, int64_t ldx, const void* d_gamma, double eps,
                                          const mm_plan* plan, mm_mx_tensor* a_out, mm_stream_t stream) {
  if (!d_gamma) return fail(MM_ERR_INVALID_ARGUMENT, "gamma is NULL");
  if (!(eps > 0.0) || !std::isfinite(eps)) return fail(MM_ERR_INVALID_ARGUMENT, "eps must be finite and > 0");
  if (!aligned(d_gamma, 16)) return fail(MM_ERR_ALIGNMENT, "gamma must be 16-byte aligned");
  return run_rq(d_x, M, ldx, plan, a_out, stream, "a_out", d_gamma, eps);
}

mm_status mm_reorder_act_bf16(const void* d_x, int64_t M, int64_t ldx, const mm_plan* plan, void* d_xr,
                              int64_t ldxr, mm_stream_t stream) {
  mm_status st = check_device();
  if (st != MM_OK) return st;
  if ((st = validate_plan(plan)) != MM_OK) return st;
  if (M < 0 || ldx < plan->K || ldxr < plan->K) return fail(MM_ERR_SHAPE, "bad shape");
  if (M > 0 && (!d_x || !d_xr)) return fail(MM_ERR_INVALID_ARGUMENT, "NULL buffer");
  cudaError_t e = launch_reorder_bf16(static_cast<const uint16_t*>(d_x), M, ldx, plan->K, plan->d_perm,
                                      static_cast<uint16_t*>(d_xr), ldxr, reinterpret_cast<cudaStream_t>(stream),
                                      &g_launches);
  if (e != cudaSuccess) return cuda_fail(e, "reorder launch");
  return MM_OK;
}

// Peer window of the fused all-gather epilogue (NEXT F1).
struct MmPeerWin {
  int rank = 0, world = 0;
  int64_t M = 0, ldy = 0;
  uint16_t* y[kMaxPeers] = {};
  uint32_t* flags[kMaxPeers] = {};
  void* ipc_base[kMaxPeers] = {};   // mappings opened by mm_peer_window_open (unmapped on close)
  uint32_t epoch = 0;
  uint64_t timeout_ns = 0;   // 0: the barrier waits forever (mm_peer_window_set_timeout)
};

static size_t peer_y_bytes(int64_t M, int64_t ldy) { return ((size_t)M * (size_t)ldy * 2 + 255) / 256 * 256; }

static GemmConfig current_cfg() {
  std::lock_guard<std::mutex> lk(g_cfg_mu);
  return g_gemm_cfg;
}

// d_ws / ws_bytes: caller workspace (see mm_gemm_workspace_bytes); no_ws = an entry
// point without a workspace argument (N-shard): never pick a path that needs one.
static mm_status gemm_common(const mm_mx_tensor* a, const mm_mx_tensor* w, const mm_plan* plan, void* d_y,
                             int64_t ldy, int64_t n_cols, mm_stream_t stream, void* d_ws, size_t ws_bytes,
                             bool no_ws, const MmPeerWin* win = nullptr, uint16_t* y_mc = nullptr,
                             int64_t mc_col_off = 0) {
  mm_status st = check_device();
  if (st != MM_OK) return st;
  if ((st = validate_plan(plan)) != MM_OK) return st;
  if (!a || !w) return fail(MM_ERR_INVALID_ARGUMENT, "operand is NULL");
  if (a->fingerprint != plan->fingerprint || w->fingerprint != plan->fingerprint)
    return fail(MM_ERR_PLAN_MISMATCH, "operands were not produced with this plan");
  if ((st = check_mx_out(plan, a, a->rows, "a")) != MM_OK) return st;
  if ((st = check_mx_out(plan, w, w->rows, "w")) != MM_OK) return st;
  const int64_t M = a->rows, N = w->rows;
  if (M < 0 || N < 0) return fail(MM_ERR_SHAPE, "negative rows");
  if (N % 16 != 0) return fail(MM_ERR_SHAPE, "N=%lld must be a multiple of 16", (long long)N);
  if (ldy < n_cols || ldy % 8 != 0) return fail(MM_ERR_SHAPE, "ldy=%lld must be >= N and a multiple of 8", (long long)ldy);
  if (M > 0 && N > 0 && (!d_y || !aligned(d_y, 16))) return fail(MM_ERR_ALIGNMENT, "Y must be 16-byte aligned");
  if (M == 0 || N == 0) return MM_OK;
  GemmArgs ga{};
  ga.M = M;
  ga.N = N;
  ga.geom = geom_of(plan);
  for (int g = 0; g < 3; ++g) {
    ga.a_codes[g] = static_cast<const uint8_t*>(a->codes[g]);
    ga.a_sf[g] = static_cast<const uint8_t*>(a->sf[g]);
    ga.w_codes[g] = static_cast<const uint8_t*>(w->codes[g]);
    ga.w_sf[g] = static_cast<const uint8_t*>(w->sf[g]);
  }
  ga.y = static_cast<uint16_t*>(d_y);
  ga.ldy = ldy;
  if (win) {
    ga.n_dst = win->world;
    for (int r = 0; r < win->world; ++r) ga.y_dst[r] = win->y[r];
    ga.y_col_off = (int64_t)win->rank * N;
  }
  if (y_mc) {   // NVLS: the multicast view of the full Y; this rank's columns start at mc_col_off
    ga.y_mc = y_mc;
    ga.y_col_off = mc_col_off;
  }
  GemmConfig cfg = current_cfg();
  cfg.no_stream_k = cfg.no_stream_k || no_ws;
  cfg.no_workspace = no_ws;
  const size_t need = gemm_workspace_bytes(ga, cfg);
  if (need > 0 && (!d_ws || ws_bytes < need || !aligned(d_ws, 256)))
    return fail(MM_ERR_WORKSPACE, "GEMM workspace: need %zu bytes (256-B aligned, zero-filled once), got %zu at %p",
                need, ws_bytes, d_ws);
  ga.ws = d_ws;
  ga.ws_bytes = ws_bytes;
  const char* err = "";
  cudaError_t e = launch_mixed_gemm(ga, cfg, reinterpret_cast<cudaStream_t>(stream), &g_launches, &err);
  if (e != cudaSuccess) return fail(MM_ERR_CUDA, "mixed GEMM launch: %s (%s)", cudaGetErrorString(e), err);
  return MM_OK;
}

mm_status mm_mixed_gemm_bf16(const mm_mx_tensor* a, const mm_mx_tensor* w, const mm_plan* plan, void* d_y,
                             int64_t ldy, void* d_ws, size_t ws_bytes, mm_stream_t stream) {
  return gemm_common(a, w, plan, d_y, ldy, w ? w->rows : 0, stream, d_ws, ws_bytes, false);
}

int64_t mm_gemm_workspace_bytes(const mm_plan* plan, int64_t M, int64_t N) {
  if (validate_plan(plan) != MM_OK || M < 0 || N < 0) return -1;
  GemmArgs ga{};
  ga.M = M;
  ga.N = N;
  ga.geom = geom_of(plan);
  return (int64_t)gemm_workspace_bytes(ga, current_cfg());
}

// ---------------------------------------------------------------- multi-GPU
struct MmComm {
  ncclComm_t comm;
  int rank, world;
};

int32_t mm_nccl_unique_id_bytes(void) { return (int32_t)sizeof(ncclUniqueId); }

mm_status mm_nccl_get_unique_id(void* h_id_out) {
  if (!h_id_out) return fail(MM_ERR_INVALID_ARGUMENT, "NULL id buffer");
  const NcclApi& api = nccl();
  if (!api.ok) return fail(MM_ERR_NCCL, "libnccl.so.2 could not be loaded");
  ncclUniqueId id;
  ncclResult_t r = api.getUniqueId(&id);
  if (r != ncclSuccess) return fail(MM_ERR_NCCL, "ncclGetUniqueId: %s", api.errStr(r));
  std::memcpy(h_id_out, &id, sizeof(id));
  return MM_OK;
}

mm_status mm_comm_init(int32_t rank, int32_t world, const void* h_unique_id, void** comm_out) {
  if (!h_unique_id || !comm_out) return fail(MM_ERR_INVALID_ARGUMENT, "NULL argument");
  if (world < 1 || rank < 0 || rank >= world) return fail(MM_ERR_INVALID_ARGUMENT, "bad rank/world");
  const NcclApi& api = nccl();
  if (!api.ok) return fail(MM_ERR_NCCL, "libnccl.so.2 could not be loaded");
  ncclUniqueId id;
  std::memcpy(&id, h_unique_id, sizeof(id));
  MmComm* c = new MmComm{nullptr, rank, world};
  ncclResult_t r = api.commInitRank(&c->comm, world, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(MM_ERR_NCCL, "ncclCommInitRank: %s", api.errStr(r));
  }
  *comm_out = c;
  return MM_OK;
}

mm_status mm_comm_destroy(void* comm) {
  if (!comm) return MM_OK;
  MmComm* c = static_cast<MmComm*>(comm);
  const NcclApi& api = nccl();
  if (api.ok && c->comm) api.commDestroy(c->comm);
  delete c;
  return MM_OK;
}

mm_status mm_mixed_gemm_bf16_nshard_allgather(const mm_mx_tensor* a, const mm_mx_tensor* w_shard,
                                              const mm_plan* plan, int64_t n_total, void* d_y_full, int64_t ldy,
                                              void* d_stage, size_t stage_bytes, void* comm, mm_stream_t stream) {
  if (!comm || !d_stage || !a || !w_shard) return fail(MM_ERR_INVALID_ARGUMENT, "NULL argument");
  MmComm* c = static_cast<MmComm*>(comm);
  const int64_t Ns = w_shard->rows;
  const int64_t M = a->rows;
  // every precondition is checked before anything is enqueued (the GEMM included)
  if (Ns * c->world != n_total) return fail(MM_ERR_SHAPE, "shard rows * world != n_total");
  if (Ns % 16 != 0) return fail(MM_ERR_SHAPE, "shard rows must be a multiple of 16");
  if (ldy < n_total || ldy % 8 != 0) return fail(MM_ERR_SHAPE, "bad ldy");
  if (!aligned(d_stage, 16)) return fail(MM_ERR_ALIGNMENT, "stage must be 16-byte aligned");
  if (M > 0 && n_total > 0 && (!d_y_full || !aligned(d_y_full, 16)))
    return fail(MM_ERR_ALIGNMENT, "Y must be non-NULL and 16-byte aligned");
  if (M > 0 && stage_bytes < (size_t)M * (size_t)n_total * 2)
    return fail(MM_ERR_WORKSPACE, "stage: need %lld bytes (BF16 [G][M][N/G]), got %zu",
                (long long)(M * n_total * 2), stage_bytes);
  const NcclApi& api = nccl();
  if (!api.ok) return fail(MM_ERR_NCCL, "libnccl.so.2 could not be loaded");
  uint16_t* stage = static_cast<uint16_t*>(d_stage);
  uint16_t* mine = stage + (int64_t)c->rank * M * Ns;
  mm_status st = gemm_common(a, w_shard, plan, mine, Ns, Ns, stream, nullptr, 0, /*no_ws=*/true);
  if (st != MM_OK) return st;
  if (M == 0 || Ns == 0) return MM_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  ncclResult_t r = api.allGather(mine, stage, (size_t)(M * Ns), ncclBfloat16, c->comm, s);
  if (r != ncclSuccess) return fail(MM_ERR_NCCL, "ncclAllGather: %s", api.errStr(r));
  cudaError_t e = launch_gather_layout(stage, c->world, M, Ns, static_cast<uint16_t*>(d_y_full), ldy, s, &g_launches);
  if (e != cudaSuccess) return cuda_fail(e, "layout launch");
  return MM_OK;
}

size_t mm_peer_buffer_bytes(int64_t M, int64_t ldy) {
  if (M < 0 || ldy < 0) return 0;
  return peer_y_bytes(M, ldy) + 64 * sizeof(uint32_t);
}

// IPC handle of the allocation containing d_buf + the byte offset of d_buf inside it
// (caching allocators such as PyTorch's sub-allocate cudaMalloc blocks).
int32_t mm_ipc_handle_bytes(void) { return (int32_t)(sizeof(cudaIpcMemHandle_t) + sizeof(uint64_t)); }

mm_status mm_ipc_get_handle(const void* d_buf, void* h_handle_out) {
  if (!d_buf || !h_handle_out) return fail(MM_ERR_INVALID_ARGUMENT, "NULL argument");
  typedef CUresult (*RangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
  static RangeFn range = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    return (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess) ? reinterpret_cast<RangeFn>(p) : nullptr;
  }();
  if (!range) return fail(MM_ERR_CUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<CUdeviceptr>(d_buf)) != CUDA_SUCCESS)
    return fail(MM_ERR_INVALID_ARGUMENT, "d_buf is not device memory");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
  const uint64_t off = (uint64_t)(reinterpret_cast<CUdeviceptr>(d_buf) - base);
  std::memcpy(h_handle_out, &h, sizeof(h));
  std::memcpy(static_cast<uint8_t*>(h_handle_out) + sizeof(h), &off, sizeof(off));
  return MM_OK;
}

static mm_status peer_window_check(int32_t rank, int32_t world, int64_t M, int64_t ldy) {
  if (world < 1 || world > kMaxPeers || rank < 0 || rank >= world)
    return fail(MM_ERR_INVALID_ARGUMENT, "rank %d / world %d (world must be 1..%d)", rank, world, kMaxPeers);
  if (M < 0 || ldy < 0 || ldy % 8 != 0) return fail(MM_ERR_SHAPE, "bad M / ldy (ldy %% 8 == 0)");
  return MM_OK;
}

mm_status mm_peer_window_from_ptrs(int32_t rank, int32_t world, void* const* h_dev_bufs, int64_t M, int64_t ldy,
                                   void** win_out) {
  mm_status st = peer_window_check(rank, world, M, ldy);
  if (st != MM_OK) return st;
  if (!h_dev_bufs || !win_out) return fail(MM_ERR_INVALID_ARGUMENT, "NULL argument");
  for (int r = 0; r < world; ++r)
    if (!h_dev_bufs[r] || !aligned(h_dev_bufs[r], 256)) return fail(MM_ERR_ALIGNMENT, "buffer %d: NULL or not 256-B aligned", r);
  MmPeerWin* w = new MmPeerWin;
  w->rank = rank;
  w->world = world;
  w->M = M;
  w->ldy = ldy;
  for (int r = 0; r < world; ++r) {
    w->y[r] = static_cast<uint16_t*>(h_dev_bufs[r]);
    w->flags[r] = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(h_dev_bufs[r]) + peer_y_bytes(M, ldy));
  }
  *win_out = w;
  return MM_OK;
}

mm_status mm_peer_window_open(int32_t rank, int32_t world, void* d_local_buf, const void* h_handles, int64_t M,
                              int64_t ldy, void** win_out) {
  mm_status st = peer_window_check(rank, world, M, ldy);
  if (st != MM_OK) return st;
  if (!d_local_buf || !h_handles || !win_out) return fail(MM_ERR_INVALID_ARGUMENT, "NULL argument");
  if (!aligned(d_local_buf, 256)) return fail(MM_ERR_ALIGNMENT, "local buffer must be 256-B aligned");
  void* bufs[kMaxPeers] = {};
  void* bases[kMaxPeers] = {};   // opened IPC mappings (allocation bases)
  bool opened[kMaxPeers] = {};
  for (int r = 0; r < world; ++r) {
    if (r == rank) { bufs[r] = d_local_buf; continue; }
    cudaIpcMemHandle_t h;
    uint64_t off = 0;
    const uint8_t* rec = static_cast<const uint8_t*>(h_handles) + (size_t)r * (sizeof(h) + sizeof(off));
    std::memcpy(&h, rec, sizeof(h));
    std::memcpy(&off, rec + sizeof(h), sizeof(off));
    cudaError_t e = cudaIpcOpenMemHandle(&bases[r], h, cudaIpcMemLazyEnablePeerAccess);
    if (e == cudaSuccess) bufs[r] = static_cast<uint8_t*>(bases[r]) + off;
    if (e != cudaSuccess) {
      for (int q = 0; q < r; ++q)
        if (opened[q]) cudaIpcCloseMemHandle(bases[q]);
      return cuda_fail(e, "cudaIpcOpenMemHandle");
    }
    opened[r] = true;
  }
  void* win = nullptr;
  st = mm_peer_window_from_ptrs(rank, world, bufs, M, ldy, &win);
  if (st != MM_OK) {
    for (int q = 0; q < world; ++q)
      if (opened[q]) cudaIpcCloseMemHandle(bases[q]);
    return st;
  }
  for (int q = 0; q < world; ++q) static_cast<MmPeerWin*>(win)->ipc_base[q] = opened[q] ? bases[q] : nullptr;
  *win_out = win;
  return MM_OK;
}

mm_status mm_peer_window_close(void* win) {
  if (!win) return MM_OK;
  MmPeerWin* w = static_cast<MmPeerWin*>(win);
  for (int r = 0; r < w->world; ++r)
    if (w->ipc_base[r]) cudaIpcCloseMemHandle(w->ipc_base[r]);
  delete w;
  return MM_OK;
}

mm_status mm_peer_barrier(void* win, mm_stream_t stream) {
  if (!win) return fail(MM_ERR_INVALID_ARGUMENT, "NULL window");
  mm_status st = check_device();
  if (st != MM_OK) return st;
  MmPeerWin* w = static_cast<MmPeerWin*>(win);
  PeerFlags fl{};
  for (int r = 0; r < w->world; ++r) fl.f[r] = w->flags[r];
  const uint32_t epoch = ++w->epoch;
  cudaError_t e = launch_peer_barrier(fl, w->rank, w->world, epoch, w->timeout_ns,
                                      reinterpret_cast<cudaStream_t>(stream), &g_launches);
  if (e != cudaSuccess) return cuda_fail(e, "peer barrier launch");
  return MM_OK;
}

mm_status mm_peer_window_set_timeout(void* win, double seconds) {
  if (!win || !(seconds >= 0.0)) return fail(MM_ERR_INVALID_ARGUMENT, "NULL window or negative timeout");
  static_cast<MmPeerWin*>(win)->timeout_ns = (uint64_t)(seconds * 1e9);
  return MM_OK;
}

mm_status mm_peer_window_error(void* win, int32_t* h_missing_rank) {
  if (!win || !h_missing_rank) return fail(MM_ERR_INVALID_ARGUMENT, "NULL argument");
  MmPeerWin* w = static_cast<MmPeerWin*>(win);
  uint32_t v = 0;
  cudaError_t e = cudaMemcpy(&v, w->flags[w->rank] + kPeerErrSlot, sizeof(v), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "reading the peer error word");
  *h_missing_rank = (int32_t)v - 1;
  return MM_OK;
}

// ---------------------------------------------------------------- NVLS (multicast) window
// NEXT F1 over NVLink SHARP: one multicast object spans every rank's Y buffer; the GEMM
// epilogue writes each output element ONCE with multimem.st and the NVSwitch replicates
// it to all ranks (per-GPU egress (G-1)x smaller than storing to each peer).  Built on
// the driver's virtual-memory API (resolved at run time; no libcuda link).
struct CuVmm {
  decltype(&cuMulticastCreate) mcCreate = nullptr;
  decltype(&cuMulticastAddDevice) mcAddDevice = nullptr;
  decltype(&cuMulticastBindMem) mcBindMem = nullptr;
  decltype(&cuMulticastUnbind) mcUnbind = nullptr;
  decltype(&cuMulticastGetGranularity) mcGranularity = nullptr;
  decltype(&cuMemCreate) memCreate = nullptr;
  decltype(&cuMemRelease) memRelease = nullptr;
  decltype(&cuMemAddressReserve) addrReserve = nullptr;
  decltype(&cuMemAddressFree) addrFree = nullptr;
  decltype(&cuMemMap) memMap = nullptr;
  decltype(&cuMemUnmap) memUnmap = nullptr;
  decltype(&cuMemSetAccess) setAccess = nullptr;
  decltype(&cuMemExportToShareableHandle) exportHandle = nullptr;
  decltype(&cuMemImportFromShareableHandle) importHandle = nullptr;
  decltype(&cuMemGetAllocationGranularity) allocGranularity = nullptr;
  decltype(&cuDeviceGet) deviceGet = nullptr;
  decltype(&cuDeviceGetAttribute) deviceAttr = nullptr;
  bool ok = false;
};
static const CuVmm& cuvmm() {
  static CuVmm api;
  static std::once_flag once;
  std::call_once(once, []() {
    auto get = [](const char* name) -> void* {
      void* p = nullptr;
      cudaDriverEntryPointQueryResult q;
      return (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess &&
              q == cudaDriverEntryPointSuccess) ? p : nullptr;
    };
    api.mcCreate = reinterpret_cast<decltype(api.mcCreate)>(get("cuMulticastCreate"));
    api.mcAddDevice = reinterpret_cast<decltype(api.mcAddDevice)>(get("cuMulticastAddDevice"));
    api.mcBindMem = reinterpret_cast<decltype(api.mcBindMem)>(get("cuMulticastBindMem"));
    api.mcUnbind = reinterpret_cast<decltype(api.mcUnbind)>(get("cuMulticastUnbind"));
    api.mcGranularity = reinterpret_cast<decltype(api.mcGranularity)>(get("cuMulticastGetGranularity"));
    api.memCreate = reinterpret_cast<decltype(api.memCreate)>(get("cuMemCreate"));
    api.memRelease = reinterpret_cast<decltype(api.memRelease)>(get("cuMemRelease"));
    api.addrReserve = reinterpret_cast<decltype(api.addrReserve)>(get("cuMemAddressReserve"));
    api.addrFree = reinterpret_cast<decltype(api.addrFree)>(get("cuMemAddressFree"));
    api.memMap = reinterpret_cast<decltype(api.memMap)>(get("cuMemMap"));
    api.memUnmap = reinterpret_cast<decltype(api.memUnmap)>(get("cuMemUnmap"));
    api.setAccess = reinterpret_cast<decltype(api.setAccess)>(get("cuMemSetAccess"));
    api.exportHandle = reinterpret_cast<decltype(api.exportHandle)>(get("cuMemExportToShareableHandle"));
    api.importHandle = reinterpret_cast<decltype(api.importHandle)>(get("cuMemImportFromShareableHandle"));
    api.allocGranularity = reinterpret_cast<decltype(api.allocGranularity)>(get("cuMemGetAllocationGranularity"));
    api.deviceGet = reinterpret_cast<decltype(api.deviceGet)>(get("cuDeviceGet"));
    api.deviceAttr = reinterpret_cast<decltype(api.deviceAttr)>(get("cuDeviceGetAttribute"));
    api.ok = api.mcCreate && api.mcAddDevice && api.mcBindMem && api.mcUnbind && api.mcGranularity &&
             api.memCreate && api.memRelease && api.addrReserve && api.addrFree && api.memMap && api.memUnmap &&
             api.setAccess && api.exportHandle && api.importHandle && api.allocGranularity && api.deviceGet &&
             api.deviceAttr;
  });
  return api;
}

// Shareable handle record exchanged by the caller (mm_mc_handle_bytes() bytes).
struct McHandleRec {
  uint32_t type;       // 0: none (world 1), 1: fabric handle, 2: POSIX fd (imported with pidfd_getfd)
  uint32_t pid;
  int32_t fd;
  uint32_t pad;
  uint8_t fabric[64];
};

struct MmMcWin {
  int rank = 0, world = 0, dev = 0;
  int64_t M = 0, ldy = 0;
  size_t bytes = 0;                      // mapped size (granularity-rounded)
  CUmemGenericAllocationHandle mc = 0, mem = 0;
  CUdeviceptr mc_va = 0, local_va = 0;
  bool bound = false;
  int exported_fd = -1;
  uint32_t epoch = 0;
  uint64_t timeout_ns = 0;
};

static mm_status cu_fail(CUresult r, const char* what) { return fail(MM_ERR_CUDA, "%s: CUresult %d", what, (int)r); }

int32_t mm_mc_handle_bytes(void) { return (int32_t)sizeof(McHandleRec); }

int32_t mm_mc_supported(void) {
  const CuVmm& api = cuvmm();
  if (!api.ok) return 0;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  CUdevice cd;
  if (api.deviceGet(&cd, dev) != CUDA_SUCCESS) return 0;
  int v = 0;
  if (api.deviceAttr(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cd) != CUDA_SUCCESS || !v) return 0;
  // The attribute is not enough: a box whose GPU is not attached to an NVSwitch fabric
  // rejects cuMulticastCreate (CUDA_ERROR_INVALID_VALUE).  Probe once per device.
  static std::mutex mu;
  static int probed[64] = {0};   // 0 unknown, 1 yes, 2 no
  std::lock_guard<std::mutex> lk(mu);
  if (dev >= 0 && dev < 64 && probed[dev]) return probed[dev] == 1;
  CUmulticastObjectProp mp{};
  mp.numDevices = 1;
  size_t g = 0;
  mp.size = 2u << 20;
  if (api.mcGranularity(&g, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED) == CUDA_SUCCESS && g > mp.size) mp.size = g;
  CUmemGenericAllocationHandle h = 0;
  const bool ok = api.mcCreate(&h, &mp) == CUDA_SUCCESS;
  if (ok) api.memRelease(h);
  if (dev >= 0 && dev < 64) probed[dev] = ok ? 1 : 2;
  return ok ? 1 : 0;
}

mm_status mm_mc_window_create(int32_t rank, int32_t world, int64_t M, int64_t ldy, void* h_handle, void** win_out) {
  mm_status st = peer_window_check(rank, world, M, ldy);
  if (st != MM_OK) return st;
  if (!win_out || (world > 1 && !h_handle)) return fail(MM_ERR_INVALID_ARGUMENT, "NULL argument");
  const CuVmm& api = cuvmm();
  if (!api.ok) return fail(MM_ERR_CUDA, "driver virtual-memory / multicast entry points unavailable");
  if (!mm_mc_supported()) return fail(MM_ERR_UNSUPPORTED_DEVICE, "device does not support multicast objects");
  MmMcWin* w = new MmMcWin;
  w->rank = rank;
  w->world = world;
  w->M = M;
  w->ldy = ldy;
  cudaGetDevice(&w->dev);
  CUdevice cd;
  api.deviceGet(&cd, w->dev);
  // size: [Y][64 flags], rounded to both granularities
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = w->dev;
  size_t ag = 0, mg = 0;
  CUmulticastObjectProp mp{};
  mp.numDevices = (unsigned)world;
  mp.size = mm_peer_buffer_bytes(M, ldy);
  CUresult r = api.allocGranularity(&ag, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
  if (r == CUDA_SUCCESS) r = api.mcGranularity(&mg, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED);
  if (r != CUDA_SUCCESS) { delete w; return cu_fail(r, "granularity"); }
  const size_t g = std::max(ag, mg);
  w->bytes = (mp.size + g - 1) / g * g;
  mp.size = w->bytes;
  McHandleRec* rec = static_cast<McHandleRec*>(h_handle);
  if (rank == 0) {
    // fabric handles first (IMEX), else a POSIX fd the peers duplicate with pidfd_getfd
    const CUmemAllocationHandleType types[2] = {CU_MEM_HANDLE_TYPE_FABRIC, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR};
    bool done = false;
    for (int k = 0; k < (world > 1 ? 2 : 1) && !done; ++k) {
      mp.handleTypes = world > 1 ? (unsigned long long)types[k] : 0ull;
      if (api.mcCreate(&w->mc, &mp) != CUDA_SUCCESS) continue;
      if (world == 1) { done = true; break; }
      McHandleRec out{};
      out.pid = (uint32_t)getpid();
      out.fd = -1;
      if (types[k] == CU_MEM_HANDLE_TYPE_FABRIC) {
        CUmemFabricHandle fh;
        if (api.exportHandle(&fh, w->mc, CU_MEM_HANDLE_TYPE_FABRIC, 0) == CUDA_SUCCESS) {
          out.type = 1;
          std::memcpy(out.fabric, fh.data, sizeof(out.fabric));
          done = true;
        }
      } else {
        int fd = -1;
        if (api.exportHandle(&fd, w->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0) == CUDA_SUCCESS) {
          out.type = 2;
          out.fd = fd;
          w->exported_fd = fd;
          done = true;
        }
      }
      if (done) *rec = out;
      else { api.memRelease(w->mc); w->mc = 0; }
    }
    if (!done) { delete w; return fail(MM_ERR_CUDA, "cuMulticastCreate / export of the multicast handle failed"); }
  } else {
    if (rec->type == 1) {
      CUmemFabricHandle fh;
      std::memcpy(fh.data, rec->fabric, sizeof(rec->fabric));
      r = api.importHandle(&w->mc, &fh, CU_MEM_HANDLE_TYPE_FABRIC);
    } else if (rec->type == 2) {
      const int pidfd = (int)syscall(434 /* SYS_pidfd_open */, (int)rec->pid, 0);
      const int fd = pidfd >= 0 ? (int)syscall(438 /* SYS_pidfd_getfd */, pidfd, rec->fd, 0) : -1;
      if (pidfd >= 0) close(pidfd);
      if (fd < 0) { delete w; return fail(MM_ERR_CUDA, "pidfd_getfd of the multicast handle failed"); }
      r = api.importHandle(&w->mc, reinterpret_cast<void*>((uintptr_t)fd), CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
      close(fd);
    } else {
      delete w;
      return fail(MM_ERR_INVALID_ARGUMENT, "bad multicast handle record");
    }
    if (r != CUDA_SUCCESS) { delete w; return cu_fail(r, "import multicast handle"); }
  }
  r = api.mcAddDevice(w->mc, cd);
  if (r != CUDA_SUCCESS) { api.memRelease(w->mc); delete w; return cu_fail(r, "cuMulticastAddDevice"); }
  *win_out = w;
  return MM_OK;
}

mm_status mm_mc_window_bind(void* win) {
  if (!win) return fail(MM_ERR_INVALID_ARGUMENT, "NULL window");
  MmMcWin* w = static_cast<MmMcWin*>(win);
  if (w->bound) return MM_OK;
  const CuVmm& api = cuvmm();
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = w->dev;
  CUresult r = api.memCreate(&w->mem, w->bytes, &ap, 0);
  if (r != CUDA_SUCCESS) return cu_fail(r, "cuMemCreate");
  r = api.mcBindMem(w->mc, 0, w->mem, 0, w->bytes, 0);
  if (r != CUDA_SUCCESS) return cu_fail(r, "cuMulticastBindMem");
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = w->dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  r = api.addrReserve(&w->local_va, w->bytes, 0, 0, 0);
  if (r == CUDA_SUCCESS) r = api.memMap(w->local_va, w->bytes, 0, w->mem, 0);
  if (r == CUDA_SUCCESS) r = api.setAccess(w->local_va, w->bytes, &acc, 1);
  if (r != CUDA_SUCCESS) return cu_fail(r, "map the local buffer");
  r = api.addrReserve(&w->mc_va, w->bytes, 0, 0, 0);
  if (r == CUDA_SUCCESS) r = api.memMap(w->mc_va, w->bytes, 0, w->mc, 0);
  if (r == CUDA_SUCCESS) r = api.setAccess(w->mc_va, w->bytes, &acc, 1);
  if (r != CUDA_SUCCESS) return cu_fail(r, "map the multicast view");
  cudaError_t e = cudaMemset(reinterpret_cast<void*>(w->local_va), 0, w->bytes);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_fail(e, "zero the window");
  w->bound = true;
  return MM_OK;
}

void* mm_mc_window_local(void* win) {
  return win ? reinterpret_cast<void*>(static_cast<MmMcWin*>(win)->local_va) : nullptr;
}

mm_status mm_mc_window_set_timeout(void* win, double seconds) {
  if (!win || !(seconds >= 0.0)) return fail(MM_ERR_INVALID_ARGUMENT, "NULL window or negative timeout");
  static_cast<MmMcWin*>(win)->timeout_ns = (uint64_t)(seconds * 1e9);
  return MM_OK;
}

mm_status mm_mc_window_error(void* win, int32_t* h_timed_out) {
  if (!win || !h_timed_out) return fail(MM_ERR_INVALID_ARGUMENT, "NULL argument");
  MmMcWin* w = static_cast<MmMcWin*>(win);
  if (!w->bound) return fail(MM_ERR_INVALID_ARGUMENT, "window not bound");
  uint32_t v = 0;
  cudaError_t e = cudaMemcpy(&v, reinterpret_cast<uint32_t*>(w->local_va + peer_y_bytes(w->M, w->ldy)) + kPeerErrSlot,
                             sizeof(v), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "reading the window error word");
  *h_timed_out = v ? 1 : 0;
  return MM_OK;
}

mm_status mm_mc_window_close(void* win) {
  if (!win) return MM_OK;
  MmMcWin* w = static_cast<MmMcWin*>(win);
  const CuVmm& api = cuvmm();
  cudaDeviceSynchronize();
  if (w->mc_va) { api.memUnmap(w->mc_va, w->bytes); api.addrFree(w->mc_va, w->bytes); }
  if (w->local_va) { api.memUnmap(w->local_va, w->bytes); api.addrFree(w->local_va, w->bytes); }
  CUdevice cd;
  api.deviceGet(&cd, w->dev);
  if (w->bound) api.mcUnbind(w->mc, cd, 0, w->bytes);
  if (w->mem) api.memRelease(w->mem);
  if (w->mc) api.memRelease(w->mc);
  if (w->exported_fd >= 0) close(w->exported_fd);
  delete w;
  return MM_OK;
}

mm_status mm_mc_barrier(void* win, mm_stream_t stream) {
  if (!win) return fail(MM_ERR_INVALID_ARGUMENT, "NULL window");
  MmMcWin* w = static_cast<MmMcWin*>(win);
  if (!w->bound) return fail(MM_ERR_INVALID_ARGUMENT, "window not bound (mm_mc_window_bind)");
  const size_t yb = peer_y_bytes(w->M, w->ldy);
  uint32_t* f_mc = reinterpret_cast<uint32_t*>(w->mc_va + yb);
  uint32_t* f_loc = reinterpret_cast<uint32_t*>(w->local_va + yb);
  const uint32_t epoch = ++w->epoch;
  cudaError_t e = launch_mc_barrier(f_mc, f_loc, w->world, epoch, w->timeout_ns, reinterpret_cast<cudaStream_t>(stream),
                                    &g_launches);
  if (e != cudaSuccess) return cuda_fail(e, "NVLS barrier launch");
  return MM_OK;
}

mm_status mm_mixed_gemm_bf16_nshard_nvls(const mm_mx_tensor* a, const mm_mx_tensor* w_shard, const mm_plan* plan,
                                         int64_t n_total, void* win, int32_t barrier, mm_stream_t stream) {
  if (!win || !a || !w_shard) return fail(MM_ERR_INVALID_ARGUMENT, "NULL argument");
  MmMcWin* w = static_cast<MmMcWin*>(win);
  if (!w->bound) return fail(MM_ERR_INVALID_ARGUMENT, "window not bound (mm_mc_window_bind)");
  const int64_t Ns = w_shard->rows;
  if (Ns * w->world != n_total) return fail(MM_ERR_SHAPE, "shard rows * world != n_total");
  if (Ns % 16 != 0) return fail(MM_ERR_SHAPE, "shard rows must be a multiple of 16");
  if (a->rows != w->M) return fail(MM_ERR_SHAPE, "activation rows %lld != window M %lld", (long long)a->rows, (long long)w->M);
  if (w->ldy < n_total) return fail(MM_ERR_SHAPE, "window ldy < n_total");
  uint16_t* y_loc = reinterpret_cast<uint16_t*>(w->local_va);
  mm_status st = gemm_common(a, w_shard, plan, y_loc + (int64_t)w->rank * Ns, w->ldy, Ns, stream, nullptr, 0,
                             /*no_ws=*/true, nullptr, reinterpret_cast<uint16_t*>(w->mc_va), (int64_t)w->rank * Ns);
  if (st != MM_OK) return st;
  if (barrier) return mm_mc_barrier(win, stream);
  return MM_OK;
}

mm_status mm_mixed_gemm_bf16_nshard_peerstore(const mm_mx_tensor* a, const mm_mx_tensor* w_shard,
                                              const mm_plan* plan, int64_t n_total, void* win, int32_t barrier,
                                              mm_stream_t stream) {
  if (!win || !a || !w_shard) return fail(MM_ERR_INVALID_ARGUMENT, "NULL argument");
  MmPeerWin* w = static_cast<MmPeerWin*>(win);
  const int64_t Ns = w_shard->rows;
  if (Ns * w->world != n_total) return fail(MM_ERR_SHAPE, "shard rows * world != n_total");
  if (Ns % 16 != 0) return fail(MM_ERR_SHAPE, "shard rows must be a multiple of 16");
  if (a->rows != w->M) return fail(MM_ERR_SHAPE, "activation rows %lld != window M %lld", (long long)a->rows, (long long)w->M);
  if (w->ldy < n_total) return fail(MM_ERR_SHAPE, "window ldy < n_total");
  mm_status st = gemm_common(a, w_shard, plan, w->y[w->rank] + (int64_t)w->rank * Ns, w->ldy, Ns, stream,
                             nullptr, 0, /*no_ws=*/true, w);
  if (st != MM_OK) return st;
  if (barrier) return mm_peer_barrier(win, stream);
  return MM_OK;
}

}  // extern "C"
