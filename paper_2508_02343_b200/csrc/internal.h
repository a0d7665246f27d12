// internal.h -- launch interfaces between the C-ABI layer (mm_api.cpp) and the
// sm_100a kernels.  Not part of the public ABI (that is include/mm.h).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <cstdint>
#include <vector>
#include <cstdlib>
#include <utility>

namespace mmx {

enum : int { F_E2M1 = 0, F_E3M2 = 1, F_E2M3 = 2, F_E4M3 = 3, F_E5M2 = 4 };

// Geometry of one quantized operand derived from a plan (see include/mm.h).
struct SegGeom {
  int n[3];        // channels per segment
  int kp[3];       // stored (padded) columns per segment = roundup(n, 128)
  int off[3];      // start of the segment in the reordered channel order
  int fmt[3];      // element format per segment
  int sc_off[3];   // Eq. 1 exponent offset per segment (emax or bias)
  int64_t pitch[3];  // code bytes per row
};

// Dynamic shared memory the reorder-quantize kernel may use for its ring, gather
// table and norm scratch (the 227 KB opt-in limit minus alignment and barriers).
constexpr size_t kRqSmemBudget = 227 * 1024 - 2048;

struct RqArgs {
  const uint16_t* x;   // BF16 bits [rows, ldx]
  int64_t rows;
  int64_t ldx;
  int K;
  const int32_t* perm; // device int32[K]
  SegGeom geom;
  uint8_t* codes[3];
  uint8_t* sf[3];
  const uint32_t* layout; // gather-slot layout (one u32 per 32-channel line) or nullptr (layout.cpp)
  const uint16_t* gamma;  // BF16 [K] RMSNorm weight, or nullptr (no norm; F2 fusion)
  double eps;             // RMSNorm epsilon (> 0) when gamma != nullptr
};

// Plan-time gather layout (layout.cpp).
std::vector<uint32_t> gather_layout(int K, const int n[3], const int32_t* perm);
long long gather_wavefronts(int K, const int n[3], const int32_t* perm, const uint32_t* layout);

// Fused reorder-and-quantize (rq.cu).
cudaError_t launch_reorder_quantize(const RqArgs& a, cudaStream_t s, int64_t* launches);
// Test entry: gathered BF16 x_r (rq.cu).
cudaError_t launch_reorder_bf16(const uint16_t* x, int64_t rows, int64_t ldx, int K,
                                const int32_t* perm, uint16_t* xr, int64_t ldxr,
                                cudaStream_t s, int64_t* launches);

// Calibration statistics (calib.cu): chmax (double), chmean (double) on device.
size_t calib_workspace_bytes(int64_t L, int K);
cudaError_t launch_calib_stats(const uint16_t* x, int64_t L, int64_t ldx, int K,
                               void* ws, double* d_chmax, double* d_chmean,
                               cudaStream_t s, int64_t* launches);

// Streaming calibration (calib.cu): state = [256-byte header: int64 rows][K x 24-byte
// per-channel partials]; accumulate adds one batch; the host turns the state into stats.
size_t calib_state_bytes(int K);
cudaError_t launch_calib_accumulate(const uint16_t* x, int64_t L, int64_t ldx, int K, void* ws, void* state,
                                    cudaStream_t s, int64_t* launches);
void calib_state_to_stats(const void* h_state, int K, double* chmax, double* chmean, int64_t* rows);

struct GemmArgs {
  int64_t M, N;
  SegGeom geom;
  const uint8_t* a_codes[3];
  const uint8_t* a_sf[3];
  const uint8_t* w_codes[3];
  const uint8_t* w_sf[3];
  uint16_t* y;   // BF16 [M, ldy]
  int64_t ldy;
  // Fused all-gather epilogue (NEXT F1): n_dst > 0 stores every tile into each
  // y_dst[d] + y_col_off (the ranks' full Y buffers, this rank's column slice).
  int n_dst = 0;
  uint16_t* y_dst[8] = {};
  int64_t y_col_off = 0;
  // Fused all-gather over NVLS (multicast): y_mc != nullptr stores every output element
  // with multimem.st into the multicast view of all ranks' Y (columns + y_col_off).
  uint16_t* y_mc = nullptr;
  // Caller-owned GEMM workspace (split-K partials / stream-K partials + flags),
  // zero-filled before its first use; the kernels leave every counter at zero.
  void* ws = nullptr;
  size_t ws_bytes = 0;
};
constexpr int kMaxPeers = 8;

struct GemmConfig {
  int block_n = 0;      // 0 = auto
  int num_stages = 0;   // 0 = auto
  int max_ctas = 0;     // 0 = #SMs
  bool no_stream_k = false;  // keep the data-parallel tiling (N-shard path: shard-independent results)
  bool no_workspace = false; // never pick a path that needs the workspace (N-shard entry points)
  int cluster_pairs = 0;     // CTA-pair GEMM: pairs per cluster (1, 2; 0 = default / MM_GEMM_CP)
};

// Mixed block-scaled GEMM (gemm.cu).
cudaError_t launch_mixed_gemm(const GemmArgs& a, const GemmConfig& cfg, cudaStream_t s,
                              int64_t* launches, const char** err);
// Workspace bytes the launch of `a` under `cfg` needs (0: none); the per-kernel parts.
size_t gemm_workspace_bytes(const GemmArgs& a, const GemmConfig& cfg);
size_t smallm_workspace_bytes(const GemmArgs& a, const GemmConfig& cfg);
size_t pair_workspace_bytes(const GemmArgs& a, const GemmConfig& cfg);
constexpr size_t ws_align(size_t b) { return (b + 255) / 256 * 256; }

// [G][M][Ns] -> [M][G*Ns] layout fix after the all-gather (comm.cu).
cudaError_t launch_gather_layout(const uint16_t* stage, int G, int64_t M, int64_t Ns,
                                 uint16_t* y, int64_t ldy, cudaStream_t s, int64_t* launches);

// Peer-window flag arrays (one per rank, mapped into this process) and the barrier
// that follows a fused all-gather GEMM (comm.cu).
struct PeerFlags {
  uint32_t* f[kMaxPeers];
};
constexpr int kPeerErrSlot = 63;   // flag-array word holding a barrier timeout (missing rank + 1)
// NVLS barrier: every rank adds 1 to word 0 of the multicast flag array (all ranks' copies)
// and waits until its own copy reaches world * epoch (comm.cu).
cudaError_t launch_mc_barrier(uint32_t* flags_mc, uint32_t* flags_local, int world, uint32_t epoch,
                              uint64_t timeout_ns, cudaStream_t s, int64_t* launches);
cudaError_t launch_peer_barrier(const PeerFlags& fl, int rank, int world, uint32_t epoch, uint64_t timeout_ns,
                                cudaStream_t s, int64_t* launches);

int sm_count();

// cuTensorMapEncodeTiled resolved through the runtime (no libcuda link); nullptr if
// the driver does not provide it (gemm.cu).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn tensor_map_encoder();

// 2-D K-major operand map of segment g (inner = K bytes, or FP6 elements via the
// 16U6_ALIGN16B type; box 128 x box_rows; 128-byte swizzle) and the block-scaled
// tcgen05 instruction descriptor for an M x N MMA of segment g (gemm.cu).
bool make_operand_map(CUtensorMap* m, const void* base, int g, int kp, int64_t rows, int64_t pitch, int box_rows);
uint32_t make_idesc_mn(int fmt, int g, int m, int n);
cudaError_t launch_mixed_gemm_smallm(const GemmArgs& a, const GemmConfig& cfg, cudaStream_t s, int64_t* launches,
                                     const char** err);
cudaError_t launch_mixed_gemm_2cta(const GemmArgs& a, const GemmConfig& cfg, cudaStream_t s, int64_t* launches,
                                   const char** err);

// Host-side launch caches (per device, thread-safe): raise a kernel's dynamic
// shared-memory limit once, and remember occupancy queries, so the hot calls do
// no redundant driver work per launch.
cudaError_t ensure_smem_attr(const void* func, size_t smem);

// Launch with programmatic stream serialization (PDL): the kernel's prologue
// overlaps the tail of the preceding kernel; the kernel itself calls
// griddepcontrol.wait before touching dependent memory.  MM_NO_PDL=1 disables it.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  static const bool no_pdl = [] { const char* e = getenv("MM_NO_PDL"); return e && atoi(e); }();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = no_pdl ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
// Same, with a thread-block cluster of `cluster` CTAs along x.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_cluster(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, int cluster,
                               Args&&... args) {
  static const bool no_pdl = [] { const char* e = getenv("MM_NO_PDL"); return e && atoi(e); }();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = no_pdl ? 1 : 2;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
cudaError_t cached_occupancy(const void* func, int threads, size_t smem, int* per_sm);

// NCCL entry points resolved with dlopen (comm.cu).
struct NcclApi {
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclAllGather) allGather = nullptr;
  decltype(&ncclGetErrorString) errStr = nullptr;
  bool ok = false;
};
const NcclApi& nccl();

}  // namespace mmx
