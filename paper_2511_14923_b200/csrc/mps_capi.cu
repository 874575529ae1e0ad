// mps_capi.cu — the C ABI (include/mps_sampler.h) over the sm_100a kernels.
//
// One context per GPU per process.  A context owns: the resident site tensors
// Gamma^[m] (or borrowed device pointers), their TMA descriptors, the per-batch
// workspaces (state ping-pong, C buffer, staged inputs/outputs) and a stream.
// Per mode it launches K1 (site_gemm_kernel) then K2+K3 (displace_draw_kernel);
// there is no host synchronisation inside the mode loop.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdlib>
#include <utility>
#include <cstdio>
#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <tuple>
#include <cstring>
#include <set>
#include <string>
#include <vector>

#include "../../include/mps_sampler.h"
#include "c64_gemm.cuh"
#include "displace_draw.cuh"
#include "ozaki_gemm.cuh"
#include "site_gemm.cuh"
#include "chain_small.cuh"
#include "chain_small2.cuh"
#include "chain_tiny.cuh"

using namespace mps;


namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D row-major float64 matrix (rows x cols doubles, row pitch in bytes), box {box_cols, box_rows};
// 16-double boxes use the 128B swizzle, 8-double boxes (sum planes of the state) the 64B one.
// Encoding a tensor map costs microseconds of host time, as much as a launch: small chains
// (chi ~ 100) re-encode the same few maps every mode, so they are cached by their arguments.
struct TmapKey {
  const void* base;
  uint64_t rows, cols, pitch;
  uint32_t box_rows, box_cols;
  int kind;
  bool operator<(const TmapKey& o) const {
    return std::tie(base, rows, cols, pitch, box_rows, box_cols, kind) <
           std::tie(o.base, o.rows, o.cols, o.pitch, o.box_rows, o.box_cols, o.kind);
  }
};
static std::map<TmapKey, CUtensorMap> g_tmap_cache;
static std::mutex g_tmap_mu;

static bool tmap_cached(CUtensorMap* map, const TmapKey& k) {
  std::lock_guard<std::mutex> lk(g_tmap_mu);
  auto it = g_tmap_cache.find(k);
  if (it == g_tmap_cache.end()) return false;
  *map = it->second;
  return true;
}
static void tmap_store(const CUtensorMap& map, const TmapKey& k) {
  std::lock_guard<std::mutex> lk(g_tmap_mu);
  if (g_tmap_cache.size() > 4096) g_tmap_cache.clear();  // buffers get reallocated: keep it bounded
  g_tmap_cache[k] = map;
}

bool make_tmap(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t pitch_bytes,
               uint32_t box_rows, uint32_t box_cols = 16, bool fp32 = false) {
  const TmapKey key{base, rows, cols, pitch_bytes, box_rows, box_cols, fp32 ? 1 : 0};
  if (tmap_cached(map, key)) return true;
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {pitch_bytes};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  const uint32_t box_bytes = box_cols * (fp32 ? 4 : 8);
  CUresult r = enc(map, fp32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   box_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  tmap_store(*map, key);
  return true;
}

inline int round_up(int x, int m) { return (x + m - 1) / m * m; }

// K bytes of a real-doubled Ozaki operand row (2 chi_l int8), padded to whole 32-byte k steps
inline int oz_ld(int K) { return round_up(2 * K, 32); }

// fp32 plane row pitch (floats): TMA needs 16-byte row strides
inline int plane_ld(int cols_fp32) { return (cols_fp32 + 3) & ~3; }

// sum-plane row pitch (doubles): TMA needs 16-byte row strides
inline int sum_ld(int cols) { return (cols + 1) & ~1; }

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

struct Site {
  int chi_l = 0, chi_r = 0;
  double2* data = nullptr;
  bool owned = false;
  CUtensorMap tmap;
  double* gsum = nullptr;  // sum plane Gr + Gi (chi_l x sum_ld(N)) for the 3M GEMM, or null
  CUtensorMap tmap_gs;
  bool loaded = false;
  // host-streamed site (MPS_SITE_HOST_STREAM): pinned host copy, uploaded per call into a ring slot
  const double2* host = nullptr;
  bool registered = false;  // we cudaHostRegister'ed it (unregister on release)
  // Ozaki (int8 tcgen05) digit planes of B_r^T, built on first use in gemm mode 8
  int8_t* oz = nullptr;
  int* oz_e = nullptr;
  int oz_S = 0, oz_ld = 0, oz_pad = 0;
  // small-chain kernel copy of the site (chain_site_kernel layout), for chi_l <= 128, chi_r D <= 1024
  double2* chain = nullptr;
  // complex64 sites: only the tcgen05 operand planes are kept (B_r^T hi / lo, 2N x ld fp32)
  float* bhi = nullptr;
  float* blo = nullptr;
  int ld = 0;
  void release() {
    if (owned && data) cudaFree(data);
    if (gsum) cudaFree(gsum);
    if (bhi) cudaFree(bhi);
    if (blo) cudaFree(blo);
    if (oz) cudaFree(oz);
    if (oz_e) cudaFree(oz_e);
    if (chain) cudaFree(chain);
    chain = nullptr;
    if (registered && host) cudaHostUnregister(const_cast<double2*>(host));
    host = nullptr;
    registered = false;
    oz = nullptr;
    oz_e = nullptr;
    data = nullptr;
    gsum = nullptr;
    bhi = blo = nullptr;
    loaded = false;
  }
};

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t cap = 0;  // elements
  cudaError_t ensure(size_t n) {
    if (n <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(&p, n * sizeof(T));
    if (e == cudaSuccess) cap = n;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};


}  // namespace

struct mps_ctx {
  std::recursive_mutex mu;  // calls on one context are serialised (SURVEY.md §8b threading contract)
  int device = 0;
  int layout = 0;
  int M = 0, D = 0;
  std::vector<Site> sites;
  cudaStream_t stream = nullptr;
  uint64_t seed = 0;
  double alpha_sigma = -1.0;
  int gemm_cfg = -1;   // -1: autotune per shape, -2: model (choose_gemm_cfg)
  int gemm_mode = 3;   // 3: 3M (default, 25% fewer DMMAs), 4: 4M real-doubled
  uint64_t launches = 0;
  std::string err;
  // lanes: the micro-batch is split into up to MAX_LANES contiguous row blocks, each run
  // as its own chain on its own stream, so one lane's draw kernel and GEMM tail overlap
  // the other lane's GEMM (per-sample results do not depend on the split)
  static constexpr int MAX_LANES = 8;
  int lanes = 2;
  cudaStream_t lane_st[MAX_LANES] = {};
  cudaEvent_t fork_ev = nullptr, join_ev[MAX_LANES] = {};
  DevBuf<double2> lv0[MAX_LANES], lv1[MAX_LANES], lcbuf[MAX_LANES];
  DevBuf<double> lvs0[MAX_LANES], lvs1[MAX_LANES];  // state sum planes (3M operand sums)
  bool sum_planes = true;                           // feed the 3M GEMM precomputed sums
  int dtype = -1;                                   // MPS_C128 / MPS_C64, fixed by the first site
  int oz_S = 7;                                     // Ozaki digits per operand (gemm mode 8)
  // gemm mode 8 site digits: 0 resident (built once per site), 1 streamed (sliced per call into a
  // 2-slot ring of column blocks on the copy stream, for sites whose planes do not fit), 2 auto
  int oz_site_mode = 2;
  int oz_block_cols = 0;                            // streamed column block (complex cols; 0 = by budget)
  DevBuf<int8_t> ozs_planes[2];
  DevBuf<int> ozs_e[2];
  bool draw_ring = true;                            // stage C rows through a TMA ring in the draw kernel
  bool forced = false;                              // teacher forcing: outcomes read from counts
  // small chains (chi <= 128, chi D <= 1024, 3M): the whole mode loop in one persistent cluster
  // kernel (chain_small.cuh); its per-site tensor maps + bond dims live in chain_meta
  int small_chain = 2;  // 0 off, 1 always when eligible, 2 auto (when the cost model prefers it), 3 = 1 without the tiny kernel
  bool chain_dirty = true;
  DevBuf<uint8_t> chain_meta;
  // host->HBM site streaming: 2-slot ring filled on a copy stream ahead of the GEMMs
  cudaStream_t copy_st = nullptr;
  cudaEvent_t slot_ready[2] = {}, slot_free[2][MAX_LANES] = {};
  DevBuf<double2> sbuf[2];
  DevBuf<double> ssum[2];
  DevBuf<int8_t> loz[MAX_LANES];                    // state digit planes per lane
  DevBuf<int> loz_e[MAX_LANES];
  DevBuf<float> la_hi[2][MAX_LANES], la_lo[2][MAX_LANES];  // c64 state planes (ping-pong)
  DevBuf<float2> lc32[MAX_LANES];                   // c64 C buffer
  DevBuf<float> ones_hi, ones_lo, in_hi, in_lo;
  DevBuf<double> ones_sum, in_sum;
  // multi-micro-batch calls (mps_set_micro_batch): a call of n > micro samples with host arrays runs
  // as micro-batches of `micro` rows whose H2D (cs_in) and D2H (cs_out) overlap the neighbouring
  // micro-batches' compute; device slots are double-buffered, one host synchronisation per call
  int micro = 0;
  cudaStream_t cs_in = nullptr, cs_out = nullptr;
  cudaEvent_t pe_in[2] = {}, pe_comp[2] = {}, pe_d2h[2] = {}, pe_out = nullptr;
  DevBuf<uint8_t> pipe_d;
  // workspaces
  DevBuf<double2> ones;
  // host arrays of a call, packed: [u | alpha | disp | counts | marginals | status] (256-B aligned
  // fields) in a pinned host buffer and its device twin, moved by one H2D and one D2H copy
  DevBuf<uint8_t> io_d;
  uint8_t* io_h = nullptr;
  size_t io_h_cap = 0;
  // live kernel timing (mps_profile): event pairs bracketing each launch on its stream
  int profile = 0;  // bit 0: time K1 launches, bit 1: time K2+K3 launches
  struct Rec {
    int kind;  // 0 site_gemm, 1 displace_draw
    cudaEvent_t a, b;
    double work;  // algorithmic flops (gemm) or bytes (draw)
  };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> event_pool;
  cudaEvent_t get_event() {
    if (!event_pool.empty()) {
      cudaEvent_t e = event_pool.back();
      event_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};

static int fail(mps_ctx* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return code;
}

static int cuda_fail(mps_ctx* c, cudaError_t e, const char* what) {
  cudaGetLastError();
  int code = (e == cudaErrorMemoryAllocation) ? MPS_ERR_RESOURCE : MPS_ERR_GENERIC;
  return fail(c, code, "%s: %s", what, cudaGetErrorString(e));
}

#define CU(c, x, what)                          \
  do {                                          \
    cudaError_t e_ = (x);                       \
    if (e_ != cudaSuccess) return cuda_fail(c, e_, what); \
  } while (0)

// Programmatic dependent launch: each chain kernel may start while its predecessor in the
// stream drains (its prologue overlaps the predecessor's tail wave); the kernels call
// griddepcontrol.wait before touching dependent data.  MPS_NO_PDL=1 disables it.
static bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MPS_NO_PDL");
    v = (e && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
}

// set while the autotuner times back-to-back launches: each must wait for its predecessor, as a
// GEMM does in the chain, so latency-bound shapes are ranked by latency, not by PDL overlap
static thread_local bool t_no_pdl = false;

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl_enabled() && !t_no_pdl) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// draw kernel instantiation for (D, dtype, ring)
static void (*draw_kernel_for(int D, bool c64, bool ring))(DrawArgs) {
  if (c64) {
    if (ring) return D == 10 ? displace_draw_kernel<10, true, true> : D == 4 ? displace_draw_kernel<4, true, true>
                                                                             : displace_draw_kernel<0, true, true>;
    return D == 10 ? displace_draw_kernel<10, true, false> : D == 4 ? displace_draw_kernel<4, true, false>
                                                                    : displace_draw_kernel<0, true, false>;
  }
  if (ring) return D == 10 ? displace_draw_kernel<10, false, true> : D == 4 ? displace_draw_kernel<4, false, true>
                                                                            : displace_draw_kernel<0, false, true>;
  return D == 10 ? displace_draw_kernel<10, false, false> : D == 4 ? displace_draw_kernel<4, false, false>
                                                                   : displace_draw_kernel<0, false, false>;
}

// Kernel attributes bind to the current device's copy of a kernel: set each (kernel, device, attr)
// once, so a process driving several GPUs configures every one of them.
static cudaError_t set_attr_once(const void* kern, cudaFuncAttribute attr, int value) {
  static std::set<std::tuple<const void*, int, int>> done;
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (done.count(std::make_tuple(kern, dev, (int)attr))) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kern, attr, value);
  if (e == cudaSuccess) done.insert(std::make_tuple(kern, dev, (int)attr));
  return e;
}
static cudaError_t set_smem_once(const void* kern, int bytes) {
  return set_attr_once(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

// K1 operands of one launch.  Vs / tgs (the sum planes) may be null: the 3M kernel then
// forms the sums with DADDs; both paths give bit-identical C.
struct GemmOps {
  const void* V;
  const double* Vs;
  int ld_vs;
  const CUtensorMap* tg;
  const CUtensorMap* tgs;
  double2* C;
  int n, K, N;
  long long ldc;
};

// K1 tile configurations, one list per product mode.  Within a mode all configs share
// BK_C = 8 and the same k-step order, so the per-element summation order (and hence
// every bit of C) is config-independent; the autotuner only changes speed.
template <class Cfg, int MODE, bool SUMS>
static cudaError_t launch_cfg_impl(const GemmOps& o, cudaStream_t st) {
  CUtensorMap tv, tvs;
  if (!make_tmap(&tv, o.V, o.n, 2 * (uint64_t)o.K, 16 * (uint64_t)o.K, Cfg::BM)) return cudaErrorInvalidValue;
  dim3 grid((o.n + Cfg::BM - 1) / Cfg::BM, (2 * o.N + Cfg::BN_R - 1) / Cfg::BN_R);
  const int KT = (o.K + Cfg::BK_C - 1) / Cfg::BK_C;
  if constexpr (MODE == 4) {
    if (cudaError_t e = set_smem_once((const void*)site_gemm_kernel<Cfg>, Cfg::SMEM_BYTES)) return e;
    return launch_pdl(site_gemm_kernel<Cfg>, grid, dim3(Cfg::THREADS), Cfg::SMEM_BYTES, st, tv, *o.tg, o.C, o.n, o.N,
                      KT, o.ldc);
  } else {
    using S = Sums3M<Cfg, SUMS>;
    if (cudaError_t e = set_smem_once((const void*)site_gemm3m_kernel<Cfg, SUMS>, S::SMEM_BYTES)) return e;
    if constexpr (SUMS) {
      if (!make_tmap(&tvs, o.Vs, o.n, (uint64_t)o.K, 8 * (uint64_t)o.ld_vs, Cfg::BM, 8)) return cudaErrorInvalidValue;
    } else {
      tvs = tv;  // unused
    }
    return launch_pdl(site_gemm3m_kernel<Cfg, SUMS>, grid, dim3(Cfg::THREADS), S::SMEM_BYTES, st, tv, *o.tg, tvs,
                      SUMS ? *o.tgs : *o.tg, o.C, o.n, o.N, KT, o.ldc);
  }
}

template <class Cfg, int MODE>
static cudaError_t launch_cfg(const GemmOps& o, cudaStream_t st) {
  if constexpr (MODE == 3 && Cfg::BN_R % 32 == 0) {
    if (o.Vs && o.tgs) return launch_cfg_impl<Cfg, 3, true>(o, st);
  }
  return launch_cfg_impl<Cfg, MODE, false>(o, st);
}

typedef cudaError_t (*LaunchFn)(const GemmOps&, cudaStream_t);
struct GemmCfgInfo {
  int bm, bn_r, occ;
  LaunchFn fn;
  const char* name;
};
template <class Cfg, int MODE>
constexpr GemmCfgInfo cfg_info(const char* name) {
  return {Cfg::BM, Cfg::BN_R, Cfg::MIN_BLOCKS, &launch_cfg<Cfg, MODE>, name};
}
//                    BM  BN_R  WARPS_M WARPS_N STAGES MIN_BLOCKS
using G128x128 = GemmCfgT<128, 128, 4, 2, 6, 1>;
using G64x128 = GemmCfgT<64, 128, 2, 4, 6, 1>;
using G64x128p = GemmCfgT<64, 128, 2, 2, 4, 2>;
using G32x64 = GemmCfgT<32, 64, 1, 2, 4, 4>;
using G16x32 = GemmCfgT<16, 32, 1, 1, 4, 8>;
using G128x64 = GemmCfgT<128, 64, 4, 2, 6, 1>;
using G64x64 = GemmCfgT<64, 64, 2, 2, 4, 3>;
using G32x128 = GemmCfgT<32, 128, 1, 4, 4, 2>;
using G64x80 = GemmCfgT<64, 80, 4, 1, 4, 3>;    // 40 complex columns: whole D=10 groups, 4000 tiles at C3
using G64x64w8 = GemmCfgT<64, 64, 4, 2, 4, 2>;  // 3M: 8 warps of 16 x 16 complex, 16 warps/SM
// 32 x 64 tiles of 2 x 2 warps (16 x 16 complex each) at 4 CTAs/SM: the config that exposed the ring's
// cross-proxy WAR race (a TMA refill landing before a slow warp's last ld.shared of the slot, ~1% of
// chains with two lanes and sum planes; fixed by fence.proxy.async before every refill)
using G32x64w4 = GemmCfgT<32, 64, 2, 2, 4, 4>;
// deep rings for short K (chi_l ~ 100: 13 k-stages): most of K in flight at once, so a small-chi
// GEMM costs ~one TMA round trip instead of one per ring refill (latency, not throughput, bound)
using G16x32d8 = GemmCfgT<16, 32, 1, 1, 8, 4>;
using G16x32d16 = GemmCfgT<16, 32, 1, 1, 16, 2>;
using G32x64d8 = GemmCfgT<32, 64, 2, 2, 8, 2>;
static const GemmCfgInfo kGemm4[] = {
    cfg_info<G128x128, 4>("4m_128x128_w4x2"), cfg_info<G64x128, 4>("4m_64x128_w2x4"),
    cfg_info<G64x128p, 4>("4m_64x128_w2x2_occ2"), cfg_info<G32x64, 4>("4m_32x64_w1x2_occ4"),
    cfg_info<G16x32, 4>("4m_16x32_w1x1_occ8"), cfg_info<G64x80, 4>("4m_64x80_w4x1_occ3")};
static const GemmCfgInfo kGemm3[] = {
    cfg_info<G128x64, 3>("3m_128x64_w4x2"), cfg_info<G64x128, 3>("3m_64x128_w2x4"),
    cfg_info<G64x64, 3>("3m_64x64_w2x2_occ3"), cfg_info<G32x64, 3>("3m_32x64_w1x2_occ4"),
    cfg_info<G16x32, 3>("3m_16x32_w1x1_occ8"), cfg_info<G32x128, 3>("3m_32x128_w1x4_occ2"),
    cfg_info<G64x80, 3>("3m_64x80_w4x1_occ3"), cfg_info<G64x64w8, 3>("3m_64x64_w4x2_occ2"),
    cfg_info<G16x32d8, 3>("3m_16x32_w1x1_s8_occ4"),
    cfg_info<G16x32d16, 3>("3m_16x32_w1x1_s16_occ2"), cfg_info<G32x64d8, 3>("3m_32x64_w2x2_s8_occ2"),
    cfg_info<G32x64w4, 3>("3m_32x64_w2x2_occ4")};
constexpr int N_GEMM4 = sizeof(kGemm4) / sizeof(kGemm4[0]);
constexpr int N_GEMM3 = sizeof(kGemm3) / sizeof(kGemm3[0]);
constexpr int N_GEMM_CFGS = N_GEMM3 > N_GEMM4 ? N_GEMM3 : N_GEMM4;  // index bound for the API
static int n_cfgs(int mode) { return mode == 3 ? N_GEMM3 : N_GEMM4; }
static const GemmCfgInfo& cfg_of(int mode, int cfg) { return mode == 3 ? kGemm3[cfg] : kGemm4[cfg]; }
static int g_num_sms = 148;

// Analytic fallback: waves x per-tile DMMA cycles (an SM's FP64 pipe shared by its
// resident CTAs) + a per-wave latency term.
static int choose_gemm_cfg(int mode, int n, int K, int N) {
  double best = 1e300;
  int arg = 0;
  for (int c = 0; c < n_cfgs(mode); ++c) {
    const GemmCfgInfo& ci = cfg_of(mode, c);
    const double tiles = (double)((n + ci.bm - 1) / ci.bm) * ((2 * N + ci.bn_r - 1) / ci.bn_r);
    const double waves = std::ceil(tiles / ((double)g_num_sms * ci.occ));
    const double tile_cycles = (double)ci.bm * ci.bn_r * 16.0 * ((K + 7) / 8) / 64.0 * ci.occ;
    const double t = waves * (tile_cycles + 3000.0);
    if (t < best * 0.999) {
      best = t;
      arg = c;
    }
  }
  return arg;
}

// Autotune cache: (n, K, N) -> config.  Every config produces bit-identical C, so the
// choice never changes results; it is made once per shape (first call, outside any
// timed region in bench.py) by timing each candidate twice on the real operands.
static std::map<std::tuple<int, int, int, int>, int> g_tuned;
static std::mutex g_tuned_mu;

static int tune_gemm(int mode, const GemmOps& o, cudaStream_t st) {
  const bool sums = o.Vs && o.tgs;
  {
    std::lock_guard<std::mutex> lk(g_tuned_mu);
    auto it = g_tuned.find({mode * 2 + (sums ? 1 : 0), o.n, o.K, o.N});
    if (it != g_tuned.end()) return it->second;
  }
  int best = 0;
  {
    // one timed run per candidate when a GEMM is long (> ~20 ms), the best of two when it is
    // ms-scale, the best of eight when it is us-scale (latency-bound shapes time noisily)
    const double est_ms = 8.0 * o.n * (double)o.K * o.N / 37e9;
    const int reps = est_ms > 20.0 ? 1 : est_ms > 0.5 ? 2 : 4;
    const int inner = est_ms > 0.5 ? 1 : 16;  // us-scale: time 16 back-to-back launches per event pair
    float best_ms = 1e30f;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int cfg = 0; cfg < n_cfgs(mode); ++cfg) {
      float ms_min = 1e30f;
      for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0, st);
        bool ok = true;
        t_no_pdl = true;
        for (int i = 0; i < inner && ok; ++i) ok = cfg_of(mode, cfg).fn(o, st) == cudaSuccess;
        t_no_pdl = false;
        if (!ok) break;
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        ms_min = std::min(ms_min, ms / inner);
      }
      if (ms_min < best_ms * 0.995f) {
        best_ms = ms_min;
        best = cfg;
      }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaGetLastError();
  }
  std::lock_guard<std::mutex> lk(g_tuned_mu);
  g_tuned[{mode * 2 + (sums ? 1 : 0), o.n, o.K, o.N}] = best;
  return best;
}

// cfg: 0..n-1 explicit, -1 autotune (cached per shape), -2 analytic model only.
static int launch_site_gemm(mps_ctx* ctx, const GemmOps& o, cudaStream_t st, int cfg, int mode) {
  if (mode == 4 || !o.Vs || !o.tgs) {
    GemmOps p = o;  // sum planes only feed the 3M kernel
    p.Vs = nullptr;
    p.tgs = nullptr;
    if (cfg == -1) cfg = tune_gemm(mode, p, st);
    if (cfg < 0 || cfg >= n_cfgs(mode)) cfg = choose_gemm_cfg(mode, o.n, o.K, o.N);
    cudaError_t e = cfg_of(mode, cfg).fn(p, st);
    if (ctx) ctx->launches++;
    if (e != cudaSuccess) return cuda_fail(ctx, e, "site_gemm launch");
    return MPS_OK;
  }
  if (cfg == -1) cfg = tune_gemm(mode, o, st);
  if (cfg < 0 || cfg >= n_cfgs(mode)) cfg = choose_gemm_cfg(mode, o.n, o.K, o.N);
  cudaError_t e = cfg_of(mode, cfg).fn(o, st);
  if (ctx) ctx->launches++;
  if (e != cudaSuccess) return cuda_fail(ctx, e, "site_gemm launch");
  return MPS_OK;
}

// ---- complex128 K1 emulated on the INT8 tensor cores (Ozaki scheme, gemm mode 8) -----------------
template <int S, int CM, int CN>
static cudaError_t launch_ozaki_cl(const int8_t* a_planes, int n_pad, const int* ea, const int8_t* b_planes, int b_pad,
                                   const int* eb, int ld, double2* C, int n, int K, int N, cudaStream_t st) {
  using Cfg = OzCfg<S, CM, CN>;
  if (cudaError_t e = set_smem_once((const void*)ozaki_gemm_kernel<Cfg>, Cfg::SMEM_BYTES)) return e;
  // grid padded to whole clusters: padding CTAs read padding rows (n_pad, b_pad are multiples of 256) and
  // store nothing
  dim3 grid(round_up((n + Cfg::BM - 1) / Cfg::BM, CM), round_up((2 * N + Cfg::BN - 1) / Cfg::BN, CN));
  const int KB = ld / Cfg::BK;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(Cfg::THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (CM * CN > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = CM;
    attr[na].val.clusterDim.y = CN;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, ozaki_gemm_kernel<Cfg>, a_planes, b_planes, ea, eb, (double*)C, n, 2 * N, KB,
                            2LL * N);
}

// diagonal-split kernel: clusters of MP CTA pairs, 128 x 128 tiles (ozaki_gemm.cuh)
template <int S, int MP>
static cudaError_t launch_ozaki2(const int8_t* a_planes, int n_pad, const int* ea, const int8_t* b_planes, int b_pad,
                                 const int* eb, int ld, double2* C, int n, int K, int N, cudaStream_t st,
                                 long long ldc_c = 0) {
  if (ldc_c == 0) ldc_c = N;  // complex elements per C row (a column block writes into a wider C)
  using Cfg = Oz2Cfg<S, MP>;
  if (cudaError_t e = set_smem_once((const void*)ozaki2_gemm_kernel<Cfg>, Cfg::SMEM_BYTES)) return e;
  const int mtiles = round_up((n + Cfg::BM - 1) / Cfg::BM, MP);
  dim3 grid(2 * mtiles, (2 * N + Cfg::BN - 1) / Cfg::BN);
  const int KS = ld / Cfg::BK;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(Cfg::THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = Cfg::CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  // K segments of <= OZ_SEG_KB steps keep every int32 diagonal sum exact; later ones add into C
  for (int kb0 = 0; kb0 < KS; kb0 += OZ_SEG_KB) {
    const int KB = std::min(OZ_SEG_KB, KS - kb0);
    cudaError_t e = cudaLaunchKernelEx(&cfg, ozaki2_gemm_kernel<Cfg>, a_planes, b_planes, ea, eb, (double*)C, n, 2 * N,
                                       KB, 2LL * ldc_c, KS, kb0, kb0 > 0 ? 1 : 0);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

static bool ozaki_v1() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MPS_OZ_KERNEL");
    v = (e && strcmp(e, "v1") == 0) ? 1 : 0;
  }
  return v == 1;
}

// K1 emulated on INT8: the diagonal-split pair kernel (default) or, with MPS_OZ_KERNEL=v1, the
// single-CTA 128 x 64 kernel that keeps all S diagonals (2/3 of the MMA rate, kept for comparison)
template <int S>
static cudaError_t launch_ozaki_s(const int8_t* a_planes, int n_pad, const int* ea, const int8_t* b_planes, int b_pad,
                                  const int* eb, int ld, double2* C, int n, int K, int N, cudaStream_t st,
                                  long long ldc_c) {
  if (ozaki_v1() && K <= OZ_MAX_K && (ldc_c == 0 || ldc_c == N))
    return launch_ozaki_cl<S, 1, 1>(a_planes, n_pad, ea, b_planes, b_pad, eb, ld, C, n, K, N, st);
  return launch_ozaki2<S, 1>(a_planes, n_pad, ea, b_planes, b_pad, eb, ld, C, n, K, N, st, ldc_c);
}

// ldc_c: complex elements per C row (0: N); a site column block passes C + c0 and the full width
static cudaError_t launch_ozaki(int S, const int8_t* a_planes, int n_pad, const int* ea, const int8_t* b_planes,
                                int b_pad, const int* eb, int ld, double2* C, int n, int K, int N, cudaStream_t st,
                                long long ldc_c = 0) {
  switch (S) {
    case 5: return launch_ozaki_s<5>(a_planes, n_pad, ea, b_planes, b_pad, eb, ld, C, n, K, N, st, ldc_c);
    case 6: return launch_ozaki_s<6>(a_planes, n_pad, ea, b_planes, b_pad, eb, ld, C, n, K, N, st, ldc_c);
    default: return launch_ozaki_s<7>(a_planes, n_pad, ea, b_planes, b_pad, eb, ld, C, n, K, N, st, ldc_c);
  }
}

// digit planes of a state (n x K complex128): S planes of n_pad x ld bytes + n exponents
static cudaError_t ozaki_slice_state(const double2* V, int n, int K, int S, int8_t* planes, int n_pad, int ld, int* e,
                                     cudaStream_t st) {
  ozaki_slice_rows_kernel<<<n, 128, 0, st>>>(V, K, S, planes, ld, e);
  return cudaGetLastError();
}

// site digit planes (B_r^T: 2N rows), built once per (site, S)
static cudaError_t ozaki_prepare_site(Site& s, int D, int S) {
  if (s.oz && s.oz_S == S) return cudaSuccess;
  if (s.oz) cudaFree(s.oz);
  if (s.oz_e) cudaFree(s.oz_e);
  s.oz = nullptr;
  s.oz_e = nullptr;
  const int N = s.chi_r * D;
  s.oz_ld = oz_ld(s.chi_l);
  s.oz_pad = round_up(2 * N, 256);
  cudaError_t e = cudaMalloc(&s.oz, (size_t)S * s.oz_pad * s.oz_ld);
  if (e == cudaSuccess) e = cudaMalloc(&s.oz_e, (size_t)2 * N * sizeof(int));
  if (e != cudaSuccess) return e;
  ozaki_slice_site_kernel<<<2 * N, 128>>>(s.data, s.chi_l, N, S, s.oz, s.oz_ld, s.oz_e);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  s.oz_S = S;
  return e;
}

// ---- complex64 K1 (tcgen05, 3xTF32) --------------------------------------------------------
using C64Big = C64Cfg<256, 2>;

// C (n x N complex64) = A planes (n x ld fp32, hi/lo of the interleaved state) . B_r planes
// multicast pairs are used when there are >= 2 M tiles (MPS_C64_NO_MULTICAST=1 disables them)
static bool c64_multicast_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MPS_C64_NO_MULTICAST");
    v = (e && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
}

// persistent variants (MPS_C64_KERNEL = p128 (default) | p256 | mc256 = one tile per CTA, 2-CTA multicast)
using C64P256 = C64Cfg<256, 2>;
using C64P128 = C64Cfg<128, 3>;
template <class Cfg>
static cudaError_t launch_c64_persistent(const float* ahi, const float* alo, const float* bhi, const float* blo, int ld,
                                         float* C, int n, int K, int N, long long ldc_f, cudaStream_t st) {
  if (cudaError_t e = set_smem_once((const void*)c64_gemm_persistent_kernel<Cfg>, Cfg::SMEM_BYTES)) return e;
  CUtensorMap tah, tal, tbh, tbl;
  const uint64_t cols = 2 * (uint64_t)K, pitch = 4 * (uint64_t)ld;
  if (!make_tmap(&tah, ahi, n, cols, pitch, Cfg::BM, 32, true) || !make_tmap(&tal, alo, n, cols, pitch, Cfg::BM, 32, true) ||
      !make_tmap(&tbh, bhi, 2 * (uint64_t)N, cols, pitch, Cfg::BN, 32, true) ||
      !make_tmap(&tbl, blo, 2 * (uint64_t)N, cols, pitch, Cfg::BN, 32, true))
    return cudaErrorInvalidValue;
  const long long ntiles = (long long)((n + Cfg::BM - 1) / Cfg::BM) * ((2 * N + Cfg::BN - 1) / Cfg::BN);
  const int KB = (int)((cols + Cfg::BK - 1) / Cfg::BK);
  dim3 grid((unsigned)std::min<long long>(ntiles, g_num_sms));
  return launch_pdl(c64_gemm_persistent_kernel<Cfg>, grid, dim3(Cfg::THREADS), Cfg::SMEM_BYTES, st, tah, tal, tbh,
                    tbl, C, n, 2 * N, KB, ldc_f);
}

static int c64_kernel_choice() {
  static int v = -1;
  if (v < 0) {
    // default (auto): persistent 128-column tiles when the grid is a few waves (C3: +10%, finer
    // tiles quantise better and the double-buffered accumulator hides the epilogue), 256-column
    // multicast pairs when it is many (C4: +11% over p128); cg2 = the cta_group::2 pair kernel (the
    // default for two or more waves of 256-wide tiles, below)
    const char* e = getenv("MPS_C64_KERNEL");
    v = !e ? 3
           : (strcmp(e, "p256") == 0 ? 1 : strcmp(e, "mc256") == 0 ? 0 : strcmp(e, "p128") == 0 ? 2
              : strcmp(e, "cg2") == 0 ? 4 : strcmp(e, "cg2p") == 0 ? 5 : 3);
  }
  return v;
}

// cta_group::2 pairs: 256 x 256 tiles (each CTA 128 rows x 256 columns of TMEM), 3-stage ring
using C64Cg2 = C64Cg2Cfg<256, 3>;
static cudaError_t launch_c64_cg2(const float* ahi, const float* alo, const float* bhi, const float* blo, int ld,
                                  float* C, int n, int K, int N, long long ldc_f, cudaStream_t st, bool persistent) {
  using Cfg = C64Cg2;
  void (*kern)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, float*, int, int, int, long long) =
      persistent ? c64_gemm_cg2p_kernel<Cfg> : c64_gemm_cg2_kernel<Cfg>;
  if (cudaError_t e = set_smem_once((const void*)kern, Cfg::SMEM_BYTES)) return e;
  CUtensorMap tah, tal, tbh, tbl;
  const uint64_t cols = 2 * (uint64_t)K, pitch = 4 * (uint64_t)ld;
  if (!make_tmap(&tah, ahi, n, cols, pitch, Cfg::BM, 32, true) || !make_tmap(&tal, alo, n, cols, pitch, Cfg::BM, 32, true) ||
      !make_tmap(&tbh, bhi, 2 * (uint64_t)N, cols, pitch, Cfg::BN / 2, 32, true) ||
      !make_tmap(&tbl, blo, 2 * (uint64_t)N, cols, pitch, Cfg::BN / 2, 32, true))
    return cudaErrorInvalidValue;
  const int KB = (int)((cols + Cfg::BK - 1) / Cfg::BK);
  const int mtiles = (n + Cfg::BM - 1) / Cfg::BM;
  const int ntile = (2 * N + Cfg::BN - 1) / Cfg::BN;
  dim3 grid((mtiles + 1) & ~1, ntile);  // pairs along M (a padding CTA stores nothing)
  if (persistent) {  // one pair per two SMs, walking the pair tiles
    const long long ptiles = (long long)((mtiles + 1) / 2) * ntile;
    grid = dim3((unsigned)(2 * std::min<long long>(ptiles, g_num_sms / 2)), 1);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(Cfg::THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, tah, tal, tbh, tbl, C, n, 2 * N, KB, ldc_f);
}

static cudaError_t launch_c64_gemm(const float* ahi, const float* alo, const float* bhi, const float* blo, int ld,
                                   float* C, int n, int K, int N, long long ldc_f, cudaStream_t st) {
  int choice = c64_kernel_choice();
  if (choice == 3) {  // auto: two to 16 waves of 256-wide tiles -> persistent cta_group::2 pairs (C3 site:
                      // 0.503 ms vs 0.525 one tile per pair, 0.548 p128); more -> one tile per pair (C4 site:
                      // 12.4 ms vs 12.6 persistent, 13.0 multicast); fewer -> persistent 128-wide tiles.
                      // All variants give the same bits.
    const long long tiles256 = (long long)((n + 127) / 128) * ((2 * N + 255) / 256);
    choice = tiles256 >= 16LL * g_num_sms ? 4 : tiles256 >= 2LL * g_num_sms ? 5 : 2;
  }
  if (choice == 4 || choice == 5) return launch_c64_cg2(ahi, alo, bhi, blo, ld, C, n, K, N, ldc_f, st, choice == 5);
  if (choice == 1) return launch_c64_persistent<C64P256>(ahi, alo, bhi, blo, ld, C, n, K, N, ldc_f, st);
  if (choice == 2) return launch_c64_persistent<C64P128>(ahi, alo, bhi, blo, ld, C, n, K, N, ldc_f, st);
  using Cfg = C64Big;
  if (cudaError_t e = set_smem_once((const void*)c64_gemm_kernel<Cfg, false>, Cfg::SMEM_BYTES)) return e;
  if (cudaError_t e = set_smem_once((const void*)c64_gemm_kernel<Cfg, true>, Cfg::SMEM_BYTES)) return e;
  const int mtiles = (n + Cfg::BM - 1) / Cfg::BM;
  const bool mc = c64_multicast_enabled() && mtiles >= 2;
  CUtensorMap tah, tal, tbh, tbl;
  const uint64_t cols = 2 * (uint64_t)K, pitch = 4 * (uint64_t)ld;
  const uint32_t brows = mc ? Cfg::BN / 2 : Cfg::BN;
  if (!make_tmap(&tah, ahi, n, cols, pitch, Cfg::BM, 32, true) || !make_tmap(&tal, alo, n, cols, pitch, Cfg::BM, 32, true) ||
      !make_tmap(&tbh, bhi, 2 * (uint64_t)N, cols, pitch, brows, 32, true) ||
      !make_tmap(&tbl, blo, 2 * (uint64_t)N, cols, pitch, brows, 32, true))
    return cudaErrorInvalidValue;
  const int KB = (int)((cols + Cfg::BK - 1) / Cfg::BK);
  if (!mc) {
    dim3 grid(mtiles, (2 * N + Cfg::BN - 1) / Cfg::BN);
    return launch_pdl(c64_gemm_kernel<Cfg, false>, grid, dim3(Cfg::THREADS), Cfg::SMEM_BYTES, st, tah, tal, tbh, tbl,
                      C, n, 2 * N, KB, ldc_f);
  }
  dim3 grid((mtiles + 1) & ~1, (2 * N + Cfg::BN - 1) / Cfg::BN);  // pairs along M (a padding CTA stores nothing)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(Cfg::THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, c64_gemm_kernel<Cfg, true>, tah, tal, tbh, tbl, C, n, 2 * N, KB, ldc_f);
}

// ---- small chains: the whole mode loop in one persistent cluster launch (chain_small.cuh) ----
// small-chain variant: 2 = halves of each group pipelined (chain_small2.cuh), 1 = lock step
static int small_chain_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MPS_SMALL_CHAIN_V2");
    v = (e && e[0] == '0') ? 1 : 2;  // default: the pipelined variant (C2 +13%, C1 +8%, same bits)
  }
  return v;
}
static void (*small_chain_kernel_for(int D))(ChainArgs) {
  if (small_chain_variant() == 2)
    return D == 10 ? small_chain2_kernel<10> : D == 4 ? small_chain2_kernel<4> : small_chain2_kernel<0>;
  return D == 10 ? small_chain_kernel<10> : D == 4 ? small_chain_kernel<4> : small_chain_kernel<0>;
}
static int sc_threads() { return small_chain_variant() == 2 ? SC2_THREADS : SC_THREADS; }
static int sc_smem() { return small_chain_variant() == 2 ? SC2_SMEM : SC_SMEM; }

// co-resident 16-CTA clusters of the instantiation for D on the current device (0: none fit)
static int small_chain_capacity(int D) {
  void (*kern)(ChainArgs) = small_chain_kernel_for(D);
  static std::map<std::pair<void*, int>, int> cap;
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cap.find({(void*)kern, dev});
    if (it != cap.end()) return it->second;
  }
  int num = 0;
  if (set_smem_once((const void*)kern, sc_smem()) == cudaSuccess &&
      set_attr_once((const void*)kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
    cudaLaunchConfig_t q = {};
    q.gridDim = dim3(SC_CL * 32);
    q.blockDim = dim3(sc_threads());
    q.dynamicSmemBytes = sc_smem();
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = SC_CL;
    a[0].val.clusterDim.y = 1;
    a[0].val.clusterDim.z = 1;
    q.attrs = a;
    q.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&num, kern, &q) != cudaSuccess) num = 0;
  }
  cudaGetLastError();
  std::lock_guard<std::mutex> lk(mu);
  cap[{(void*)kern, dev}] = num;
  return num;
}

// ---- tiny chains: one CTA per 8-row group, every site in shared memory (chain_tiny.cuh) ----
static void (*tiny_chain_kernel_for(int D))(ChainArgs) {
  return D == 4 ? tiny_chain_kernel<4> : D == 10 ? tiny_chain_kernel<10> : tiny_chain_kernel<0>;
}
static int tiny_smem(const mps_ctx* c, int m_begin, int m_end) {
  long long b = TC_OFF_SITES;
  for (int m = m_begin; m < m_end; ++m) b += tc_site_bytes(c->sites[m].chi_l, c->sites[m].chi_r, c->D);
  return b + 1024 <= TC_SMEM_MAX ? (int)(b + 1024) : -1;  // + the 1 KB alignment slack
}
// Whether the call takes the tiny-chain kernel: small-chain modes 1 / 2 (not 0, not 3), complex128 3M,
// chi_l <= 32, chi_r <= 32, chi_r D <= 256 at every site, and the range's sites fit in shared memory.
// It replaces both the cluster kernel and the per-mode kernels for such chains at any n (its CTAs
// persist over 8-row groups), with the same bits.
static bool tiny_chain_ok(const mps_ctx* c, int m_begin, int m_end, int n) {
  if ((c->small_chain != 1 && c->small_chain != 2) || c->dtype != MPS_C128 || c->gemm_mode != 3 || n < 1)
    return false;
  if (m_end - m_begin > TC_MMAX || c->D > DMAX) return false;
  for (int m = m_begin; m < m_end; ++m) {
    const Site& s = c->sites[m];
    if (s.host || !s.chain || s.chi_l > TC_KMAX || s.chi_r > TC_RMAX || s.chi_r * c->D > TC_NMAX) return false;
  }
  return tiny_smem(c, m_begin, m_end) > 0;
}
static cudaError_t launch_tiny_chain(mps_ctx* c, const ChainArgs& P, cudaStream_t st) {
  void (*kern)(ChainArgs) = tiny_chain_kernel_for(c->D);
  const int smem = tiny_smem(c, P.m_begin, P.m_end);
  if (smem < 0) return cudaErrorNotSupported;
  cudaError_t e = set_smem_once((const void*)kern, TC_SMEM_MAX);
  if (e != cudaSuccess) return e;
  static std::map<std::tuple<void*, int, int>, int> occ;  // (kernel, device, smem) -> CTAs per SM
  static std::mutex mu;
  int dev = 0, per_sm = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = occ.find({(void*)kern, dev, smem});
    if (it != occ.end()) per_sm = it->second;
  }
  if (per_sm == 0) {
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TC_THREADS, smem);
    if (e != cudaSuccess || per_sm < 1) return e != cudaSuccess ? e : cudaErrorNotSupported;
    std::lock_guard<std::mutex> lk(mu);
    occ[{(void*)kern, dev, smem}] = per_sm;
  }
  const int groups = (P.n + TC_ROWS - 1) / TC_ROWS;
  return launch_pdl(kern, dim3(std::min(groups, per_sm * g_num_sms)), dim3(TC_THREADS), (size_t)smem, st, P);
}

// Whether a call of n samples over [m_begin, m_end) takes the small-chain kernel.  Auto mode
// compares two latency models fitted to the C1/C2 sweeps (profiles/r01_small_chain_crossover.txt):
// the fused kernel costs ~3.5 us + its 16-row K1 slice (~2.4 TFLOP/s per cluster) per mode and per
// wave of co-resident clusters; the per-mode kernels ~13 us per mode or their K1 work at ~20 TFLOP/s.
// Both paths give the same bits, so the choice only moves time.
static bool small_chain_ok(const mps_ctx* c, int m_begin, int m_end, int n) {
  if (!c->small_chain || c->dtype != MPS_C128 || c->gemm_mode != 3 || n < 1) return false;
  if (tiny_chain_ok(c, m_begin, m_end, n)) return true;
  for (int m = m_begin; m < m_end; ++m) {
    const Site& s = c->sites[m];
    if (s.host || !s.chain || s.chi_l > SC_KMAX || s.chi_r * c->D > SC_NMAX) return false;
  }
  const int cap = small_chain_capacity(c->D);
  if (cap < 1) return false;
  if (c->small_chain == 1 || c->small_chain == 3) return true;
  const int waves = ((n + SC_CL - 1) / SC_CL + cap - 1) / cap;
  double t_chain = 0.0, t_mode = 0.0;
  const bool v2 = small_chain_variant() == 2;
  for (int m = m_begin; m < m_end; ++m) {
    const double fl = 8.0 * c->sites[m].chi_l * (double)c->sites[m].chi_r * c->D;  // per sample row
    if (v2) {  // fitted to the round-2 sweeps (C1: n = 100..600, C2: n = 100..500)
      t_chain += waves * (3.0e-6 + SC_CL * fl / 3.3e12);
      t_mode += 10.5e-6 + n * fl / 30e12;
    } else {
      t_chain += waves * (3.5e-6 + SC_CL * fl / 2.4e12);
      t_mode += std::max(13e-6, n * fl / 20e12);
    }
  }
  return t_chain <= t_mode;
}

// per-site chain-layout pointers and chi_0..chi_M in device memory
static cudaError_t chain_meta_upload(mps_ctx* c) {
  if (!c->chain_dirty) return cudaSuccess;
  const int M = c->M;
  const size_t ptr_bytes = (size_t)M * sizeof(double2*);
  std::vector<uint8_t> h(ptr_bytes + (M + 1) * sizeof(int), 0);
  double2** ptrs = reinterpret_cast<double2**>(h.data());
  int* chi = reinterpret_cast<int*>(h.data() + ptr_bytes);
  for (int m = 0; m < M; ++m) {
    const Site& s = c->sites[m];
    if (!s.loaded) continue;
    ptrs[m] = s.chain;
    chi[m] = s.chi_l;
    chi[m + 1] = s.chi_r;
  }
  cudaError_t e = c->chain_meta.ensure(h.size());
  if (e == cudaSuccess) e = cudaMemcpy(c->chain_meta.p, h.data(), h.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) c->chain_dirty = false;
  return e;
}

static cudaError_t launch_small_chain(mps_ctx* c, const ChainArgs& P, cudaStream_t st) {
  void (*kern)(ChainArgs) = small_chain_kernel_for(c->D);
  const int mc = small_chain_capacity(c->D);
  if (mc < 1) return cudaErrorNotSupported;
  const int groups = (P.n + SC_CL - 1) / SC_CL;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(SC_CL * std::min(groups, mc));
  cfg.blockDim = dim3(sc_threads());
  cfg.dynamicSmemBytes = sc_smem();
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = SC_CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // the kernels call griddepcontrol.wait
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl_enabled() && !t_no_pdl) ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, P);
}

extern "C" {

int mps_create(int n_dev, const int* dev_ids, int layout, mps_ctx** out) {
  if (!out) return MPS_ERR_VALIDATION;
  *out = nullptr;
  if (n_dev != 1) return MPS_ERR_VALIDATION;  // one context per GPU per process
  if (layout != 0 && layout != 1) return MPS_ERR_VALIDATION;
  int dev = dev_ids ? dev_ids[0] : 0;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    return MPS_ERR_RESOURCE;
  }
  if (dev < 0 || dev >= count) return MPS_ERR_VALIDATION;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess || prop.major != 10) return MPS_ERR_RESOURCE;
  if (cudaSetDevice(dev) != cudaSuccess) return MPS_ERR_GENERIC;
  if (!get_encode_fn()) return MPS_ERR_GENERIC;
  g_num_sms = prop.multiProcessorCount;
  mps_ctx* c = new mps_ctx();
  c->device = dev;
  c->layout = layout;
  bool ok = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming) == cudaSuccess;
  for (int l = 0; ok && l < mps_ctx::MAX_LANES; ++l)
    ok = cudaStreamCreateWithFlags(&c->lane_st[l], cudaStreamNonBlocking) == cudaSuccess &&
         cudaEventCreateWithFlags(&c->join_ev[l], cudaEventDisableTiming) == cudaSuccess;
  ok = ok && cudaStreamCreateWithFlags(&c->copy_st, cudaStreamNonBlocking) == cudaSuccess;
  ok = ok && cudaStreamCreateWithFlags(&c->cs_in, cudaStreamNonBlocking) == cudaSuccess &&
       cudaStreamCreateWithFlags(&c->cs_out, cudaStreamNonBlocking) == cudaSuccess &&
       cudaEventCreateWithFlags(&c->pe_out, cudaEventDisableTiming) == cudaSuccess;
  for (int w = 0; ok && w < 2; ++w)
    ok = cudaEventCreateWithFlags(&c->pe_in[w], cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&c->pe_comp[w], cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&c->pe_d2h[w], cudaEventDisableTiming) == cudaSuccess;
  for (int w = 0; ok && w < 2; ++w) {
    ok = cudaEventCreateWithFlags(&c->slot_ready[w], cudaEventDisableTiming) == cudaSuccess;
    for (int l = 0; ok && l < mps_ctx::MAX_LANES; ++l)
      ok = cudaEventCreateWithFlags(&c->slot_free[w][l], cudaEventDisableTiming) == cudaSuccess;
  }
  if (!ok) {
    cudaGetLastError();
    delete c;
    return MPS_ERR_GENERIC;
  }
  {
    const char* e = getenv("MPS_DRAW_RING");
    if (e && e[0] == '0') c->draw_ring = false;
    e = getenv("MPS_SMALL_CHAIN");
    if (e && (e[0] == '0' || e[0] == '1' || e[0] == '3')) c->small_chain = e[0] - '0';
  }
  *out = c;
  return MPS_OK;
}

int mps_configure(mps_ctx* c, int M, int D) {
  if (!c) return MPS_ERR_VALIDATION;
  std::lock_guard<std::recursive_mutex> lk_(c->mu);
  if (M < 1) return fail(c, MPS_ERR_VALIDATION, "M must be >= 1, got %d", M);
  if (D < 1 || D > DMAX) return fail(c, MPS_ERR_VALIDATION, "D must lie in [1, %d], got %d", DMAX, D);
  cudaSetDevice(c->device);
  for (auto& s : c->sites) s.release();
  c->sites.assign(M, Site());
  c->chain_dirty = true;
  c->dtype = -1;
  c->M = M;
  c->D = D;
  return MPS_OK;
}

int mps_set_site(mps_ctx* c, int m, int chi_l, int chi_r, int D, const void* gamma, int flags, int dtype) {
  if (!c) return MPS_ERR_VALIDATION;
  std::lock_guard<std::recursive_mutex> lk_(c->mu);
  if (c->M == 0) return fail(c, MPS_ERR_VALIDATION, "mps_configure must precede mps_set_site");
  if (m < 0 || m >= c->M) return fail(c, MPS_ERR_VALIDATION, "site index %d outside [0, %d)", m, c->M);
  if (D != c->D) return fail(c, MPS_ERR_VALIDATION, "site %d: D=%d but the chain has D=%d", m, D, c->D);
  if (chi_l < 1 || chi_r < 1) return fail(c, MPS_ERR_VALIDATION, "site %d: bond dims must be >= 1", m);
  if (dtype != MPS_C128 && dtype != MPS_C64)
    return fail(c, MPS_ERR_VALIDATION, "site %d: dtype %d is neither complex128 (0) nor complex64 (1)", m, dtype);
  if (c->dtype >= 0 && c->dtype != dtype)
    return fail(c, MPS_ERR_VALIDATION, "site %d: dtype %d differs from the chain's %d", m, dtype, c->dtype);
  if (!gamma) return fail(c, MPS_ERR_VALIDATION, "site %d: null tensor", m);
  if (m > 0 && c->sites[m - 1].loaded && c->sites[m - 1].chi_r != chi_l)
    return fail(c, MPS_ERR_VALIDATION, "site %d: chi_l=%d != chi_r=%d of site %d", m, chi_l, c->sites[m - 1].chi_r,
                m - 1);
  if (m + 1 < c->M && c->sites[m + 1].loaded && c->sites[m + 1].chi_l != chi_r)
    return fail(c, MPS_ERR_VALIDATION, "site %d: chi_r=%d != chi_l=%d of site %d", m, chi_r, c->sites[m + 1].chi_l,
                m + 1);
  cudaSetDevice(c->device);
  Site& s = c->sites[m];
  s.release();
  s = Site();
  c->chain_dirty = true;
  const size_t elems = (size_t)chi_l * chi_r * D;
  const bool dev = is_device_ptr(gamma);
  if (dtype == MPS_C64 && flags == MPS_SITE_HOST_STREAM)
    return fail(c, MPS_ERR_VALIDATION, "site %d: host streaming is implemented for complex128 sites", m);
  if (dtype == MPS_C64) {
    // keep only the tcgen05 operand planes of B_r^T (2N x ld fp32, hi / lo)
    const int N = chi_r * D, ld = plane_ld(2 * chi_l);
    const float2* src = (const float2*)gamma;
    float2* tmp = nullptr;
    if (!dev) {
      CU(c, cudaMalloc(&tmp, elems * sizeof(float2)), "cudaMalloc(site staging)");
      CU(c, cudaMemcpy(tmp, gamma, elems * sizeof(float2), cudaMemcpyHostToDevice), "copy site");
      src = tmp;
    }
    cudaError_t e1 = cudaMalloc(&s.bhi, (size_t)2 * N * ld * sizeof(float));
    cudaError_t e2 = e1 == cudaSuccess ? cudaMalloc(&s.blo, (size_t)2 * N * ld * sizeof(float)) : e1;
    if (e2 != cudaSuccess) {
      if (tmp) cudaFree(tmp);
      s.release();
      return cuda_fail(c, e2, "cudaMalloc(c64 site planes)");
    }
    const long long t = (long long)2 * N * ld;
    c64_site_planes_kernel<<<(unsigned)((t + 255) / 256), 256>>>(src, chi_l, N, s.bhi, s.blo, ld);
    cudaError_t e3 = cudaGetLastError();
    if (e3 == cudaSuccess) e3 = cudaDeviceSynchronize();
    if (tmp) cudaFree(tmp);
    if (e3 != cudaSuccess) {
      s.release();
      return cuda_fail(c, e3, "c64 site planes");
    }
    s.ld = ld;
    s.chi_l = chi_l;
    s.chi_r = chi_r;
    s.loaded = true;
    c->dtype = MPS_C64;
    return MPS_OK;
  }
  if (flags == MPS_SITE_HOST_STREAM) {
    if (dev) return fail(c, MPS_ERR_VALIDATION, "site %d: HOST_STREAM needs a host pointer", m);
    cudaPointerAttributes at;
    const bool pinned = cudaPointerGetAttributes(&at, gamma) == cudaSuccess && at.type == cudaMemoryTypeHost;
    cudaGetLastError();
    if (!pinned) {
      CU(c, cudaHostRegister(const_cast<void*>(gamma), elems * sizeof(double2), cudaHostRegisterReadOnly),
         "cudaHostRegister(site)");
      s.registered = true;
    }
    s.host = (const double2*)gamma;
    s.chi_l = chi_l;
    s.chi_r = chi_r;
    s.loaded = true;
    c->dtype = MPS_C128;
    return MPS_OK;
  }
  if (flags == MPS_SITE_DEVICE_BORROW) {
    if (!dev) return fail(c, MPS_ERR_VALIDATION, "site %d: BORROW needs a device pointer", m);
    s.data = (double2*)gamma;
  } else {
    CU(c, cudaMalloc(&s.data, elems * sizeof(double2)), "cudaMalloc(site)");
    s.owned = true;
    CU(c, cudaMemcpy(s.data, gamma, elems * sizeof(double2), dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice),
       "copy site");
  }
  s.chi_l = chi_l;
  s.chi_r = chi_r;
  s.loaded = true;
  c->dtype = MPS_C128;
  const uint64_t N = (uint64_t)chi_r * D;
  if (!make_tmap(&s.tmap, s.data, chi_l, 2 * N, 16 * N, 8))
    return fail(c, MPS_ERR_GENERIC, "site %d: cuTensorMapEncodeTiled failed", m);
  // small-chain copy of the site in the ring's fragment layout (small sites only; no copy -> per-mode path)
  if (chi_l <= SC_KMAX && (int)N <= SC_NMAX) {
    const long long total = (long long)((chi_l + 7) / 8) * (((int)N + 7) / 8) * 64;
    if (cudaMalloc(&s.chain, total * sizeof(double2)) == cudaSuccess) {
      chain_site_kernel<<<(unsigned)((total + 255) / 256), 256>>>(s.data, chi_l, (int)N, s.chain);
      if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
        cudaFree(s.chain);
        s.chain = nullptr;
      }
    } else {
      s.chain = nullptr;
    }
    cudaGetLastError();
  }
  // sum plane Gr + Gi for the 3M GEMM (+50% of the site's bytes); skipped when memory is short
  if (c->sum_planes) {
    const int ld = sum_ld((int)N);
    if (cudaMalloc(&s.gsum, (size_t)chi_l * ld * sizeof(double)) == cudaSuccess) {
      const long long total = (long long)chi_l * (long long)N;
      sum_plane_kernel<<<(unsigned)((total + 255) / 256), 256>>>(s.data, chi_l, (int)N, s.gsum, ld);
      if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess ||
          !make_tmap(&s.tmap_gs, s.gsum, chi_l, N, 8 * (uint64_t)ld, 8)) {
        cudaFree(s.gsum);
        s.gsum = nullptr;
      }
    } else {
      s.gsum = nullptr;
    }
    cudaGetLastError();
  }
  return MPS_OK;
}

int mps_set_streams(mps_ctx* c, uint64_t seed, double alpha_sigma) {
  if (!c) return MPS_ERR_VALIDATION;
  std::lock_guard<std::recursive_mutex> lk_(c->mu);
  if (!(alpha_sigma == alpha_sigma)) return fail(c, MPS_ERR_VALIDATION, "alpha_sigma is NaN");
  // numpy routes a key list holding an int >= 2^63 through float64: the uniform stream keeps that
  // quirk (numpy_key0) but the alpha stream's [seed, 2^62 + i/64] keys would collapse, so refuse
  if (seed >= (1ull << 63)) return fail(c, MPS_ERR_VALIDATION, "seed must be < 2^63, got %llu",
                                        (unsigned long long)seed);
  c->seed = seed;
  c->alpha_sigma = alpha_sigma;
  return MPS_OK;
}

// Device-side pointers of one chain call (host arrays already staged by mps_sample_range).
struct ChainIO {
  const double* u;
  int64_t ld_u;
  const double2* alpha;
  const double2* disp;
  int32_t* counts;
  int64_t ld_c;
  double* marg;
  uint8_t* status;
};

// The mode loop of one micro-batch of n samples over sites [m_begin, m_end) on stream st: the
// persistent small-chain kernel, or K1 + K2/K3 per mode over up to `lanes` row-block chains.
// Every pointer in io is device memory; nothing here synchronises the host.
static int run_chain(mps_ctx* c, int m_begin, int m_end, int64_t first_index, int n, const ChainIO& io,
                     const void* state_in, void* state_out, cudaStream_t st) {
  const int M = c->M, D = c->D;
  const double* u_dev = io.u;
  const int64_t ldu = io.ld_u, ld_c = io.ld_c;
  const double2* alpha_dev = io.alpha;
  const double2* disp_dev = io.disp;
  int32_t* counts_dev = io.counts;
  double* marg_dev = io.marg;
  uint8_t* status_dev = io.status;
  int chi_max = 1;
  for (int m = m_begin; m < m_end; ++m) chi_max = std::max(chi_max, std::max(c->sites[m].chi_l, c->sites[m].chi_r));
  size_t cmax = 0;
  for (int m = m_begin; m < m_end; ++m) cmax = std::max(cmax, (size_t)c->sites[m].chi_r * D);
  // lanes: only when every lane keeps >= 64 rows (below that one chain is latency-bound anyway)
  int L = std::max(1, std::min(c->lanes, n / 64));
  int lane_r0[mps_ctx::MAX_LANES + 1];
  for (int l = 0; l <= L; ++l) lane_r0[l] = (int)((long long)n * l / L);
  const bool c64 = c->dtype == MPS_C64;
  for (int l = 0; l < L; ++l) {
    const size_t nl = (size_t)(lane_r0[l + 1] - lane_r0[l]);
    if (c64) {
      for (int w = 0; w < 2; ++w) {
        CU(c, c->la_hi[w][l].ensure(nl * plane_ld(2 * chi_max)), "alloc c64 state planes");
        CU(c, c->la_lo[w][l].ensure(nl * plane_ld(2 * chi_max)), "alloc c64 state planes");
      }
      CU(c, c->lc32[l].ensure(nl * cmax), "alloc c64 C buffer");
      continue;
    }
    CU(c, c->lv0[l].ensure(nl * chi_max), "alloc state");
    CU(c, c->lv1[l].ensure(nl * chi_max), "alloc state");
    CU(c, c->lcbuf[l].ensure(nl * cmax), "alloc C buffer");
    if (c->gemm_mode == 8) {
      CU(c, c->loz[l].ensure((size_t)c->oz_S * round_up((int)nl, 256) * oz_ld(chi_max)), "alloc digits");
      CU(c, c->loz_e[l].ensure(nl), "alloc digit exponents");
    }
    if (c->sum_planes && c->gemm_mode == 3) {
      CU(c, c->lvs0[l].ensure(nl * sum_ld(chi_max)), "alloc state sums");
      CU(c, c->lvs1[l].ensure(nl * sum_ld(chi_max)), "alloc state sums");
    }
  }
  const bool use_sums = !c64 && c->sum_planes && c->gemm_mode == 3;
  const bool ozaki = !c64 && c->gemm_mode == 8;
  bool oz_stream = false;  // site digits sliced per call, column block by column block
  int oz_cols = 0;         // complex columns per streamed block
  if (ozaki) {
    for (int m = m_begin; m < m_end; ++m) {
      if (c->sites[m].host) return fail(c, MPS_ERR_VALIDATION, "host-streamed sites do not support gemm mode 8");
    }
    size_t need = 0, widest = 0;  // plane bytes still to build; widest per-column plane bytes
    for (int m = m_begin; m < m_end; ++m) {
      const Site& sm = c->sites[m];
      const size_t per_col = (size_t)c->oz_S * 2 * oz_ld(sm.chi_l);
      widest = std::max(widest, per_col);
      if (!(sm.oz && sm.oz_S == c->oz_S)) need += per_col * (size_t)round_up(2 * sm.chi_r * D, 256) / 2;
    }
    oz_stream = c->oz_site_mode == 1;
    if (c->oz_site_mode == 2 && need > 0) {
      size_t free_b = 0, total_b = 0;
      cudaMemGetInfo(&free_b, &total_b);
      oz_stream = need + ((size_t)4 << 30) > free_b;  // keep 4 GB for the call's workspaces
    }
    if (oz_stream) {
      // two ring slots of column blocks: ~4 GB each by default (C5: 10^5 columns in ~7 blocks per site)
      oz_cols = c->oz_block_cols > 0 ? round_up(c->oz_block_cols, 64)
                                     : std::max(64, (int)(((size_t)4 << 30) / widest) / 64 * 64);
      int ncol_max = 0;
      for (int m = m_begin; m < m_end; ++m) ncol_max = std::max(ncol_max, c->sites[m].chi_r * D);
      oz_cols = std::min(oz_cols, round_up(ncol_max, 64));
      for (int w = 0; w < 2; ++w) {
        CU(c, c->ozs_planes[w].ensure(widest / 2 * (size_t)round_up(2 * oz_cols, 256)), "alloc Ozaki digit ring");
        CU(c, c->ozs_e[w].ensure((size_t)2 * oz_cols), "alloc Ozaki digit ring");
      }
      CU(c, cudaEventRecord(c->fork_ev, st), "stream fork");
      CU(c, cudaStreamWaitEvent(c->copy_st, c->fork_ev, 0), "stream fork wait");
    } else {
      for (int m = m_begin; m < m_end; ++m) CU(c, ozaki_prepare_site(c->sites[m], D, c->oz_S), "Ozaki site digits");
    }
  }
  int oz_block = 0;  // streamed blocks issued in this call (ring slot = oz_block % 2)
  mps_ctx::Rec oz_rec[mps_ctx::MAX_LANES];


  if (small_chain_ok(c, m_begin, m_end, n)) {
    CU(c, chain_meta_upload(c), "chain metadata");
    ChainArgs P;
    P.sites = reinterpret_cast<const double2* const*>(c->chain_meta.p);
    P.chi = reinterpret_cast<const int*>(c->chain_meta.p + (size_t)M * sizeof(double2*));
    P.m_begin = m_begin;
    P.m_end = m_end;
    P.n = n;
    P.state_in = (const double2*)state_in;
    P.state_out = (double2*)state_out;
    DrawArgs& a = P.d;
    a = DrawArgs{};
    a.tie_eps = TIE_EPS;
    a.forced = c->forced ? 1 : 0;
    a.D = D;
    a.M = M;
    a.first_index = first_index;
    a.u = u_dev;
    a.ld_u = ldu;
    a.seed = c->seed;
    a.disp = disp_dev;
    a.alpha = alpha_dev;
    a.alpha_sigma = (disp_dev || alpha_dev) ? -1.0 : c->alpha_sigma;
    a.counts = counts_dev;
    a.ld_c = ld_c;
    a.marg = marg_dev;
    a.status = status_dev;
    double flops = 0.0;  // K1 algorithmic flops of the chain (8 per complex MAC)
    for (int m = m_begin; m < m_end; ++m) flops += 8.0 * n * c->sites[m].chi_l * (double)c->sites[m].chi_r * D;
    mps_ctx::Rec rg{0, nullptr, nullptr, flops};
    if (c->profile & 1) {
      rg.a = c->get_event();
      rg.b = c->get_event();
      cudaEventRecord(rg.a, st);
    }
    const cudaError_t le = tiny_chain_ok(c, m_begin, m_end, n) ? launch_tiny_chain(c, P, st) : launch_small_chain(c, P, st);
    if (le != cudaSuccess) {
      // the launch did not happen (no co-resident 16-CTA cluster fits right now: other kernels or
      // MPS clients hold the SMs, cudaErrorClusterOutOfResources / NotSupported ...): the per-mode
      // kernels give the same bits, so fall back to them for this and later calls
      cudaGetLastError();
      c->small_chain = 0;
      if (c->profile & 1) c->event_pool.insert(c->event_pool.end(), {rg.a, rg.b});
    } else {
      c->launches++;
      if (c->profile & 1) {
        cudaEventRecord(rg.b, st);
        c->recs.push_back(rg);
      }
      return MPS_OK;
    }
  }

  // ---- the mode loop: L lanes (row blocks), each a chain on its own stream ----
  const int chi0 = c->sites[m_begin].chi_l;
  if (c64) {
    if (!state_in) {
      CU(c, c->ones_hi.ensure((size_t)n * 4), "alloc ones");
      CU(c, c->ones_lo.ensure((size_t)n * 4), "alloc ones");
      fill_ones_planes_kernel<<<(4 * n + 255) / 256, 256, 0, st>>>(c->ones_hi.p, c->ones_lo.p, n);
    } else {
      const int ld0 = plane_ld(2 * chi0);
      CU(c, c->in_hi.ensure((size_t)n * ld0), "alloc input planes");
      CU(c, c->in_lo.ensure((size_t)n * ld0), "alloc input planes");
      const long long t = (long long)n * ld0;
      split_planes_kernel<<<(unsigned)((t + 255) / 256), 256, 0, st>>>((const float2*)state_in, n, chi0, c->in_hi.p,
                                                                        c->in_lo.p, ld0);
    }
    c->launches++;
  } else if (!state_in) {
    CU(c, c->ones.ensure((size_t)n), "alloc ones");
    CU(c, c->ones_sum.ensure((size_t)n * 2), "alloc ones");
    fill_ones_kernel<<<(n + 255) / 256, 256, 0, st>>>(c->ones.p, c->ones_sum.p, n);
    c->launches++;
  } else if (use_sums) {
    CU(c, c->in_sum.ensure((size_t)n * sum_ld(chi0)), "alloc input sums");
    const long long total = (long long)n * chi0;
    sum_plane_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>((const double2*)state_in, n, chi0, c->in_sum.p,
                                                                      sum_ld(chi0));
    c->launches++;
  }
  cudaStream_t lst[mps_ctx::MAX_LANES];
  if (L == 1) {
    lst[0] = st;
  } else {
    CU(c, cudaEventRecord(c->fork_ev, st), "fork");
    for (int l = 0; l < L; ++l) {
      lst[l] = c->lane_st[l];
      CU(c, cudaStreamWaitEvent(lst[l], c->fork_ev, 0), "fork wait");
    }
  }
  const double2* v_in[mps_ctx::MAX_LANES];
  const double* vs_in[mps_ctx::MAX_LANES];
  int ld_vs_in = sum_ld(chi0);
  int cur[mps_ctx::MAX_LANES];
  const float *a_hi[mps_ctx::MAX_LANES], *a_lo[mps_ctx::MAX_LANES];  // c64 state planes in
  for (int l = 0; l < L; ++l) {
    const int r0 = lane_r0[l];
    cur[l] = 0;
    if (c64) {
      const int ld0 = state_in ? plane_ld(2 * chi0) : 4;
      a_hi[l] = (state_in ? c->in_hi.p : c->ones_hi.p) + (size_t)r0 * ld0;
      a_lo[l] = (state_in ? c->in_lo.p : c->ones_lo.p) + (size_t)r0 * ld0;
      continue;
    }
    v_in[l] = state_in ? (const double2*)state_in + (size_t)r0 * chi0 : c->ones.p + r0;
    vs_in[l] = !use_sums ? nullptr : state_in ? c->in_sum.p + (size_t)r0 * ld_vs_in : c->ones_sum.p + (size_t)r0 * 2;
  }
  // host-streamed sites: stage the next two into the ring ahead of their GEMMs (copy stream)
  std::vector<int> streamed;
  for (int m = m_begin; m < m_end; ++m)
    if (c->sites[m].host) streamed.push_back(m);
  if (!streamed.empty()) {
    size_t smax = 0, sumax = 0;
    for (int m : streamed) {
      smax = std::max(smax, (size_t)c->sites[m].chi_l * c->sites[m].chi_r * D);
      sumax = std::max(sumax, (size_t)c->sites[m].chi_l * sum_ld(c->sites[m].chi_r * D));
    }
    for (int w = 0; w < 2; ++w) {
      CU(c, c->sbuf[w].ensure(smax), "alloc site ring");
      if (use_sums) CU(c, c->ssum[w].ensure(sumax), "alloc site ring sums");
    }
    CU(c, cudaEventRecord(c->fork_ev, st), "stream fork");
    CU(c, cudaStreamWaitEvent(c->copy_st, c->fork_ev, 0), "stream fork wait");
  }
  auto upload = [&](int k) -> int {  // k-th streamed site of this call into slot k % 2
    const int m = streamed[k], w = k % 2;
    const Site& ss = c->sites[m];
    if (k >= 2)  // the slot's previous occupant must have been consumed by every lane's GEMM
      for (int l = 0; l < L; ++l) CU(c, cudaStreamWaitEvent(c->copy_st, c->slot_free[w][l], 0), "slot wait");
    const size_t elems = (size_t)ss.chi_l * ss.chi_r * D;
    CU(c, cudaMemcpyAsync(c->sbuf[w].p, ss.host, elems * sizeof(double2), cudaMemcpyHostToDevice, c->copy_st),
       "H2D streamed site");
    if (use_sums) {
      const long long tot = (long long)elems;
      sum_plane_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, c->copy_st>>>(c->sbuf[w].p, ss.chi_l, ss.chi_r * D,
                                                                             c->ssum[w].p, sum_ld(ss.chi_r * D));
      c->launches++;
    }
    CU(c, cudaEventRecord(c->slot_ready[w], c->copy_st), "slot ready");
    return MPS_OK;
  };
  for (int k = 0; k < (int)streamed.size() && k < 2; ++k)
    if (int rc = upload(k)) return rc;
  int next_stream = 0;

  for (int m = m_begin; m < m_end; ++m) {
    const Site& s0 = c->sites[m];
    Site sl;  // a streamed site's ring view (its own tensor maps)
    int slot = -1;
    if (s0.host) {
      slot = next_stream % 2;
      sl = s0;
      sl.host = nullptr;
      sl.registered = false;
      sl.data = c->sbuf[slot].p;
      sl.gsum = use_sums ? c->ssum[slot].p : nullptr;
      const uint64_t Nn = (uint64_t)s0.chi_r * D;
      if (!make_tmap(&sl.tmap, sl.data, s0.chi_l, 2 * Nn, 16 * Nn, 8) ||
          (sl.gsum && !make_tmap(&sl.tmap_gs, sl.gsum, s0.chi_l, Nn, 8 * (uint64_t)sum_ld((int)Nn), 8)))
        return fail(c, MPS_ERR_GENERIC, "mode %d: streamed site tensor map failed", m);
      for (int l = 0; l < L; ++l) CU(c, cudaStreamWaitEvent(lst[l], c->slot_ready[slot], 0), "slot ready wait");
    }
    const Site& s = s0.host ? sl : s0;
    const int N = s.chi_r * D;
    if (m > m_begin) ld_vs_in = sum_ld(s.chi_l);
    for (int l = 0; l < L; ++l) {  // K1 of every lane, then K2+K3 of every lane
      const int nl = lane_r0[l + 1] - lane_r0[l];
      mps_ctx::Rec rg{0, nullptr, nullptr, 8.0 * nl * (double)s.chi_l * N};
      if (c->profile & 1) {
        rg.a = c->get_event();
        rg.b = c->get_event();
        cudaEventRecord(rg.a, lst[l]);
      }
      if (c64) {
        cudaError_t e = launch_c64_gemm(a_hi[l], a_lo[l], s.bhi, s.blo, s.ld, (float*)c->lc32[l].p, nl, s.chi_l, N,
                                        2LL * N, lst[l]);
        c->launches++;
        if (e != cudaSuccess) return cuda_fail(c, e, "c64 site_gemm launch");
      } else if (ozaki && !oz_stream) {
        const int n_pad = round_up(nl, 256);
        CU(c, ozaki_slice_state(v_in[l], nl, s.chi_l, c->oz_S, c->loz[l].p, n_pad, s.oz_ld, c->loz_e[l].p, lst[l]),
           "Ozaki state digits");
        cudaError_t e = launch_ozaki(c->oz_S, c->loz[l].p, n_pad, c->loz_e[l].p, s.oz, s.oz_pad, s.oz_e, s.oz_ld,
                                     c->lcbuf[l].p, nl, s.chi_l, N, lst[l]);
        c->launches += 2;
        if (e != cudaSuccess) return cuda_fail(c, e, "Ozaki site_gemm launch");
      } else if (ozaki) {  // streamed digits: the state's now, the site's per column block below
        const int n_pad = round_up(nl, 256);
        CU(c, ozaki_slice_state(v_in[l], nl, s.chi_l, c->oz_S, c->loz[l].p, n_pad, oz_ld(s.chi_l), c->loz_e[l].p,
                                lst[l]), "Ozaki state digits");
        c->launches++;
      } else {
        GemmOps o{v_in[l], vs_in[l], ld_vs_in, &s.tmap, s.gsum ? &s.tmap_gs : nullptr, c->lcbuf[l].p, nl, s.chi_l, N,
                  N};
        int rc = launch_site_gemm(c, o, lst[l], c->gemm_cfg, c->gemm_mode);
        if (rc) return rc;
      }
      if (c->profile & 1) {
        if (ozaki && oz_stream) {  // timed around the streamed blocks below instead
          c->event_pool.insert(c->event_pool.end(), {rg.a, rg.b});
        } else {
          cudaEventRecord(rg.b, lst[l]);
          c->recs.push_back(rg);
        }
      }
    }
    if (ozaki && oz_stream) {
      // site digits of this mode, column block by column block, sliced on the copy stream into the
      // 2-slot ring while the previous block's GEMMs run; every lane's GEMM of a block waits for it
      const int ld = oz_ld(s.chi_l), nblk = (N + oz_cols - 1) / oz_cols;
      for (int bk = 0; bk < nblk; ++bk, ++oz_block) {
        const int w = oz_block % 2, c0 = bk * oz_cols, nb = std::min(oz_cols, N - c0);
        if (oz_block >= 2)
          for (int l = 0; l < L; ++l) CU(c, cudaStreamWaitEvent(c->copy_st, c->slot_free[w][l], 0), "digit slot wait");
        ozaki_slice_site_kernel<<<2 * nb, 128, 0, c->copy_st>>>(s.data + c0, s.chi_l, nb, c->oz_S, c->ozs_planes[w].p, ld,
                                                                c->ozs_e[w].p, (long long)N);
        CU(c, cudaGetLastError(), "Ozaki site digits (streamed)");
        c->launches++;
        CU(c, cudaEventRecord(c->slot_ready[w], c->copy_st), "digit slot ready");
        for (int l = 0; l < L; ++l) {
          const int r0 = lane_r0[l], nl = lane_r0[l + 1] - r0;
          if ((c->profile & 1) && bk == 0) {  // K1 of this mode on lane l: first block .. last block
            oz_rec[l] = mps_ctx::Rec{0, c->get_event(), c->get_event(), 8.0 * nl * (double)s.chi_l * N};
            cudaEventRecord(oz_rec[l].a, lst[l]);
          }
          CU(c, cudaStreamWaitEvent(lst[l], c->slot_ready[w], 0), "digit slot ready wait");
          cudaError_t e = launch_ozaki(c->oz_S, c->loz[l].p, round_up(nl, 256), c->loz_e[l].p, c->ozs_planes[w].p,
                                       round_up(2 * nb, 256), c->ozs_e[w].p, ld, c->lcbuf[l].p + c0, nl, s.chi_l, nb,
                                       lst[l], (long long)N);
          c->launches++;
          if (e != cudaSuccess) return cuda_fail(c, e, "Ozaki site_gemm launch (streamed)");
          CU(c, cudaEventRecord(c->slot_free[w][l], lst[l]), "digit slot free");
          if ((c->profile & 1) && bk == nblk - 1) {
            cudaEventRecord(oz_rec[l].b, lst[l]);
            c->recs.push_back(oz_rec[l]);
          }
        }
      }
    }
    if (slot >= 0) {  // the GEMMs of this mode are queued: free the slot for streamed site k+2
      for (int l = 0; l < L; ++l) CU(c, cudaEventRecord(c->slot_free[slot][l], lst[l]), "slot free");
      if (next_stream + 2 < (int)streamed.size())
        if (int rc = upload(next_stream + 2)) return rc;
      ++next_stream;
    }
    for (int l = 0; l < L; ++l) {
      const int r0 = lane_r0[l], nl = lane_r0[l + 1] - r0;
      const bool last_out = (m == m_end - 1 && state_out);
      double2* v_out = c64 ? nullptr
                           : last_out ? (double2*)state_out + (size_t)r0 * s.chi_r : (cur[l] ? c->lv1[l].p : c->lv0[l].p);
      DrawArgs a;
      a.C = c64 ? nullptr : c->lcbuf[l].p;
      a.C32 = c64 ? c->lc32[l].p : nullptr;
      a.v_out32 = (c64 && last_out) ? (float2*)state_out + (size_t)r0 * s.chi_r : nullptr;
      a.a_hi = (c64 && !last_out) ? c->la_hi[cur[l]][l].p : nullptr;
      a.a_lo = (c64 && !last_out) ? c->la_lo[cur[l]][l].p : nullptr;
      a.ld_a = plane_ld(2 * s.chi_r);
      a.tie_eps = c64 ? 1e-4 : TIE_EPS;
      a.forced = c->forced ? 1 : 0;
      a.ldc = N;
      a.chi_r = s.chi_r;
      a.D = D;
      a.m = m;
      a.M = M;
      a.first_index = first_index + r0;
      a.u = u_dev ? u_dev + (size_t)r0 * ldu : nullptr;
      a.ld_u = ldu;
      a.seed = c->seed;
      a.disp = disp_dev ? disp_dev + (size_t)r0 * M * D * D : nullptr;
      a.alpha = alpha_dev ? alpha_dev + (size_t)r0 * M : nullptr;
      a.alpha_sigma = (disp_dev || alpha_dev) ? -1.0 : c->alpha_sigma;
      a.v_out = v_out;
      a.vs_out = (use_sums && !last_out) ? (cur[l] ? c->lvs1[l].p : c->lvs0[l].p) : nullptr;
      a.ld_vs = sum_ld(s.chi_r);
      a.counts = counts_dev + (size_t)r0 * ld_c;
      a.ld_c = ld_c;
      a.marg = marg_dev ? marg_dev + (size_t)r0 * ld_c * D : nullptr;
      a.status = status_dev + r0;
      // algorithmic bytes: C read once, v' written, u read, count written
      mps_ctx::Rec rd{1, nullptr, nullptr, 16.0 * nl * N + 16.0 * nl * s.chi_r + 12.0 * nl};
      if (c->profile & 2) {
        rd.a = c->get_event();
        rd.b = c->get_event();
        cudaEventRecord(rd.a, lst[l]);
      }
      {
        // the C row streams through a shared-memory TMA ring when its bytes are 16-B granular
        const size_t esz = c64 ? 8 : 16;
        const bool ring = c->draw_ring && ((size_t)N * esz) % 16 == 0;
        const size_t ring_bytes =
            ring ? (size_t)(c64 ? draw_ring_slots<true>() : draw_ring_slots<false>()) * DRAW_THREADS * D * esz : 0;
        void (*dk)(DrawArgs) = draw_kernel_for(D, c64, ring);
        if (ring) CU(c, set_smem_once((const void*)dk, 4 * DRAW_THREADS * DMAX * 16), "draw ring smem");
        CU(c, launch_pdl(dk, dim3(nl), dim3(DRAW_THREADS), ring_bytes, lst[l], a), "displace_draw launch");
      }
      c->launches++;
      if (c->profile & 2) {
        cudaEventRecord(rd.b, lst[l]);
        c->recs.push_back(rd);
      }
      v_in[l] = v_out;
      vs_in[l] = a.vs_out;
      a_hi[l] = a.a_hi;
      a_lo[l] = a.a_lo;
      cur[l] ^= 1;
    }
  }
  if (L > 1) {
    for (int l = 0; l < L; ++l) {
      CU(c, cudaEventRecord(c->join_ev[l], lst[l]), "join");
      CU(c, cudaStreamWaitEvent(st, c->join_ev[l], 0), "join wait");
    }
  }
  if (!streamed.empty() || oz_stream) {  // the copy stream's work is older than the GEMMs that waited on it
    CU(c, cudaEventRecord(c->join_ev[0], c->copy_st), "copy join");
    CU(c, cudaStreamWaitEvent(st, c->join_ev[0], 0), "copy join wait");
  }

  return MPS_OK;
}

// One call over n samples with host arrays, as micro-batches of c->micro rows.  Micro-batches are
// grouped into chunks of G (about 2 MB of inputs, at most 64 micro-batches): chunk k's inputs go up on
// cs_in in one copy per field while chunk k-1 computes on st, its outputs come down on cs_out while
// chunk k+1 computes.  Inside a chunk the micro-batches' kernels follow each other on st with nothing
// in between, so programmatic dependent launch overlaps each kernel's prologue with its
// predecessor's tail (an event wait or a copy between two kernels would serialise them).  Host
// arrays that are pinned are copied directly; pageable ones are packed into (inputs) / unpacked from
// (outputs) the context's pinned staging for the whole call.  Device slots are double-buffered per
// chunk: the H2D of chunk k waits for the compute and the D2H of chunk k-2.  One host
// synchronisation per call.  Results are bit-identical to the single-shot path (per-sample results
// do not depend on the split).
static bool is_pinned_host(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

static int sample_pipelined(mps_ctx* c, int m_begin, int m_end, int64_t first_index, int n, const double* uniforms,
                            int64_t ld_u, const void* disp, const void* alpha, const void* state_in, void* state_out,
                            int32_t* counts, int64_t ld_c, double* marginals, uint8_t* status, cudaStream_t st) {
  const int M = c->M, D = c->D, nb = c->micro;
  const int chi0 = c->sites[m_begin].chi_l, chiM = c->sites[m_end - 1].chi_r;
  // fields: host pointer, bytes per row, device-or-host, direction (in / out)
  struct Field {
    const uint8_t* hin;  // host source (inputs)
    uint8_t* hout;       // host destination (outputs)
    size_t row;          // bytes per sample row
    bool in, out;        // host -> device, device -> host
    bool pinned;
    size_t stage_off;    // offset in the pinned whole-call staging (pageable arrays)
    size_t slot_off;     // offset in a device slot
  };
  const bool counts_in = (m_end - m_begin < M || c->forced);
  const bool marg_in = m_end - m_begin < M;
  Field f[6];
  const void* dptr[6] = {uniforms, alpha, disp, counts, marginals, status};
  const size_t rows[6] = {(size_t)ld_u * 8, (size_t)M * 16, (size_t)M * D * D * 16, (size_t)ld_c * 4,
                          (size_t)ld_c * D * 8, 1};
  bool host[6];
  for (int i = 0; i < 6; ++i) host[i] = dptr[i] && !is_device_ptr(dptr[i]);
  size_t in_row = 0;  // host input bytes per sample row
  for (int i = 0; i < 6; ++i) in_row += host[i] ? rows[i] : 0;
  const int T = (n + nb - 1) / nb;
  const int G = (int)std::max<size_t>(1, std::min<size_t>({(size_t)64, (size_t)T,
                                                              ((size_t)2 << 20) / std::max<size_t>(1, (size_t)nb * in_row)}));
  const size_t slot_rows = (size_t)G * nb;
  size_t stage_bytes = 0, slot_bytes = 0;
  for (int i = 0; i < 6; ++i) {
    Field& x = f[i];
    x.row = rows[i];
    x.in = host[i] && (i < 3 || (i == 3 && counts_in) || (i == 4 && marg_in) || i == 5);
    x.out = host[i] && i >= 3;
    x.hin = (const uint8_t*)dptr[i];
    x.hout = (uint8_t*)dptr[i];
    x.pinned = host[i] && is_pinned_host(dptr[i]);
    x.stage_off = stage_bytes;
    if (host[i] && !x.pinned) stage_bytes += ((size_t)n * x.row + 255) & ~(size_t)255;
    x.slot_off = slot_bytes;
    if (host[i] || (i == 5 && !status)) slot_bytes += (slot_rows * x.row + 255) & ~(size_t)255;
  }
  CU(c, c->pipe_d.ensure(2 * slot_bytes), "alloc micro-batch slots");
  if (stage_bytes > c->io_h_cap) {
    if (c->io_h) cudaFreeHost(c->io_h);
    c->io_h = nullptr;
    c->io_h_cap = 0;
    CU(c, cudaMallocHost(&c->io_h, stage_bytes), "alloc pinned staging");
    c->io_h_cap = stage_bytes;
  }
  for (int i = 0; i < 6; ++i)  // pageable inputs: pack once for the whole call
    if (f[i].in && !f[i].pinned) memcpy(c->io_h + f[i].stage_off, f[i].hin, (size_t)n * f[i].row);
  auto hsrc = [&](int i, size_t r0) -> const uint8_t* {
    return (f[i].pinned ? f[i].hin : c->io_h + f[i].stage_off) + r0 * f[i].row;
  };
  auto hdst = [&](int i, size_t r0) -> uint8_t* {
    return (f[i].pinned ? f[i].hout : c->io_h + f[i].stage_off) + r0 * f[i].row;
  };
  auto drain = [&]() {  // queued copies still use the caller's arrays and the staging buffer
    cudaStreamSynchronize(c->cs_in);
    cudaStreamSynchronize(c->cs_out);
    cudaStreamSynchronize(st);
  };
  // the copy streams start after everything already queued on st (the caller's prior work)
  CU(c, cudaEventRecord(c->fork_ev, st), "fork");
  CU(c, cudaStreamWaitEvent(c->cs_in, c->fork_ev, 0), "fork wait");
  CU(c, cudaStreamWaitEvent(c->cs_out, c->fork_ev, 0), "fork wait");
  const int NC = (T + G - 1) / G;
  for (int k = 0; k < NC; ++k) {
    const int w = k & 1;
    const size_t r0 = (size_t)k * slot_rows;
    const int nr = (int)std::min<size_t>(slot_rows, (size_t)n - r0);  // rows of this chunk
    uint8_t* slot = c->pipe_d.p + (size_t)w * slot_bytes;
    if (k >= 2) {  // slot w: chunk k-2's kernels AND the D2H of its in-out fields are done
      CU(c, cudaStreamWaitEvent(c->cs_in, c->pe_comp[w], 0), "slot free");
      CU(c, cudaStreamWaitEvent(c->cs_in, c->pe_d2h[w], 0), "slot read back");
    }
    for (int i = 0; i < 6; ++i)
      if (f[i].in)
        CU(c, cudaMemcpyAsync(slot + f[i].slot_off, hsrc(i, r0), (size_t)nr * f[i].row, cudaMemcpyHostToDevice,
                              c->cs_in), "H2D chunk");
    CU(c, cudaEventRecord(c->pe_in[w], c->cs_in), "inputs ready");
    CU(c, cudaStreamWaitEvent(st, c->pe_in[w], 0), "inputs wait");
    if (!status) CU(c, cudaMemsetAsync(slot + f[5].slot_off, 0, nr, st), "zero status");
    for (int r = 0; r < nr; r += nb) {  // the chunk's micro-batches, back to back on st
      const int nt = std::min(nb, nr - r);
      const size_t g0 = r0 + r;  // global row of this micro-batch
      ChainIO io;
      io.u = !uniforms ? nullptr : host[0] ? (const double*)(slot + f[0].slot_off) + (size_t)r * ld_u : uniforms + g0 * ld_u;
      io.ld_u = ld_u;
      io.alpha = !alpha ? nullptr : host[1] ? (const double2*)(slot + f[1].slot_off) + (size_t)r * M
                                            : (const double2*)alpha + g0 * M;
      io.disp = !disp ? nullptr : host[2] ? (const double2*)(slot + f[2].slot_off) + (size_t)r * M * D * D
                                          : (const double2*)disp + g0 * M * D * D;
      io.counts = host[3] ? (int32_t*)(slot + f[3].slot_off) + (size_t)r * ld_c : counts + g0 * ld_c;
      io.ld_c = ld_c;
      io.marg = !marginals ? nullptr : host[4] ? (double*)(slot + f[4].slot_off) + (size_t)r * ld_c * D
                                               : marginals + g0 * ld_c * D;
      io.status = (!status || host[5]) ? slot + f[5].slot_off + r : status + g0;
      const void* sin = state_in ? (const void*)((const double2*)state_in + g0 * chi0) : nullptr;
      void* sout = state_out ? (void*)((double2*)state_out + g0 * chiM) : nullptr;
      if (c->dtype == MPS_C64) {
        sin = state_in ? (const void*)((const float2*)state_in + g0 * chi0) : nullptr;
        sout = state_out ? (void*)((float2*)state_out + g0 * chiM) : nullptr;
      }
      if (int rc = run_chain(c, m_begin, m_end, first_index + (int64_t)g0, nt, io, sin, sout, st)) {
        drain();
        return rc;
      }
    }
    CU(c, cudaEventRecord(c->pe_comp[w], st), "compute done");
    CU(c, cudaStreamWaitEvent(c->cs_out, c->pe_comp[w], 0), "outputs wait");
    for (int i = 3; i < 6; ++i)
      if (f[i].out)
        CU(c, cudaMemcpyAsync(hdst(i, r0), slot + f[i].slot_off, (size_t)nr * f[i].row, cudaMemcpyDeviceToHost,
                              c->cs_out), "D2H chunk");
    CU(c, cudaEventRecord(c->pe_d2h[w], c->cs_out), "outputs read");
  }
  CU(c, cudaEventRecord(c->pe_out, c->cs_out), "outputs done");
  CU(c, cudaStreamWaitEvent(st, c->pe_out, 0), "join");
  CU(c, cudaStreamSynchronize(st), "stream sync");
  for (int i = 3; i < 6; ++i)  // pageable outputs: unpack once
    if (f[i].out && !f[i].pinned) memcpy(f[i].hout, c->io_h + f[i].stage_off, (size_t)n * f[i].row);
  return MPS_OK;
}

int mps_sample_range(mps_ctx* c, int m_begin, int m_end, int64_t first_index, int n, const double* uniforms,
                     int64_t ld_u, const void* disp, const void* alpha, const void* state_in, void* state_out,
                     int32_t* counts, int64_t ld_c, double* marginals, uint8_t* status, uint64_t stream) {
  if (!c) return MPS_ERR_VALIDATION;
  std::lock_guard<std::recursive_mutex> lk_(c->mu);
  c->err.clear();
  if (c->M == 0) return fail(c, MPS_ERR_VALIDATION, "context not configured");
  if (m_begin < 0 || m_end > c->M || m_begin >= m_end)
    return fail(c, MPS_ERR_VALIDATION, "mode range [%d, %d) invalid for M=%d", m_begin, m_end, c->M);
  if (n < 0) return fail(c, MPS_ERR_VALIDATION, "n must be >= 0");
  if (first_index < 0) return fail(c, MPS_ERR_VALIDATION, "first_index must be >= 0");
  if (!counts) return fail(c, MPS_ERR_VALIDATION, "counts output is required");
  if (ld_c < c->M || (uniforms && ld_u < c->M)) return fail(c, MPS_ERR_VALIDATION, "row strides must be >= M");
  for (int m = m_begin; m < m_end; ++m)
    if (!c->sites[m].loaded) return fail(c, MPS_ERR_VALIDATION, "site %d not loaded", m);
  for (int m = m_begin + 1; m < m_end; ++m)
    if (c->sites[m].chi_l != c->sites[m - 1].chi_r)
      return fail(c, MPS_ERR_VALIDATION, "bond mismatch between sites %d and %d", m - 1, m);
  if (n == 0) return MPS_OK;
  if (!state_in && c->sites[m_begin].chi_l != 1)
    return fail(c, MPS_ERR_VALIDATION, "state_in is required when chi_l of site %d is %d", m_begin,
                c->sites[m_begin].chi_l);
  if (state_in && !is_device_ptr(state_in)) return fail(c, MPS_ERR_VALIDATION, "state_in must be device memory");
  if (state_out && !is_device_ptr(state_out)) return fail(c, MPS_ERR_VALIDATION, "state_out must be device memory");

  cudaSetDevice(c->device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);  // 0 = legacy default stream
  const int M = c->M, D = c->D;
  // ---- inputs: host arrays are packed into one pinned buffer and moved by ONE H2D copy (and the
  //      host outputs come back by one D2H): at C1/C2 sizes a call pays per-copy API latency, not
  //      bytes ----
  const bool u_host = uniforms && !is_device_ptr(uniforms);
  const bool alpha_host = alpha && !is_device_ptr(alpha);
  const bool disp_host = disp && !is_device_ptr(disp);
  const bool counts_host = !is_device_ptr(counts);
  const bool marg_host = marginals && !is_device_ptr(marginals);
  const bool status_host = status && !is_device_ptr(status);
  const bool status_own = !status || status_host;  // the library's status row (zeroed or copied in)
  if (c->micro > 0 && n > c->micro && (u_host || alpha_host || disp_host || counts_host || marg_host || status_host))
    return sample_pipelined(c, m_begin, m_end, first_index, n, uniforms, ld_u, disp, alpha, state_in, state_out,
                            counts, ld_c, marginals, status, st);
  size_t io_off = 0;
  auto field = [&](bool on, size_t bytes) {
    const size_t o = io_off;
    if (on) io_off += (bytes + 255) & ~(size_t)255;
    return o;
  };
  const size_t o_u = field(u_host, (size_t)n * ld_u * sizeof(double));
  const size_t o_a = field(alpha_host, (size_t)n * M * sizeof(double2));
  const size_t o_d = field(disp_host, (size_t)n * M * D * D * sizeof(double2));
  const size_t o_io = io_off;  // outputs (and in-out fields) from here on
  const size_t o_c = field(counts_host, (size_t)n * ld_c * sizeof(int32_t));
  const size_t o_m = field(marg_host, (size_t)n * ld_c * D * sizeof(double));
  const size_t o_s = field(status_own, (size_t)n);
  const size_t io_total = io_off;
  if (io_total > 0) {
    CU(c, c->io_d.ensure(io_total), "alloc staging");
    if (c->io_h_cap < io_total) {
      if (c->io_h) cudaFreeHost(c->io_h);
      c->io_h = nullptr;
      c->io_h_cap = 0;
      CU(c, cudaMallocHost(&c->io_h, io_total), "alloc pinned staging");
      c->io_h_cap = io_total;
    }
  }
  uint8_t* const hb = c->io_h;
  uint8_t* const db = c->io_d.p;
  const bool counts_in = counts_host && (m_end - m_begin < M || c->forced);  // untouched columns / forced outcomes
  const bool marg_in = marg_host && m_end - m_begin < M;
  if (u_host) memcpy(hb + o_u, uniforms, (size_t)n * ld_u * sizeof(double));
  if (alpha_host) memcpy(hb + o_a, alpha, (size_t)n * M * sizeof(double2));
  if (disp_host) memcpy(hb + o_d, disp, (size_t)n * M * D * D * sizeof(double2));
  if (counts_in) memcpy(hb + o_c, counts, (size_t)n * ld_c * sizeof(int32_t));
  if (marg_in) memcpy(hb + o_m, marginals, (size_t)n * ld_c * D * sizeof(double));
  if (status_host) memcpy(hb + o_s, status, n);
  // inputs, plus the in-out tail when any of it carries data in.  Every call that copies from the
  // pinned buffer synchronises before returning (host inputs or host outputs), so the next call may
  // refill it; a library-owned status row is zeroed on the device instead (no host staging).
  const size_t h2d = (status_host || counts_in || marg_in) ? io_total : o_io;
  if (h2d > 0) CU(c, cudaMemcpyAsync(db, hb, h2d, cudaMemcpyHostToDevice, st), "H2D inputs");
  if (!status) CU(c, cudaMemsetAsync(db + o_s, 0, n, st), "zero status");
  ChainIO io;
  io.u = u_host ? reinterpret_cast<const double*>(db + o_u) : uniforms;
  io.ld_u = ld_u;
  io.alpha = alpha_host ? reinterpret_cast<const double2*>(db + o_a) : (const double2*)alpha;
  io.disp = disp_host ? reinterpret_cast<const double2*>(db + o_d) : (const double2*)disp;
  io.counts = counts_host ? reinterpret_cast<int32_t*>(db + o_c) : counts;
  io.ld_c = ld_c;
  io.marg = marg_host ? reinterpret_cast<double*>(db + o_m) : marginals;
  io.status = status_own ? db + o_s : status;

  // ---- outputs back to the host: one D2H of the in-out tail, then host copies ----
  const bool host_out = counts_host || marg_host || status_host;
  const bool host_in = u_host || alpha_host || disp_host;
  auto finish = [&]() -> int {
    if (host_out) CU(c, cudaMemcpyAsync(hb + o_io, db + o_io, io_total - o_io, cudaMemcpyDeviceToHost, st), "D2H outputs");
    // host inputs: the pinned staging is reused by the next call
    if (host_out || host_in) CU(c, cudaStreamSynchronize(st), "stream sync");
    if (counts_host) memcpy(counts, hb + o_c, (size_t)n * ld_c * sizeof(int32_t));
    if (marg_host) memcpy(marginals, hb + o_m, (size_t)n * ld_c * D * sizeof(double));
    if (status_host) memcpy(status, hb + o_s, n);
    return MPS_OK;
  };

  if (int rc = run_chain(c, m_begin, m_end, first_index, n, io, state_in, state_out, st)) return rc;
  return finish();
}

int mps_sample(mps_ctx* c, int64_t first_index, int n, const double* uniforms, const void* disp, const void* alpha,
               int32_t* counts, double* marginals, uint64_t* n_flagged) {
  if (!c) return MPS_ERR_VALIDATION;
  std::lock_guard<std::recursive_mutex> lk_(c->mu);
  if (c->M == 0) return fail(c, MPS_ERR_VALIDATION, "context not configured");
  if (n < 0) return fail(c, MPS_ERR_VALIDATION, "n must be >= 0");
  std::vector<uint8_t> st(n > 0 ? n : 1, 0);
  int rc = mps_sample_range(c, 0, c->M, first_index, n, uniforms, c->M, disp, alpha, nullptr, nullptr, counts, c->M,
                            marginals, st.data(), reinterpret_cast<uint64_t>(c->stream));
  if (rc) return rc;
  uint64_t fl = 0;
  for (int i = 0; i < n; ++i) fl += (st[i] & ST_FLAGGED) ? 1 : 0;
  if (n_flagged) *n_flagged = fl;
  return MPS_OK;
}

uint64_t mps_kernel_launches(const mps_ctx* c) { return c ? c->launches : 0; }

int mps_profile(mps_ctx* c, int enable) {
  if (!c) return MPS_ERR_VALIDATION;
  std::lock_guard<std::recursive_mutex> lk_(c->mu);
  c->profile = enable & 3;
  return MPS_OK;
}

int mps_profile_read(mps_ctx* c, double* out6) {
  if (!c || !out6) return MPS_ERR_VALIDATION;
  std::lock_guard<std::recursive_mutex> lk_(c->mu);
  double acc[6] = {0, 0, 0, 0, 0, 0};  // gemm: ms, launches, flops; draw: ms, launches, bytes
  for (auto& r : c->recs) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    acc[3 * r.kind + 0] += ms;
    acc[3 * r.kind + 1] += 1;
    acc[3 * r.kind + 2] += r.work;
    c->event_pool.push_back(r.a);
    c->event_pool.push_back(r.b);
  }
  c->recs.clear();
  for (int i = 0; i < 6; ++i) out6[i] = acc[i];
  return MPS_OK;
}

const char* mps_last_error(const mps_ctx* c) { return c ? c->err.c_str() : "null context"; }

void mps_destroy(mps_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (auto& s : c->sites) s.release();
  for (int w = 0; w < 2; ++w)
    for (int l = 0; l < mps_ctx::MAX_LANES; ++l) {
      c->la_hi[w][l].release();
      c->la_lo[w][l].release();
    }
  for (int l = 0; l < mps_ctx::MAX_LANES; ++l) {
    c->lc32[l].release();
    c->loz[l].release();
    c->loz_e[l].release();
  }
  c->ones_hi.release();
  c->ones_lo.release();
  c->in_hi.release();
  c->in_lo.release();
  c->ones_sum.release();
  c->in_sum.release();
  for (int l = 0; l < mps_ctx::MAX_LANES; ++l) {
    c->lvs0[l].release();
    c->lvs1[l].release();
    c->lv0[l].release();
    c->lv1[l].release();
    c->lcbuf[l].release();
    if (c->lane_st[l]) cudaStreamDestroy(c->lane_st[l]);
    if (c->join_ev[l]) cudaEventDestroy(c->join_ev[l]);
  }
  if (c->fork_ev) cudaEventDestroy(c->fork_ev);
  for (int w = 0; w < 2; ++w) {
    c->sbuf[w].release();
    c->ssum[w].release();
    if (c->slot_ready[w]) cudaEventDestroy(c->slot_ready[w]);
    for (int l = 0; l < mps_ctx::MAX_LANES; ++l)
      if (c->slot_free[w][l]) cudaEventDestroy(c->slot_free[w][l]);
  }
  if (c->copy_st) cudaStreamDestroy(c->copy_st);
  if (c->cs_in) cudaStreamDestroy(c->cs_in);
  if (c->cs_out) cudaStreamDestroy(c->cs_out);
  for (int w = 0; w < 2; ++w) {
    if (c->pe_in[w]) cudaEventDestroy(c->pe_in[w]);
    if (c->pe_comp[w]) cudaEventDestroy(c->pe_comp[w]);
    if (c->pe_d2h[w]) cudaEventDestroy(c->pe_d2h[w]);
  }
  if (c->pe_out) cudaEventDestroy(c->pe_out);
  c->pipe_d.release();
  for (int w = 0; w < 2; ++w) {
    c->ozs_planes[w].release();
    c->ozs_e[w].release();
  }
  c->ones.release();
  c->io_d.release();
  if (c->io_h) cudaFreeHost(c->io_h);
  c->chain_meta.release();
  for (auto& r : c->recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : c->event_pool) cudaEventDestroy(e);
  cudaStreamDestroy(c->stream);
  delete c;
}

int mps_site_gemm_cfg(const void* V, const void* G, void* C, int n, int K, int N, int64_t ldc, uint64_t stream,
                      int cfg, int mode) {
  if (!V || !G || !C || n < 1 || K < 1 || N < 1 || ldc < N) return MPS_ERR_VALIDATION;
  if (mode != 3 && mode != 4) return MPS_ERR_VALIDATION;
  if (cfg < -2 || cfg >= n_cfgs(mode)) return MPS_ERR_VALIDATION;
  CUtensorMap tg;
  if (!make_tmap(&tg, G, K, 2 * (uint64_t)N, 16 * (uint64_t)N, 8)) return MPS_ERR_GENERIC;
  GemmOps o{V, nullptr, 0, &tg, nullptr, (double2*)C, n, K, N, ldc};
  return launch_site_gemm(nullptr, o, reinterpret_cast<cudaStream_t>(stream), cfg, mode);
}

int mps_site_gemm(const void* V, const void* G, void* C, int n, int K, int N, int64_t ldc, uint64_t stream) {
  return mps_site_gemm_cfg(V, G, C, n, K, N, ldc, stream, -1, 3);
}

int mps_site_gemm_ozaki(const void* V, const void* G, void* C, int n, int K, int N, int S, uint64_t stream) {
  if (!V || !G || !C || n < 1 || K < 1 || N < 1 || S < 5 || S > 7) return MPS_ERR_VALIDATION;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int ld = oz_ld(K), n_pad = round_up(n, 256), b_pad = round_up(2 * N, 256);
  int8_t *ap = nullptr, *bp = nullptr;
  int *ea = nullptr, *eb = nullptr;
  if (cudaMallocAsync(&ap, (size_t)S * n_pad * ld, st) != cudaSuccess ||
      cudaMallocAsync(&bp, (size_t)S * b_pad * ld, st) != cudaSuccess ||
      cudaMallocAsync(&ea, (size_t)n * sizeof(int), st) != cudaSuccess ||
      cudaMallocAsync(&eb, (size_t)2 * N * sizeof(int), st) != cudaSuccess) {
    cudaGetLastError();
    return MPS_ERR_RESOURCE;
  }
  ozaki_slice_rows_kernel<<<n, 128, 0, st>>>((const double2*)V, K, S, ap, ld, ea);
  ozaki_slice_site_kernel<<<2 * N, 128, 0, st>>>((const double2*)G, K, N, S, bp, ld, eb);
  cudaError_t e = launch_ozaki(S, ap, n_pad, ea, bp, b_pad, eb, ld, (double2*)C, n, K, N, st);
  cudaFreeAsync(ap, st);
  cudaFreeAsync(bp, st);
  cudaFreeAsync(ea, st);
  cudaFreeAsync(eb, st);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return MPS_ERR_GENERIC;
  }
  return cudaGetLastError() == cudaSuccess ? MPS_OK : MPS_ERR_GENERIC;
}

int mps_ozaki_state_planes(const void* V, int n, int K, int S, int8_t* planes, int* e, int ld, int n_pad,
                           uint64_t stream) {
  if (!V || !planes || !e || n < 1 || K < 1 || S < 5 || S > 7 || ld < 2 * K || ld % 32 || n_pad < n || n_pad % 256)
    return MPS_ERR_VALIDATION;
  return ozaki_slice_state((const double2*)V, n, K, S, planes, n_pad, ld, e, reinterpret_cast<cudaStream_t>(stream)) ==
                 cudaSuccess
             ? MPS_OK
             : MPS_ERR_GENERIC;
}

int mps_ozaki_site_planes(const void* G, int K, int N, int S, int8_t* planes, int* e, int ld, int b_pad,
                          uint64_t stream) {
  if (!G || !planes || !e || K < 1 || N < 1 || S < 5 || S > 7 || ld < 2 * K || ld % 32 || b_pad < 2 * N ||
      b_pad % 256)
    return MPS_ERR_VALIDATION;
  ozaki_slice_site_kernel<<<2 * N, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>((const double2*)G, K, N, S, planes,
                                                                                     ld, e);
  return cudaGetLastError() == cudaSuccess ? MPS_OK : MPS_ERR_GENERIC;
}

int mps_ozaki_gemm_planes(const int8_t* a_planes, int n_pad, const int* ea, const int8_t* b_planes, int b_pad,
                          const int* eb, int ld, void* C, int n, int K, int N, int S, uint64_t stream) {
  if (!a_planes || !b_planes || !ea || !eb || !C || n < 1 || K < 1 || N < 1 || S < 5 || S > 7 || ld < 2 * K ||
      ld % 32 || n_pad < n || n_pad % 256 || b_pad < 2 * N || b_pad % 256)
    return MPS_ERR_VALIDATION;
  return launch_ozaki(S, a_planes, n_pad, ea, b_planes, b_pad, eb, ld, (double2*)C, n, K, N,
                      reinterpret_cast<cudaStream_t>(stream)) == cudaSuccess
             ? MPS_OK
             : MPS_ERR_GENERIC;
}

int mps_c64_state_planes(const void* V, int rows, int cols, float* hi, float* lo, int ld, uint64_t stream) {
  if (!V || !hi || !lo || rows < 1 || cols < 1 || ld < 2 * cols || ld % 4) return MPS_ERR_VALIDATION;
  const long long t = (long long)rows * ld;
  split_planes_kernel<<<(unsigned)((t + 255) / 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      (const float2*)V, rows, cols, hi, lo, ld);
  return cudaGetLastError() == cudaSuccess ? MPS_OK : MPS_ERR_GENERIC;
}

int mps_c64_site_planes(const void* G, int K, int N, float* hi, float* lo, int ld, uint64_t stream) {
  if (!G || !hi || !lo || K < 1 || N < 1 || ld < 2 * K || ld % 4) return MPS_ERR_VALIDATION;
  const long long t = (long long)2 * N * ld;
  c64_site_planes_kernel<<<(unsigned)((t + 255) / 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      (const float2*)G, K, N, hi, lo, ld);
  return cudaGetLastError() == cudaSuccess ? MPS_OK : MPS_ERR_GENERIC;
}

int mps_c64_gemm_planes(const float* ahi, const float* alo, const float* bhi, const float* blo, int ld, void* C, int n,
                        int K, int N, uint64_t stream) {
  if (!ahi || !alo || !bhi || !blo || !C || n < 1 || K < 1 || N < 1 || ld < 2 * K || ld % 4)
    return MPS_ERR_VALIDATION;
  return launch_c64_gemm(ahi, alo, bhi, blo, ld, (float*)C, n, K, N, 2LL * N, reinterpret_cast<cudaStream_t>(stream)) ==
                 cudaSuccess
             ? MPS_OK
             : MPS_ERR_GENERIC;
}

int mps_site_gemm_c64(const void* V, const void* G, void* C, int n, int K, int N, uint64_t stream) {
  if (!V || !G || !C || n < 1 || K < 1 || N < 1) return MPS_ERR_VALIDATION;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int ld = plane_ld(2 * K);
  float *ahi = nullptr, *alo = nullptr, *bhi = nullptr, *blo = nullptr;
  const size_t a_bytes = (size_t)n * ld * 4, b_bytes = (size_t)2 * N * ld * 4;
  if (cudaMallocAsync(&ahi, a_bytes, st) != cudaSuccess || cudaMallocAsync(&alo, a_bytes, st) != cudaSuccess ||
      cudaMallocAsync(&bhi, b_bytes, st) != cudaSuccess || cudaMallocAsync(&blo, b_bytes, st) != cudaSuccess) {
    cudaGetLastError();
    return MPS_ERR_RESOURCE;
  }
  const long long at = (long long)n * ld, bt = (long long)2 * N * ld;
  split_planes_kernel<<<(unsigned)((at + 255) / 256), 256, 0, st>>>((const float2*)V, n, K, ahi, alo, ld);
  c64_site_planes_kernel<<<(unsigned)((bt + 255) / 256), 256, 0, st>>>((const float2*)G, K, N, bhi, blo, ld);
  cudaError_t e = launch_c64_gemm(ahi, alo, bhi, blo, ld, (float*)C, n, K, N, 2LL * N, st);
  cudaFreeAsync(ahi, st);
  cudaFreeAsync(alo, st);
  cudaFreeAsync(bhi, st);
  cudaFreeAsync(blo, st);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return MPS_ERR_GENERIC;
  }
  return cudaGetLastError() == cudaSuccess ? MPS_OK : MPS_ERR_GENERIC;
}

int mps_set_forced(mps_ctx* c, int enable) {
  if (!c) return MPS_ERR_VALIDATION;
  std::lock_guard<std::recursive_mutex> lk_(c->mu);
  c->forced = enable != 0;
  return MPS_OK;
}

int mps_set_sum_planes(mps_ctx* c, int enable) {
  if (!c) return MPS_ERR_VALIDATION;
  std::lock_guard<std::recursive_mutex> lk_(c->mu);
  c->sum_planes = enable != 0;
  c->chain_dirty = true;
  if (!c->sum_planes)
    for (auto& s : c->sites)
      if (s.gsum) {
        cudaFree(s.gsum);
        s.gsum = nullptr;
      }
  return MPS_OK;
}

int mps_set_small_chain(mps_ctx* c, int mode) {
  if (!c) return MPS_ERR_VALIDATION;
  std::lock_guard<std::recursive_mutex> lk_(c->mu);
  if (mode < 0 || mode > 3) return fail(c, MPS_ERR_VALIDATION, "small-chain mode must be 0, 1, 2 or 3, got %d", mode);
  c->small_chain = mode;
  return MPS_OK;
}

#ifdef TC_TRACE
int mps_debug_tiny_trace(long long* out) {
  return cudaMemcpyFromSymbol(out, tc_trace, sizeof(tc_trace)) == cudaSuccess ? MPS_OK : MPS_ERR_GENERIC;
}
#endif
#ifdef DRAW_TRACE
int mps_debug_draw_trace(int m, long long* out) {  // m >= 0: arm the trace for mode m; m < 0: read it
  if (m >= 0) return cudaMemcpyToSymbol(dr_trace_m, &m, sizeof(int)) == cudaSuccess ? MPS_OK : MPS_ERR_GENERIC;
  return cudaMemcpyFromSymbol(out, dr_trace, sizeof(dr_trace)) == cudaSuccess ? MPS_OK : MPS_ERR_GENERIC;
}
#endif
#ifdef SC_TRACE
int mps_debug_chain_trace(long long* out) {
  return cudaMemcpyFromSymbol(out, sc_trace, sizeof(sc_trace)) == cudaSuccess ? MPS_OK : MPS_ERR_GENERIC;
}
int mps_debug_chain2_trace(long long* out) {
  return cudaMemcpyFromSymbol(out, sc2_trace, sizeof(sc2_trace)) == cudaSuccess ? MPS_OK : MPS_ERR_GENERIC;
}
#endif

int mps_small_chain_eligible(const mps_ctx* c, int m_begin, int m_end, int n) {
  if (!c || m_begin < 0 || m_end > c->M || m_begin >= m_end) return 0;
  for (int m = m_begin; m < m_end; ++m)
    if (!c->sites[m].loaded) return 0;
  return !small_chain_ok(c, m_begin, m_end, n) ? 0 : tiny_chain_ok(c, m_begin, m_end, n) ? 2 : 1;
}

int mps_set_micro_batch(mps_ctx* c, int micro) {
  if (!c) return MPS_ERR_VALIDATION;
  std::lock_guard<std::recursive_mutex> lk_(c->mu);
  if (micro < 0) return fail(c, MPS_ERR_VALIDATION, "micro-batch size must be >= 0, got %d", micro);
  c->micro = micro;
  return MPS_OK;
}

int mps_set_lanes(mps_ctx* c, int lanes) {
  if (!c) return MPS_ERR_VALIDATION;
  std::lock_guard<std::recursive_mutex> lk_(c->mu);
  if (lanes < 1 || lanes > mps_ctx::MAX_LANES)
    return fail(c, MPS_ERR_VALIDATION, "lanes must lie in [1, %d], got %d", mps_ctx::MAX_LANES, lanes);
  c->lanes = lanes;
  return MPS_OK;
}

int mps_set_gemm_mode(mps_ctx* c, int mode) {
  if (!c) return MPS_ERR_VALIDATION;
  std::lock_guard<std::recursive_mutex> lk_(c->mu);
  if (mode != 3 && mode != 4 && mode != 8)
    return fail(c, MPS_ERR_VALIDATION, "gemm mode must be 3 (3M), 4 (4M) or 8 (Ozaki int8), got %d", mode);
  c->gemm_mode = mode;
  return MPS_OK;
}

int mps_set_ozaki_site_mode(mps_ctx* c, int mode, int block_cols) {
  if (!c) return MPS_ERR_VALIDATION;
  std::lock_guard<std::recursive_mutex> lk_(c->mu);
  if (mode < 0 || mode > 2) return fail(c, MPS_ERR_VALIDATION, "Ozaki site mode must be 0, 1 or 2, got %d", mode);
  if (block_cols < 0) return fail(c, MPS_ERR_VALIDATION, "block_cols must be >= 0");
  c->oz_site_mode = mode;
  c->oz_block_cols = block_cols;
  return MPS_OK;
}

int mps_set_ozaki_digits(mps_ctx* c, int S) {
  if (!c) return MPS_ERR_VALIDATION;
  std::lock_guard<std::recursive_mutex> lk_(c->mu);
  if (S < 5 || S > OZ_MAX_S) return fail(c, MPS_ERR_VALIDATION, "Ozaki digits must lie in [5, %d], got %d", OZ_MAX_S, S);
  c->oz_S = S;  // the sites' digit planes are re-sliced on the next gemm-mode-8 call
  return MPS_OK;
}

int mps_set_gemm_config(mps_ctx* c, int cfg) {
  if (!c) return MPS_ERR_VALIDATION;
  std::lock_guard<std::recursive_mutex> lk_(c->mu);
  if (cfg < -2 || cfg >= N_GEMM_CFGS) return fail(c, MPS_ERR_VALIDATION, "gemm config %d outside [-2, %d)", cfg,
                                                  N_GEMM_CFGS);
  c->gemm_cfg = cfg;
  return MPS_OK;
}

int mps_displacement(const void* alpha, int count, int D, void* out, uint64_t stream) {
  if (!alpha || !out || count < 0 || D < 1 || D > DMAX) return MPS_ERR_VALIDATION;
  if (count == 0) return MPS_OK;
  displacement_kernel<<<(count + 127) / 128, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      (const double2*)alpha, count, D, (double2*)out);
  return cudaGetLastError() == cudaSuccess ? MPS_OK : MPS_ERR_GENERIC;
}

// ---- fused stage hand-off over peer memory (mode-pipelined layout) ------------------------------
// The next stage's receive buffers are exported with CUDA IPC and mapped by the previous stage's
// process (NVLink peer memory); its last draw kernel then writes the n x chi state straight into
// them (state_out = the mapped pointer), and interprocess events order producer and consumer on
// the GPU.  No collective runs on the data path.
int mps_ipc_alloc(uint64_t bytes, void** dptr, void* mem_handle64) {
  if (!dptr || !mem_handle64 || bytes == 0) return MPS_ERR_VALIDATION;
  *dptr = nullptr;
  if (cudaMalloc(dptr, bytes) != cudaSuccess) {
    cudaGetLastError();
    return MPS_ERR_RESOURCE;
  }
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, *dptr) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(*dptr);
    *dptr = nullptr;
    return MPS_ERR_GENERIC;
  }
  memcpy(mem_handle64, &h, sizeof(h));
  return MPS_OK;
}
int mps_ipc_free(void* dptr) { return cudaFree(dptr) == cudaSuccess ? MPS_OK : MPS_ERR_GENERIC; }
int mps_ipc_open(const void* mem_handle64, void** dptr) {
  if (!mem_handle64 || !dptr) return MPS_ERR_VALIDATION;
  cudaIpcMemHandle_t h;
  memcpy(&h, mem_handle64, sizeof(h));
  if (cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
    cudaGetLastError();
    return MPS_ERR_GENERIC;
  }
  return MPS_OK;
}
int mps_ipc_close(void* dptr) { return cudaIpcCloseMemHandle(dptr) == cudaSuccess ? MPS_OK : MPS_ERR_GENERIC; }
int mps_ipc_event_create(void** ev, void* ev_handle64) {
  if (!ev || !ev_handle64) return MPS_ERR_VALIDATION;
  cudaEvent_t e;
  if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming | cudaEventInterprocess) != cudaSuccess) {
    cudaGetLastError();
    return MPS_ERR_GENERIC;
  }
  cudaIpcEventHandle_t h;
  if (cudaIpcGetEventHandle(&h, e) != cudaSuccess) {
    cudaGetLastError();
    cudaEventDestroy(e);
    return MPS_ERR_GENERIC;
  }
  memcpy(ev_handle64, &h, sizeof(h));
  *ev = e;
  return MPS_OK;
}
int mps_ipc_event_open(const void* ev_handle64, void** ev) {
  if (!ev_handle64 || !ev) return MPS_ERR_VALIDATION;
  cudaIpcEventHandle_t h;
  memcpy(&h, ev_handle64, sizeof(h));
  cudaEvent_t e;
  if (cudaIpcOpenEventHandle(&e, h) != cudaSuccess) {
    cudaGetLastError();
    return MPS_ERR_GENERIC;
  }
  *ev = e;
  return MPS_OK;
}
int mps_event_record(void* ev, uint64_t stream) {
  return cudaEventRecord((cudaEvent_t)ev, reinterpret_cast<cudaStream_t>(stream)) == cudaSuccess ? MPS_OK
                                                                                                  : MPS_ERR_GENERIC;
}
int mps_stream_wait_event(uint64_t stream, void* ev) {
  return cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(stream), (cudaEvent_t)ev, 0) == cudaSuccess
             ? MPS_OK
             : MPS_ERR_GENERIC;
}
int mps_event_destroy(void* ev) { return cudaEventDestroy((cudaEvent_t)ev) == cudaSuccess ? MPS_OK : MPS_ERR_GENERIC; }

int mps_stream_uniforms(uint64_t seed, int64_t first, int count, int M, double* out, uint64_t stream) {
  if (!out || count < 0 || M < 1 || first < 0) return MPS_ERR_VALIDATION;
  if (count == 0) return MPS_OK;
  long long total = (long long)count * M;
  stream_uniforms_kernel<<<(unsigned)((total + 255) / 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      seed, first, count, M, out, M);
  return cudaGetLastError() == cudaSuccess ? MPS_OK : MPS_ERR_GENERIC;
}

}  // extern "C"
