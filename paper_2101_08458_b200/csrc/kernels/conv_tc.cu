// Host side of the tcgen05 implicit-GEMM kernels: plan selection (tile,
// stages, split-K), TMA tensor-map encoding (tiled / im2col), launch.
//
// The plan is the device realisation of the reference's tensorize schedule
// (tile_and_reorder + GPU sketch, /root/reference/proj/src/rewriter.cpp:245-303,
// 1069-1164): BM x BN is the pragma window (tcgen05 M128 x N), the K block is
// one 128-byte SWIZZLE_128B row (4 MMAs of K=32 i8 / K=16 f16), and
// split_reduction becomes split-K over K blocks with a wrap-add fix-up.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <map>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../tzc_b200_internal.hpp"
#include "conv_tc.cuh"
#include "conv_tc2.cuh"
#include "conv_ws.cuh"
#include "stem_ws.cuh"

#ifdef TZC_TRACE
int g_debug_flags = 0;  // tools/trace_ws only
#endif

namespace {
#if defined(TZC_TRACE) || defined(TZC_CHECKS)
constexpr int kStaticSmem = 1024;  // s_trace / the checks build's per-CTA store bounds
#else
constexpr int kStaticSmem = 0;
#endif
// General-kernel SMEM: EG int8 staging tiles (128 x BN) + the A/B ring + barriers.
int ring_smem(int bn, int kb, int eg, int stages) { return 1024 + eg * 128 * bn + stages * (128 + bn) * kb + 256; }
// Resident-B variant: the ring carries A blocks only, B (num_kb blocks) stays.
int bres_smem(int bn, int kb, int eg, int stages, int num_kb) {
  return 1024 + eg * 128 * bn + stages * 128 * kb + num_kb * bn * kb + 256 + 8 * num_kb;
}
// A-ring depth with all of B resident (0: B does not fit next to a 4-deep ring).
int bres_stages(int bn, int kb, int eg, int num_kb, int static_smem) {
  const int avail = 227 * 1024 - static_smem - 1024 - 256 - 8 * num_kb - eg * 128 * bn - num_kb * bn * kb;
  const int st = std::min(8, avail / (128 * kb));
  return st >= 4 ? st : 0;
}
using tzcb200::Options;
// Ping-pong epilogue groups for tiles of <= o.pingpong_kb K blocks.
int epi_groups_for(int kb_per_tile, const Options& o) { return kb_per_tile <= o.pingpong_kb ? 2 : 1; }

// How the tiles are cut along K.  none: every unit a whole tile.  classic
// split-K (fewer tiles than SMs): every tile split.  tail split: the last,
// less-than-half-full round of tiles is split `splits` ways, so it costs
// ~1/splits of a round instead of a whole one (c5 layers: 196 tiles on 148
// SMs).  Whole tiles keep the fused epilogue; split ones go through the
// int32 fix-up kernel, exact because wrapping adds are associative.
struct WorkSplit {
  int splits = 1;
  int full = 0;  // whole-tile units (they come first)
};
// "split_min_kb": automatic split-K for under-filled grids keeps >= this many
// K blocks per split.  Off by default: in the multi-branch graph step other
// layers' CTAs fill idle SMs, and the int32 partial round trip + fix-up
// launch cost more (batch 32: 511 -> 572 TOPS without it, batch 64: 660 ->
// 804).  "tail_split": measured slower with the separate fix-up kernel.
WorkSplit work_split(int tiles, int tiles_n, int num_kb, int sms, bool ok16, int forced, const Options& o) {
  WorkSplit w;
  w.full = tiles;
  if (forced > 0) {
    w.splits = std::min(forced, num_kb);
    w.full = w.splits > 1 ? 0 : tiles;
    return w;
  }
  if (!ok16) return w;
  if (tiles < sms) {
    // fill the machine, keeping >= split_min_kb K blocks per split (0: off).
    // Off by default: measured at batch 32 (profiles/r02_summary.md §6) a
    // split costs more than the idle SMs it fills even with the in-kernel
    // fix-up (c5_3x3_512: 15.4 us unsplit, 17.5-34 us split 2-4 ways), and in
    // the multi-branch step other layers' CTAs fill those SMs anyway.
    const int min_kb = o.split_min_kb > 0 ? o.split_min_kb : (1 << 20);
    const int s = std::min(std::min((sms + tiles - 1) / tiles, 4), num_kb / std::max(1, min_kb));
    if (s >= 2) {
      w.splits = s;
      w.full = 0;
    }
    return w;
  }
  const int tail = tiles % sms;
  if (o.tail_split && tail > 0 && 2 * tail <= sms && num_kb >= 8) {
    int full = tiles - tail;
    full -= full % tiles_n;  // the split region starts on an M-tile boundary
    const int s = std::min(num_kb / 4, sms / (tiles - full));
    if (s >= 2) {
      w.splits = s;
      w.full = full;
    }
  }
  return w;
}
int ring_stages(int bn, int kb, int eg) {
  return std::min(8, (227 * 1024 - kStaticSmem - 1024 - 256 - eg * 128 * bn) / ((128 + bn) * kb));
}

tzcdev::FastDiv make_fdiv(int64_t d) {
  tzcdev::FastDiv f{};
  f.d = (uint32_t)d;
  if (d > 1) {  // m = ceil(2^64 / d)
    const unsigned __int128 one = (unsigned __int128)1 << 64;
    f.m = (uint64_t)((one + (unsigned __int128)d - 1) / (unsigned __int128)d);
  }
  return f;
}
}  // namespace

namespace tzcb200 {

using tzcdev::ConvCfg;
using tzcdev::ConvKernelParams;

std::atomic<uint64_t> g_launches{0};
thread_local tzc_launch_info g_last_launch{};
thread_local bool g_have_last_launch = false;
void note_launch(int kernel, int cta_group, int bm, int bn, int bk, int a_mode, int grid, int splits) {
  g_last_launch = tzc_launch_info{kernel, cta_group, bm, bn, bk, a_mode, grid, splits};
  g_have_last_launch = true;
}
bool last_launch(tzc_launch_info* out) {
  if (!g_have_last_launch) return false;
  *out = g_last_launch;
  return true;
}

namespace {

PFN_cuTensorMapEncodeTiled_v12000 p_encode_tiled = nullptr;
PFN_cuTensorMapEncodeIm2col_v12000 p_encode_im2col = nullptr;
std::once_flag g_driver_once;
int g_driver_version = 0;

Status load_driver() {
  std::call_once(g_driver_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      p_encode_tiled = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    fn = nullptr;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeIm2col", &fn, 12000, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      p_encode_im2col = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(fn);
    cudaDriverGetVersion(&g_driver_version);
  });
  if (!p_encode_tiled || !p_encode_im2col)
    return Status(TZC_E_DEVICE, "cannot resolve cuTensorMapEncode* from the CUDA driver");
  return Status();
}

}  // namespace

// Per-device facts, cached by device ordinal (a process may drive several
// B200s, one host thread and stream each: SURVEY.md §3.5 step 6).
namespace {
constexpr int kMaxDev = 64;
std::atomic<int> g_dev_state[kMaxDev];  // 0 unknown; low byte 1 = sm_100, 2 = unusable; SM count << 8
int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return dev < kMaxDev ? dev : -1;
}
int dev_state(int dev) {
  if (dev < 0) return 2;
  int st = g_dev_state[dev].load(std::memory_order_acquire);
  if (st) return st;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) {
    cudaGetLastError();
    st = 2;
  } else {
    st = ((prop.major == 10 && prop.minor == 0) ? 1 : 2) | (prop.multiProcessorCount << 8);
  }
  g_dev_state[dev].store(st, std::memory_order_release);
  return st;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device: one bit per
// device ordinal per kernel instantiation.
template <typename Kern>
Status ensure_smem_attr(Kern kern, std::atomic<uint64_t>& done) {
  const int dev = current_device();
  const uint64_t bit = dev >= 0 ? (uint64_t(1) << dev) : 0;
  if (bit && (done.load(std::memory_order_acquire) & bit)) return Status();
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024 - kStaticSmem);
  if (e != cudaSuccess) return Status(TZC_E_DEVICE, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
  done.fetch_or(bit, std::memory_order_acq_rel);
  return Status();
}
}  // namespace

int device_ok() { return (dev_state(current_device()) & 0xff) == 1 ? 1 : 0; }

int num_sms() {
  const int st = dev_state(current_device());
  return (st >> 8) > 0 ? (st >> 8) : 148;
}

namespace {

// Launch with programmatic stream serialization (PDL): the kernel's
// prologue (barrier init, TMEM alloc, descriptor prefetch) overlaps the
// previous grid's tail; griddepcontrol.wait in the kernel keeps the data
// dependency.  Captured into CUDA graphs as programmatic edges.

template <typename Kern>
cudaError_t launch_pdl(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       const ConvKernelParams& p) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, p);
}

template <int BN, int KB, bool F16, int AM, bool BMN, int EPM>
Status launch_kernel(const ConvKernelParams& p, int grid, cudaStream_t stream) {
  auto kern = tzcdev::conv_tc_kernel<BN, KB, F16, AM, BMN, EPM>;
  static std::atomic<uint64_t> attr_done{0};  // per instantiation, one bit per device
  Status sa = ensure_smem_attr(kern, attr_done);
  if (!sa.ok()) return sa;
  const int eg = p.tma_store ? p.epi_groups : 0;  // staging only for TMA stores
  const int smem = p.b_res ? bres_smem(BN, KB, eg, p.stages, p.num_kb) : ring_smem(BN, KB, eg, p.stages);
  cudaError_t e = launch_pdl(kern, dim3(grid), dim3(tzcdev::EpiCfg<BN>::THREADS), smem, stream, p);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  note_launch(0, 1, 128, BN, KB, AM, grid, p.splits);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return Status(TZC_E_DEVICE, std::string("conv_tc launch: ") + cudaGetErrorString(e));
  return Status();
}

// CTA-pair kernel (conv_tc2.cuh): clusters of 2 along x, PDL as above.
int pair_smem(int bn, int stages) { return 1024 + 128 * bn + stages * (128 + bn / 2) * 128 + 256; }
int pair_stages(int bn) { return std::min(8, (227 * 1024 - kStaticSmem - 1024 - 256 - 128 * bn) / ((128 + bn / 2) * 128)); }

template <int BN, int AM>
Status launch_pair(const ConvKernelParams& p, int grid, cudaStream_t stream) {
  auto kern = tzcdev::conv_tc2_kernel<BN, AM>;
  static std::atomic<uint64_t> attr_done{0};  // per instantiation, one bit per device
  Status sa = ensure_smem_attr(kern, attr_done);
  if (!sa.ok()) return sa;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(tzcdev::EpiCfg<BN>::THREADS);
  cfg.dynamicSmemBytes = pair_smem(BN, p.stages);
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = 2;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, p);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  note_launch(3, 2, 256, BN, 128, AM, grid, 1);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return Status(TZC_E_DEVICE, std::string("conv_tc2 launch: ") + cudaGetErrorString(e));
  return Status();
}

Status launch_pair_any(const ConvKernelParams& p, int bn, int am, int grid, cudaStream_t stream) {
  if (bn == 256) return am == tzcdev::A_IM2COL ? launch_pair<256, tzcdev::A_IM2COL>(p, grid, stream)
                                               : launch_pair<256, tzcdev::A_TILED>(p, grid, stream);
  return am == tzcdev::A_IM2COL ? launch_pair<128, tzcdev::A_IM2COL>(p, grid, stream)
                                : launch_pair<128, tzcdev::A_TILED>(p, grid, stream);
}

template <bool F16, int EPM>
Status launch_reduce(const ConvKernelParams& p, cudaStream_t stream) {
  int64_t groups = (int64_t)p.red_rows * (p.Ngemm / 16);
  int blocks = (int)std::min<int64_t>((groups + 255) / 256, 4 * 148);
  cudaError_t e = launch_pdl(tzcdev::splitk_reduce_kernel<F16, EPM>, dim3(blocks), dim3(256), 0, stream, p);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return Status(TZC_E_DEVICE, std::string("split-K reduce launch: ") + cudaGetErrorString(e));
  return Status();
}

// Epilogue mode from the requested kind (i8 kernels: raw i32 or requant;
// f16 kernels: raw f32 or fp16 cast).
template <int BN, int KB, bool F16, int AM, bool BMN>
Status launch_impl(const ConvKernelParams& p, int grid, cudaStream_t stream) {
  const int epm = (p.ep_kind == tzcdev::EP_REQUANT_I8) ? tzcdev::EPM_REQUANT
                  : (p.ep_kind == tzcdev::EP_CAST_F16) ? tzcdev::EPM_F16
                                                       : tzcdev::EPM_RAW;
  constexpr int kAlt = F16 ? tzcdev::EPM_F16 : tzcdev::EPM_REQUANT;
  if (p.splits > 1 && p.splitk_cnt) {  // split-K with the in-kernel fix-up: one launch, the real epilogue
    if (epm == tzcdev::EPM_RAW) return launch_kernel<BN, KB, F16, AM, BMN, tzcdev::EPM_RAW>(p, grid, stream);
    if ((epm == tzcdev::EPM_F16) != F16) return Status(TZC_E_TYPE, "epilogue kind does not match the profile");
    return launch_kernel<BN, KB, F16, AM, BMN, kAlt>(p, grid, stream);
  }
  if (p.splits > 1 && p.full_units == 0) {  // classic split-K: every unit writes partials
    ConvKernelParams pk = p;
    pk.ep_kind = tzcdev::EP_PARTIAL;  // raw partials; the fix-up applies the epilogue
    Status st = launch_kernel<BN, KB, F16, AM, BMN, tzcdev::EPM_RAW>(pk, grid, stream);
    if (!st.ok()) return st;
    return epm == tzcdev::EPM_RAW ? launch_reduce<F16, tzcdev::EPM_RAW>(p, stream) : launch_reduce<F16, kAlt>(p, stream);
  }
  if (p.splits > 1) {  // tail split: whole tiles finish in-kernel, the split tail in the fix-up
    Status st = epm == tzcdev::EPM_RAW ? launch_kernel<BN, KB, F16, AM, BMN, tzcdev::EPM_RAW>(p, grid, stream)
                                       : ((epm == tzcdev::EPM_F16) != F16
                                              ? Status(TZC_E_TYPE, "epilogue kind does not match the profile")
                                              : launch_kernel<BN, KB, F16, AM, BMN, kAlt>(p, grid, stream));
    if (!st.ok()) return st;
    return epm == tzcdev::EPM_RAW ? launch_reduce<F16, tzcdev::EPM_RAW>(p, stream) : launch_reduce<F16, kAlt>(p, stream);
  }
  if (epm == tzcdev::EPM_RAW) return launch_kernel<BN, KB, F16, AM, BMN, tzcdev::EPM_RAW>(p, grid, stream);
  if ((epm == tzcdev::EPM_F16) != F16) return Status(TZC_E_TYPE, "epilogue kind does not match the profile");
  return launch_kernel<BN, KB, F16, AM, BMN, kAlt>(p, grid, stream);
}

using LaunchFn = Status (*)(const ConvKernelParams&, int, cudaStream_t);

#define TZC_KEY(BN, KB, F16, AM, BMN) (((BN) << 8) | ((KB) << 1) | ((F16) << 20) | ((AM) << 21) | ((BMN) << 22))

struct Entry {
  int key;
  LaunchFn fn;
  int smem;
  int stages;
};

#define TZC_E(BN, KB, F16, AM, BMN) \
  {TZC_KEY(BN, KB, F16, AM, BMN), &launch_impl<BN, KB, F16, AM, BMN>, ConvCfg<BN, KB>::SMEM_BYTES, ConvCfg<BN, KB>::STAGES}
#define TZC_E_BN(KB, F16, AM, BMN) TZC_E(64, KB, F16, AM, BMN), TZC_E(128, KB, F16, AM, BMN), TZC_E(256, KB, F16, AM, BMN)

const Entry kTable[] = {
    TZC_E_BN(128, 0, 0, 0), TZC_E_BN(64, 0, 0, 0), TZC_E_BN(128, 0, 1, 0), TZC_E_BN(64, 0, 1, 0),
    TZC_E_BN(128, 1, 0, 0), TZC_E_BN(64, 1, 0, 0), TZC_E_BN(128, 1, 1, 0), TZC_E_BN(64, 1, 1, 0),
    TZC_E(64, 128, 1, 0, 1), TZC_E(128, 128, 1, 0, 1),
};

const Entry* find_entry(int bn, int kb, int f16, int am, int bmn) {
  int key = TZC_KEY(bn, kb, f16, am, bmn);
  for (const auto& e : kTable)
    if (e.key == key) return &e;
  return nullptr;
}

CUtensorMapSwizzle swz(int kb) { return kb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B; }

Status enc_check(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) return Status(TZC_E_DEVICE, std::string(what) + " failed (CUresult " + std::to_string((int)r) + ")");
  return Status();
}

// Device scratch, cached per (device, stream, slot) — slot 0: split-K
// partials, 1: K7 im2col rows / S2D pixels, 2: K7 padded / S2D weights.  Per
// stream so that independent ops captured on parallel graph branches never
// share scratch; launches on one stream are ordered, so reuse within a stream
// is safe.  A buffer that has to grow is RETIRED, not freed: a CUDA graph
// captured earlier on this stream may still hold its address, and freeing it
// would make that graph's next replay read freed memory.  Growth is
// geometric, so the retired bytes stay below the live ones.
std::mutex g_ws_mu;
struct Scratch {  // slot 3: split-K arrival counters (zeroed when allocated)
  void* p[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t bytes[4] = {0, 0, 0, 0};
};
std::map<std::pair<int, cudaStream_t>, Scratch> g_ws;
std::vector<void*> g_ws_retired;

Status workspace(int slot, size_t bytes, void** out, cudaStream_t stream) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  Scratch& s = g_ws[{current_device(), stream}];
  if (bytes > s.bytes[slot]) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(stream, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone)
      return Status(TZC_E_DEVICE,
                    "workspace: scratch must grow while the stream is being captured; run the op once eagerly "
                    "on this stream before capturing it");
    const size_t want = std::max(bytes, s.bytes[slot] + s.bytes[slot] / 2);
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, want);
    if (e != cudaSuccess) return Status(TZC_E_DEVICE, std::string("workspace: ") + cudaGetErrorString(e));
    if (slot == 3) {  // counters start at zero; every use leaves them zero again
      e = cudaMemset(p, 0, want);
      if (e != cudaSuccess) return Status(TZC_E_DEVICE, std::string("workspace: ") + cudaGetErrorString(e));
    }
    if (s.p[slot]) g_ws_retired.push_back(s.p[slot]);
    s.p[slot] = p;
    s.bytes[slot] = want;
  }
  *out = s.p[slot];
  return Status();
}

}  // namespace

// ---- K7 (thin-channel) rewrite ------------------------------------------------
bool needs_k7(const Problem& pb) { return pb.b_kn == 0 && ((int64_t)pb.c * (pb.f16 ? 2 : 1)) % 16 != 0; }

Problem k7_gemm(const Problem& pb, int* kp_out) {
  const int e = pb.f16 ? 2 : 1;
  const int rsc = pb.r * pb.s * pb.c;
  const int kp = (int)((((int64_t)rsc * e + 63) / 64) * 64 / e);  // K padded to 64 bytes
  Problem g = pb;
  g.a_mode = tzcdev::A_TILED;
  g.n = 1;
  g.hp = 1;
  g.wp = (int)pb.m;
  g.r = g.s = g.stride = 1;
  g.oh = 1;
  g.ow = (int)pb.m;
  g.taps = 1;
  g.c = kp;
  g.a_kdim = kp;
  g.a_rows = pb.m;
  g.a_row_stride = kp;
  g.w_stride_k = kp;
  g.w_stride_tap = kp;
  *kp_out = kp;
  return g;
}

struct WsPlan {
  int bn = 0, kb = 0, pair = 0, c_blocks = 0, sr = 0, box_rows = 0, a_slots = 0, smem = 0, tiles = 0, grid = 0;
  int mt = 1;  // 128-row tiles per work unit
  int halo = 0;
  int64_t p_rows = 0;
};
bool ws_plan(const Problem& pb, bool pair, const Options& o, WsPlan* w);
bool s2d_eligible(const Problem& pb);
Problem s2d_problem(const Problem& pb);

// The one routing decision shared by planning and launch: does this problem
// run on the weight-stationary shifted-window kernel (q = the problem it
// runs, the space-to-depth rewrite for the stem)?  A forced split-K (the
// op's split_reduction schedule or the "splits" option) runs on the general
// kernel, which implements it; so does everything the ws kernel cannot hold.
bool stem_fused_eligible(const Problem& pb, const Options& o);
bool ws_route(const Problem& pb, const Options& o, Problem* q, WsPlan* w, bool* s2d) {
  const bool k7 = needs_k7(pb);
  const int forced = pb.forced_splits ? pb.forced_splits : o.splits;
  *s2d = k7 && s2d_eligible(pb);
  if (forced >= 2) return false;
  if (!*s2d && (k7 || !o.shifted_window)) return false;
  *q = *s2d ? s2d_problem(pb) : pb;
  return ws_plan(*q, *s2d && !pb.f16, o, w);
}

// ---- planning ----------------------------------------------------------------
Status plan_problem(const Problem& pb_in, const Options& o, tzc_plan* plan) {
  {
    // the shifted-window kernel (a_mode 2) and the space-to-depth stem (a_mode 3)
    bool s2d = false;
    Problem q;
    WsPlan w;
    if (ws_route(pb_in, o, &q, &w, &s2d)) {
      plan->bm = 128 * w.mt;  // rows per work unit
      plan->bn = w.bn;
      plan->bk_bytes = w.kb;
      plan->stages = w.a_slots;
      plan->a_mode = s2d ? 3 : 2;
      plan->splits = 1;
      plan->grid = w.grid;
      plan->smem_bytes = w.smem;
      plan->tiles_m = w.tiles;
      plan->tiles_n = 1;
      plan->workspace_bytes =
          s2d && !stem_fused_eligible(pb_in, o) ? (int64_t)q.n * q.hp * q.wp * 16 * (pb_in.f16 ? 2 : 1) : 0;
      return Status();
    }
  }
  int kp = 0;
  const Problem pb = needs_k7(pb_in) ? k7_gemm(pb_in, &kp) : pb_in;
  const int e = pb.f16 ? 2 : 1;
  const int64_t krow_bytes = (int64_t)pb.c * e;  // contiguous K run per tap
  // K block: one 128-byte (SWIZZLE_128B) or 64-byte (SWIZZLE_64B) smem row.
  // A ragged last block per tap is zero-filled by TMA out-of-bounds handling
  // (the channel / K extent is the innermost tensor-map dimension), which is
  // exact: zero products (the reference's own pad argument, rewriter.cpp:175-204).
  if (krow_bytes % 16 != 0)
    return Status(TZC_E_INJECT, "reduction run of " + std::to_string(krow_bytes) +
                                    " bytes is not a multiple of 16 (TMA stride); use the K7 path");
  int kb = (krow_bytes % 128 == 0) ? 128 : (krow_bytes % 64 == 0) ? 64 : (krow_bytes > 64 ? 128 : 64);
  if (pb.b_kn) kb = 128;  // MN-major fp16 path is instantiated for 128-byte K blocks
  const int64_t M = pb.m;
  if (M <= 0 || M > INT32_MAX) return Status(TZC_E_SHAPE, "GEMM M out of range");
  // Widest N tile that divides the output channels: every extra N tile
  // re-streams the whole A operand (im2col rows) through L2, which is the
  // binding resource for these layers (ncu: L2-throughput-bound at BN=64).
  int bn = pb.ngemm % 256 == 0 ? 256 : (pb.ngemm % 128 == 0 ? 128 : 64);
  if (pb.b_kn) bn = pb.ngemm % 128 == 0 ? 128 : 64;  // MN-major path instantiated for 64/128
  if (o.bn && pb.ngemm % o.bn == 0 && !(pb.b_kn && o.bn == 256)) bn = o.bn;
  const int sms = num_sms();
  const int tiles_m = (int)((M + 127) / 128);
  const int tiles_n = (pb.ngemm + bn - 1) / bn;
  const int num_kb = (int)(pb.taps * ((krow_bytes + kb - 1) / kb));
  const int tiles = tiles_m * tiles_n;
  const WorkSplit wsplit =
      work_split(tiles, tiles_n, num_kb, sms, pb.ngemm % 16 == 0, pb.forced_splits ? pb.forced_splits : o.splits, o);
  const int splits = wsplit.splits;
  const int64_t red_m0 = (int64_t)(wsplit.full / tiles_n) * 128;
  const Entry* ent = find_entry(bn, kb, pb.f16, pb.a_mode, pb.b_kn);
  if (!ent) return Status(TZC_E_INTERNAL, "no kernel instantiation for this plan");
  plan->bm = 128;
  plan->bn = bn;
  plan->bk_bytes = kb;
  // ping-pong epilogue groups where the epilogue dominates (one K block
  // per tile); otherwise one group and the deepest ring
  const int eg = epi_groups_for(num_kb / splits, o);
  plan->stages = ring_stages(bn, kb, eg);
  plan->a_mode = pb.a_mode;
  plan->splits = splits;
  plan->tiles_m = tiles_m;
  plan->tiles_n = tiles_n;
  plan->grid = std::min(wsplit.full + (tiles - wsplit.full) * splits, sms);
  plan->smem_bytes = ring_smem(bn, kb, eg, plan->stages);
  plan->workspace_bytes = splits > 1 ? (int64_t)splits * (M - red_m0) * pb.ngemm * 4 : 0;
  if ((o.b_res == 1 || (o.b_res == 2 && pb.taps == 1)) && splits == 1 && wsplit.full == tiles &&
      plan->grid % tiles_n == 0 && tiles >= 2 * plan->grid) {
    const int st = bres_stages(bn, kb, 0, num_kb, kStaticSmem);  // as run_problem decides (no TMA-store staging)
    if (st) {
      plan->stages = st;
      plan->smem_bytes = bres_smem(bn, kb, 0, st, num_kb);
    }
  }
  return Status();
}

// Output layout, seed and fused-epilogue fields shared by both kernels.
void fill_epilogue(ConvKernelParams* pp, const Problem& pb, const Options& o, const void* seed, void* out,
                   const tzc_epilogue& ep);
// ---- weight-stationary shifted-window path (conv_ws.cuh) --------------------------

namespace {

// A super-tile TMA geometry: boxes of <= 256 rows.  Pair mode reads the
// 16-byte pixels as 128-byte rows of 8 pixels (8x fewer TMA requests; the
// SMEM bytes are the same dense pixel array).
void ws_boxes(const WsPlan& w, int* nbox, int* box_rows, int* box_bytes, int* div) {
  if (w.pair) {
    *div = 8;
    *box_rows = (w.sr + 7) / 8 + 1;  // +1: q0/8 alignment slack is zero (q0 % 128 == 0), keep one spare row
    *nbox = 1;
    *box_bytes = *box_rows * 128;
    return;
  }
  // <= 256-row boxes, each a multiple of 8 rows so consecutive boxes continue
  // the swizzle pattern of one contiguous super-tile
  *div = 1;
  *nbox = (w.sr + 255) / 256;
  *box_rows = ((w.sr + *nbox - 1) / *nbox + 7) / 8 * 8;
  *box_bytes = *box_rows * w.kb;
}

int ws_smem(const WsPlan& w, int taps) {
  const int b = ((taps * w.c_blocks * w.bn * w.kb + 1023) / 1024) * 1024;
  int nbox, rows, bytes, div;
  ws_boxes(w, &nbox, &rows, &bytes, &div);
  const int slot = ((nbox * bytes + 1023) / 1024) * 1024;
  return 1024 + b + w.a_slots * slot + 256;
}

template <int BN, int KB, bool F16, bool PAIR, int EPM>
Status launch_ws_kernel(const ConvKernelParams& p, int grid, int smem, cudaStream_t stream) {
  auto kern = tzcdev::conv_ws_kernel<BN, KB, F16, PAIR, EPM>;
  static std::atomic<uint64_t> attr_done{0};  // per instantiation, one bit per device
  Status sa = ensure_smem_attr(kern, attr_done);
  if (!sa.ok()) return sa;
  cudaError_t e = launch_pdl(kern, dim3(grid), dim3(tzcdev::EpiCfg<BN>::THREADS), smem, stream, p);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  note_launch(PAIR ? 2 : 1, 1, 128 * p.mt, BN, KB, PAIR ? 3 : 2, grid, 1);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return Status(TZC_E_DEVICE, std::string("conv_ws launch: ") + cudaGetErrorString(e));
  return Status();
}

template <int BN, int KB, bool F16, bool PAIR>
Status launch_ws_epm(const ConvKernelParams& p, int grid, int smem, cudaStream_t stream) {
  if (p.ep_kind == tzcdev::EP_REQUANT_I8) {
    if constexpr (F16) return Status(TZC_E_TYPE, "requant epilogue on an fp16 op");
    else return launch_ws_kernel<BN, KB, F16, PAIR, tzcdev::EPM_REQUANT>(p, grid, smem, stream);
  }
  if (p.ep_kind == tzcdev::EP_CAST_F16) {
    if constexpr (!F16) return Status(TZC_E_TYPE, "fp16 cast epilogue on an int8 op");
    else return launch_ws_kernel<BN, KB, F16, PAIR, tzcdev::EPM_F16>(p, grid, smem, stream);
  }
  return launch_ws_kernel<BN, KB, F16, PAIR, tzcdev::EPM_RAW>(p, grid, smem, stream);
}

using WsFn = Status (*)(const ConvKernelParams&, int, int, cudaStream_t);

WsFn ws_fn(int bn, int kb, bool f16, bool pair) {
#define TZC_WS(BN, KB, F16, PAIR) \
  if (bn == BN && kb == KB && f16 == F16 && pair == PAIR) return &launch_ws_epm<BN, KB, F16, PAIR>;
  TZC_WS(64, 64, false, false) TZC_WS(128, 64, false, false) TZC_WS(256, 64, false, false)
  TZC_WS(64, 128, false, false) TZC_WS(128, 128, false, false) TZC_WS(256, 128, false, false)
  TZC_WS(64, 16, false, true) TZC_WS(128, 16, false, true) TZC_WS(256, 16, false, true)
  TZC_WS(64, 64, true, false) TZC_WS(128, 64, true, false) TZC_WS(256, 64, true, false)
  TZC_WS(64, 128, true, false) TZC_WS(128, 128, true, false) TZC_WS(256, 128, true, false)
  TZC_WS(64, 32, true, false) TZC_WS(128, 32, true, false) TZC_WS(256, 32, true, false)
#undef TZC_WS
  return nullptr;
}

}  // namespace

// Eligibility + resources of the shifted-window kernel for a stride-1 conv
// (pair = 16-byte pixels, the space-to-depth stem).
bool ws_plan(const Problem& pb, bool pair, const Options& o, WsPlan* w) {
  if (pb.b_kn || pb.stride != 1 || needs_k7(pb)) return false;
  if (o.bn && o.bn != pb.ngemm) return false;  // a narrower N tile (the instruction's N) runs on the general kernel
  // 1x1: weight-stationary pays off only for a single 64-wide N tile and one
  // K block (c2_1x1_64_64: 43 -> 31 us at batch 256); wider layers keep the
  // TMA-store general kernel (measured, tools/layer_timing.py --opt ws_1x1=1)
  // With the direct 256-bit-store epilogue the single-K-block 1x1 layers of
  // any width gain too (c2_1x1_64_256: 96 -> 76 us): "ws_1x1_k" bytes of K.
  if (pb.taps < 2 && !o.ws_1x1 && !(pb.ngemm == 64 && (int64_t)pb.c * (pb.f16 ? 2 : 1) <= 128) &&
      !((int64_t)pb.c * (pb.f16 ? 2 : 1) <= o.ws_1x1_k))
    return false;
  if (!(pb.ngemm == 64 || pb.ngemm == 128 || pb.ngemm == 256)) return false;
  const int e = pb.f16 ? 2 : 1;
  const int64_t cb = (int64_t)pb.c * e;
  WsPlan x;
  x.bn = pb.ngemm;
  x.pair = pair ? 1 : 0;
  if (pair) {
    // the pair kernel is specialised for the 4 x 4-tap space-to-depth stem (8 MMAs per tile)
    if (cb != 16 || pb.r != 4 || pb.s != 4 || pb.f16) return false;
    x.kb = 16;
  } else {
    x.kb = cb % 128 == 0 ? 128 : (cb % 64 == 0 ? 64 : (pb.f16 && cb == 32 ? 32 : 0));  // 32: the fp16 S2D stem
    if (!x.kb) return false;
  }
  x.c_blocks = (int)(cb / x.kb);
  if ((pair ? pb.taps / 2 : pb.taps * (x.kb / 32)) > 64) return false;  // ConvKernelParams::mma_a capacity
  if ((int64_t)pb.taps * x.c_blocks * x.bn * x.kb > 160 * 1024) return false;  // weights must stay resident
  x.halo = (pb.r - 1) * pb.wp + (pb.s - 1);
  if (128 + x.halo > 1024) return false;
  // padded-grid waste: (Hp*Wp)/(OH*OW) extra MMA rows
  if ((double)pb.hp * pb.wp > 1.35 * (double)pb.oh * pb.ow) return false;
  x.p_rows = (int64_t)pb.n * pb.hp * pb.wp;
  if (x.p_rows + 128 >= (int64_t(1) << 22) || (int64_t)pb.hp * pb.wp >= (1 << 18)) return false;  // exact magic division
  const int tiles = (int)((x.p_rows + 127) / 128);
  const int sms = num_sms();
  // MT tiles per unit: the largest that fits TMEM (2*MT*BN <= 512) and SMEM
  // (>= 2 super-tile slots next to the resident weights), keeps every CTA
  // busy for >= 8 units and loses <= 6% to the last round's imbalance.  A
  // forced "ws_mt" skips the occupancy rules (only the resources bind), so
  // tests can run every MT at small batches.
  for (int mt : {4, 2, 1}) {
    if (2 * mt * x.bn > 512) continue;
    if (o.ws_mt && mt != o.ws_mt) continue;
    const int units = (tiles + mt - 1) / mt;
    if (mt > 1 && !o.ws_mt) {
      if (units < 8 * sms) continue;
      const double rounds = std::ceil((double)units / sms), ideal = (double)units / sms;
      if (rounds > 1.06 * ideal) continue;
    }
    WsPlan y = x;
    y.mt = mt;
    y.sr = mt * 128 + x.halo;
    for (y.a_slots = 6; y.a_slots >= 2; --y.a_slots)
      if (ws_smem(y, pb.taps) <= 227 * 1024 - kStaticSmem) break;
    if (y.a_slots < 2) continue;
    if (mt > 1 && y.a_slots < 3) continue;  // a deeper ring beats a bigger unit
    y.smem = ws_smem(y, pb.taps);
    y.tiles = units;
    y.grid = std::min(units, sms);
    *w = y;
    return true;
  }
  return false;
}

Status run_ws(const Problem& pb, const WsPlan& w, const Options& o, const void* a, const void* b, const void* seed,
              void* out, const tzc_epilogue& ep, cudaStream_t stream) {
  const int e = pb.f16 ? 2 : 1;
  const int KE = w.kb / e;
  const CUtensorMapDataType dt = pb.f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_UINT8;
  const CUtensorMapSwizzle sw = w.kb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : w.kb == 64  ? CU_TENSOR_MAP_SWIZZLE_64B
                                : w.kb == 32  ? CU_TENSOR_MAP_SWIZZLE_32B
                                              : CU_TENSOR_MAP_SWIZZLE_NONE;
  ConvKernelParams p;
  std::memset(&p, 0, sizeof(p));
  Status st;
  int nbox, box_rows, box_bytes, div;
  ws_boxes(w, &nbox, &box_rows, &box_bytes, &div);
  {  // A: the input as a [N*Hp*Wp pixel rows, C] matrix (pair mode: [P/8, 128 B])
    cuuint64_t dims[2] = {(cuuint64_t)pb.c, (cuuint64_t)w.p_rows};
    cuuint64_t strides[1] = {(cuuint64_t)pb.c * e};
    cuuint32_t box[2] = {(cuuint32_t)KE, (cuuint32_t)box_rows};
    if (w.pair) {  // workspace is padded to a whole number of 8-pixel rows
      dims[0] = 128;
      dims[1] = (cuuint64_t)((w.p_rows + 7) / 8);
      strides[0] = 128;
      box[0] = 128;
    }
    cuuint32_t es[2] = {1, 1};
    st = enc_check(p_encode_tiled(&p.tmA, dt, 2, const_cast<void*>(a), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                  sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
                   "cuTensorMapEncodeTiled(ws A)");
    if (!st.ok()) return st;
  }
  {  // B: (c, k_out, tap); the pair kernel takes two taps per box
    const int64_t sk = pb.w_stride_k * e, stap = pb.w_stride_tap * e;
    cuuint64_t dims[3] = {(cuuint64_t)pb.c, (cuuint64_t)pb.ngemm, (cuuint64_t)pb.taps};
    cuuint64_t strides[2] = {(cuuint64_t)sk, (cuuint64_t)stap};
    cuuint32_t box[3] = {(cuuint32_t)KE, (cuuint32_t)w.bn, (cuuint32_t)(w.pair ? 2 : 1)};
    cuuint32_t es[3] = {1, 1, 1};
    st = enc_check(p_encode_tiled(&p.tmB, dt, 3, const_cast<void*>(b), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                  sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
                   "cuTensorMapEncodeTiled(ws B)");
    if (!st.ok()) return st;
  }
  p.M = (int32_t)pb.m;
  p.Ngemm = pb.ngemm;
  p.c_blocks = w.c_blocks;
  p.S = pb.s;
  p.R = pb.r;
  p.Hp = pb.hp;
  p.Wp = pb.wp;
  p.OH = pb.oh;
  p.OWv = pb.ow;
  p.P = (int32_t)w.p_rows;
  p.SR = w.sr;
  p.box_rows = box_rows;
  p.a_nbox = nbox;
  {  // MMA table of one channel block (kernel adds cb * b_tile to B)
    const int b_tile = w.bn * w.kb;
    int i = 0;
    for (int r = 0; r < pb.r; ++r)
      for (int s = 0; s < pb.s; s += (w.pair ? 2 : 1))
        for (int k = 0; k < (w.pair ? 1 : w.kb / 32); ++k, ++i) {
          if (w.pair) {
            p.mma_a[i] = (uint32_t)(r * pb.wp + s);  // 16-byte pixels
            p.mma_b[i] = (uint32_t)(((r * pb.s + s) * b_tile) >> 4);
          } else {
            p.mma_a[i] = (uint32_t)(((r * pb.wp + s) * w.kb + 32 * k) >> 4);
            p.mma_b[i] = (uint32_t)((((r * pb.s + s) * w.c_blocks) * b_tile + 32 * k) >> 4);
          }
        }
    p.n_mma = i;
  }
#ifdef TZC_TRACE
  p.debug_flags = ::g_debug_flags;
#endif
  p.pol_a = (o.l2_hints & 1) ? tzcdev::kL2EvictFirst : 0;
  p.pol_b = (o.l2_hints & 2) ? tzcdev::kL2EvictLast : 0;
  p.magic_hw = ((uint64_t(1) << 40) + (uint64_t)pb.hp * pb.wp - 1) / ((uint64_t)pb.hp * pb.wp);
  p.magic_wp = ((uint64_t(1) << 40) + (uint64_t)pb.wp - 1) / (uint64_t)pb.wp;
  p.a_box_bytes = box_bytes;
  p.a_coord_div = div;
  p.num_tiles = w.tiles;
  p.splits = w.a_slots;  // ring depth (the kernel has no split-K)
  p.mt = w.mt;
  // as many accumulators as TMEM holds (<= 4): the epilogue may lag the MMAs
  // by NACC-1 units (the ping-pong epilogue groups need exactly 2)
  // epilogue groups: "ws_epi_groups" 1 / 2, or 0 = by shape: two ping-pong
  // groups for the 3x3 layers (a unit's 9-tap MMA phase is long enough for the
  // groups to alternate; c2_3x3_64 38.0 -> 36.7 us, c3_3x3_128 27.4 -> 26.1),
  // one for 1x1 and the pair-mode stem (stem 86.0 -> 87.9 with two)
  const int eg = o.ws_epi_groups ? o.ws_epi_groups : (!w.pair && pb.r * pb.s >= 9 ? 2 : 1);
  p.nacc = eg == 2 ? 2 : std::min(4, 512 / (w.mt * w.bn));
  p.epi_groups = eg;
  fill_epilogue(&p, pb, o, seed, out, ep);
  WsFn fn = ws_fn(w.bn, w.kb, pb.f16 != 0, w.pair != 0);
  if (!fn) return Status(TZC_E_INTERNAL, "no conv_ws instantiation");
  return fn(p, w.grid, w.smem, stream);
}

// ---- the fused space-to-depth stem (stem_ws.cuh) ----------------------------
// Eligible: int8 C = 3 stride-2 stems whose space-to-depth problem has a pair
// plan (ws_plan), 16-byte aligned input, 32-bit byte offsets.  q = the S2D
// problem (s2d_problem), w = its plan.
bool stem_fused_eligible(const Problem& pb, const Options& o) {
  return o.stem_fused && !pb.f16 && pb.c == 3 && pb.stride == 2 && pb.r <= 8 && pb.s <= 8 &&
         (int64_t)pb.n * pb.hp * pb.wp * 3 < (int64_t(1) << 31) - 65536;
}

template <int BN, int EPM>
Status launch_stem(const ConvKernelParams& p, int grid, int smem, cudaStream_t stream) {
  auto kern = tzcdev::stem_ws_kernel<BN, EPM>;
  static std::atomic<uint64_t> attr_done{0};
  Status sa = ensure_smem_attr(kern, attr_done);
  if (!sa.ok()) return sa;
  cudaError_t e = launch_pdl(kern, dim3(grid), dim3(tzcdev::EpiCfg<BN>::THREADS), smem, stream, p);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  note_launch(5, 1, 128 * p.mt, BN, 16, 3, grid, 1);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return Status(TZC_E_DEVICE, std::string("stem_ws launch: ") + cudaGetErrorString(e));
  return Status();
}

Status run_stem_fused(const Problem& pb, const Problem& q, const WsPlan& w, const Options& o, const void* x,
                      const void* wt, const void* seed, void* out, const tzc_epilogue& ep, cudaStream_t stream) {
  ConvKernelParams p;
  std::memset(&p, 0, sizeof(p));
  // raw bytes one work unit needs: from its first S2D row's first raw byte to
  // the last byte of its last pixel's two raw rows (exact, over all units)
  const int64_t hw4 = (int64_t)q.hp * q.wp, P = (int64_t)q.n * hw4, unit = (int64_t)w.mt * 128;
  int64_t need = 0;
  for (int64_t q0 = 0; q0 < P; q0 += unit) {
    const int64_t n0 = q0 / hw4, i0 = (q0 % hw4) / q.wp;
    const int64_t base = ((n0 * pb.hp + 2 * i0) * pb.wp * 3) & ~int64_t(15);  // 16-byte aligned box start
    const int64_t ql = std::min(q0 + w.sr, P) - 1;
    const int64_t n = ql / hw4, i = (ql % hw4) / q.wp;
    const int64_t h = std::min<int64_t>(2 * i + 1, pb.hp - 1);
    const int64_t end = ((n * pb.hp + h) * pb.wp + pb.wp) * 3;  // through the end of that raw row
    need = std::max(need, end - base);
  }
  p.raw_boxes = (int)((need + 255) / 256);
  // + slack: the transform reads a masked row h+1 one raw row past the last
  // staged byte (odd image heights), and 12-byte word groups past a row end
  p.raw_slot = ((p.raw_boxes * 256 + pb.wp * 3 + 64 + 1023) / 1024) * 1024;
  const int b_bytes = ((16 * w.bn * 16 + 1023) / 1024) * 1024;
  const int a_slot = ((w.sr * 16 + 1023) / 1024) * 1024;
  int a_slots = 4, r_slots = 3;
  auto smem_of = [&](int as, int rs) { return 1024 + b_bytes + as * a_slot + rs * p.raw_slot + 512; };
  while (smem_of(a_slots, r_slots) > 227 * 1024 - kStaticSmem && (a_slots > 2 || r_slots > 2)) {
    if (a_slots >= r_slots && a_slots > 2) --a_slots;
    else --r_slots;
  }
  const int smem = smem_of(a_slots, r_slots);
  if (smem > 227 * 1024 - kStaticSmem) return Status(TZC_E_INTERNAL, "fused stem: shared memory");
  {  // A: the input as a 1-D byte tensor (TMA boxes of 256 bytes, 16-byte aligned starts)
    cuuint64_t dims[1] = {(cuuint64_t)pb.n * pb.hp * pb.wp * 3};
    cuuint64_t strides[1] = {dims[0]};  // rank 1 has no strides; the driver wants a valid array
    cuuint32_t box[1] = {256};
    cuuint32_t es[1] = {1};
    Status st = enc_check(p_encode_tiled(&p.tmA, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, const_cast<void*>(x), dims, strides,
                                         box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
                          "cuTensorMapEncodeTiled(stem raw)");
    if (!st.ok()) return st;
  }
  p.wraw = wt;
  if (const char* dbg = std::getenv("TZC_STEM_DEBUG")) p.debug_flags = std::atoi(dbg);  // bring-up only
  p.w_sk = pb.w_stride_k;
  p.w_st = pb.w_stride_tap;
  p.w_r = pb.r;
  p.w_s = pb.s;
  p.raw_hp = pb.hp;
  p.raw_wp = pb.wp;
  p.raw_c = 3;
  p.raw_slots = r_slots;
  p.M = (int32_t)pb.m;
  p.Ngemm = pb.ngemm;
  p.Hp = q.hp;
  p.Wp = q.wp;
  p.OH = pb.oh;
  p.OWv = pb.ow;
  p.P = (int32_t)P;
  p.SR = w.sr;
  {  // MMA table: pair MMAs over taps (r, s), (r, s+1) of the 4 x 4 S2D filter
    int i = 0;
    for (int r = 0; r < 4; ++r)
      for (int s = 0; s < 4; s += 2, ++i) {
        p.mma_a[i] = (uint32_t)(r * q.wp + s);
        p.mma_b[i] = (uint32_t)(((r * 4 + s) * w.bn * 16) >> 4);
      }
    p.n_mma = i;
  }
  p.magic_hw = ((uint64_t(1) << 40) + (uint64_t)hw4 - 1) / (uint64_t)hw4;
  p.magic_wp = ((uint64_t(1) << 40) + (uint64_t)q.wp - 1) / (uint64_t)q.wp;
  p.magic_wp32 = (uint32_t)(((uint64_t(1) << 32) + (uint64_t)q.wp - 1) / (uint64_t)q.wp);
  if ((int64_t)w.sr + q.wp >= 65536) return Status(TZC_E_INTERNAL, "fused stem: unit too long for the 16-bit divide");
  p.num_tiles = w.tiles;
  p.splits = a_slots;
  p.mt = w.mt;
  p.nacc = o.ws_epi_groups == 2 ? 2 : std::min(4, 512 / (w.mt * w.bn));  // the fused stem: one group unless forced
  p.epi_groups = o.ws_epi_groups == 2 ? 2 : 1;
  fill_epilogue(&p, pb, o, seed, out, ep);
  const bool rq = ep.kind == tzcdev::EP_REQUANT_I8;
  if (ep.kind != tzcdev::EP_I32 && !rq) return Status(TZC_E_TYPE, "fused stem: int8 ops take i32 or requant epilogues");
  switch (w.bn) {
    case 64: return rq ? launch_stem<64, tzcdev::EPM_REQUANT>(p, w.grid, smem, stream)
                       : launch_stem<64, tzcdev::EPM_RAW>(p, w.grid, smem, stream);
    case 128: return rq ? launch_stem<128, tzcdev::EPM_REQUANT>(p, w.grid, smem, stream)
                        : launch_stem<128, tzcdev::EPM_RAW>(p, w.grid, smem, stream);
    default: return rq ? launch_stem<256, tzcdev::EPM_REQUANT>(p, w.grid, smem, stream)
                       : launch_stem<256, tzcdev::EPM_RAW>(p, w.grid, smem, stream);
  }
}

// Space-to-depth geometry for a stride-2 conv with 4*C*e <= 16 (the stem).
// int8: 16-byte S2D pixels (pair mode); fp16: C = 3 only (12 of 16 halfs per
// 32-byte pixel, one K=16 MMA per tap), even padded extents.
bool s2d_eligible(const Problem& pb) {
  if (pb.stride != 2 || pb.b_kn || pb.r <= 1 || !(pb.ngemm == 64 || pb.ngemm == 128 || pb.ngemm == 256)) return false;
  if (pb.f16) return pb.c == 3 && pb.hp % 2 == 0 && pb.wp % 2 == 0;
  return pb.c * 4 <= 16;
}

Problem s2d_problem(const Problem& pb) {
  Problem q = pb;
  q.hp = (pb.hp + 1) / 2;
  q.wp = (pb.wp + 1) / 2;
  q.c = 16;
  q.r = (pb.r + 1) / 2;
  q.s = (pb.s + 1) / 2;
  q.stride = 1;
  q.taps = q.r * q.s;
  q.w_stride_k = (int64_t)q.r * q.s * 16;
  q.w_stride_tap = 16;
  q.a_mode = tzcdev::A_IM2COL;
  // oh / ow / m stay the original op's: the epilogue keeps rows with oh < OH, ow < OW
  return q;
}

// Output layout, seed and fused-epilogue fields shared by both kernels.
void fill_epilogue(ConvKernelParams* pp, const Problem& pb, const Options& o, const void* seed, void* out,
                   const tzc_epilogue& ep) {
  ConvKernelParams& p = *pp;
  p.out = out;
  p.seed = seed;
  {  // byte extent of the output layout (last element + 1)
    const int eo = (ep.kind == tzcdev::EP_REQUANT_I8) ? 1 : (ep.kind == tzcdev::EP_CAST_F16) ? 2 : 4;
    const int64_t nl = pb.ngemm - 1, nb = std::max<int64_t>(1, pb.out.nb);
    p.out_bytes = ((nl / nb) * pb.out.stride_blk + (pb.m - 1) * pb.out.stride_m + nl % nb + 1) * eo;
  }
  p.out_nb = pb.out.nb;
  p.out_stride_m = pb.out.stride_m;
  p.out_stride_blk = pb.out.stride_blk;
  p.ep_kind = ep.kind;
  p.scale = ep.scale;
  {
    // vectorised epilogue: every 16-column piece of out / seed starts 16-byte aligned
    const int eo = (ep.kind == tzcdev::EP_REQUANT_I8) ? 1 : (ep.kind == tzcdev::EP_CAST_F16) ? 2 : 4;
    auto al = [](int64_t elems, int eb) { return (elems * eb) % 16 == 0; };
    bool ok = pb.ngemm % 16 == 0 && (pb.out.nb % 16 == 0) && al(pb.out.stride_m, eo) && al(pb.out.stride_blk, eo) &&
              reinterpret_cast<uintptr_t>(out) % 16 == 0;
    if (seed) ok = ok && al(pb.out.stride_m, 4) && al(pb.out.stride_blk, 4) && reinterpret_cast<uintptr_t>(seed) % 16 == 0;
    p.vec_ok = ok ? 1 : 0;
  }
  p.pow2_k = -1;
  // |seed + sum| < 2^24 is guaranteed without a seed when K*255*128 < 2^24
  // (u8 x i8 products): the requant then needs no RNE24 range check.
  p.range_check = (seed != nullptr || pb.f16 || (int64_t)pb.c * pb.taps * 255 * 128 >= (1 << 24)) ? 1 : 0;
  {
    // exact power-of-two scale 2^-k, k in [0, 126]: integer requant path
    int ex = 0;
    const float fr = std::frexp(ep.scale, &ex);  // scale = fr * 2^ex, fr in [0.5, 1)
    if (fr == 0.5f && ex - 1 <= 0 && ex - 1 >= -24) p.pow2_k = -(ex - 1);
    if (p.pow2_k >= 0) p.pow2_mul24 = 1u << (24 - p.pow2_k);
  }
  p.simple = (ep.kind == tzcdev::EP_REQUANT_I8 && p.pow2_k >= 2 && !pb.f16 && seed == nullptr && p.vec_ok &&
              pb.out.nb == pb.ngemm)
                 ? 1
                 : 0;
  p.vec32 = (p.simple && o.st256 && pb.out.stride_m % 32 == 0 && reinterpret_cast<uintptr_t>(out) % 32 == 0) ? 1 : 0;
  {
    const int eo = (ep.kind == tzcdev::EP_REQUANT_I8) ? 1 : (ep.kind == tzcdev::EP_CAST_F16) ? 2 : 4;
    auto al32 = [eo](int64_t elems) { return (elems * eo) % 32 == 0; };
    p.st32 = (o.st256 && eo > 1 && p.vec_ok && al32(pb.out.stride_m) && al32(pb.out.stride_blk) && al32(pb.out.nb) &&
              reinterpret_cast<uintptr_t>(out) % 32 == 0)
                 ? 1
                 : 0;
  }
}

// ---- launch --------------------------------------------------------------------
Status run_problem(const Problem& pb, const Options& o, const void* a, const void* b, const void* seed, void* out,
                   const tzc_epilogue& ep, cudaStream_t stream) {
  if (!device_ok()) return Status(TZC_E_DEVICE, "no usable sm_100 (B200) device");
  Status st = load_driver();
  if (!st.ok()) return st;
  {
    bool s2d = false;
    Problem q;
    WsPlan w;
    if (ws_route(pb, o, &q, &w, &s2d)) {
      if (!s2d) return run_ws(pb, w, o, a, b, seed, out, ep, stream);
      if (stem_fused_eligible(pb, o)) return run_stem_fused(pb, q, w, o, a, b, seed, out, ep, stream);
      // the stem: space-to-depth to 16-byte pixels, then the shifted-window
      // kernel in pair mode (two taps per K=32 MMA)
      void* x4 = nullptr;
      void* w4 = nullptr;
      const int eb = pb.f16 ? 2 : 1;
      st = workspace(1, (size_t)(((int64_t)q.n * q.hp * q.wp + 7) / 8 * 8) * 16 * eb, &x4, stream);
      if (st.ok()) st = workspace(2, (size_t)q.ngemm * q.taps * 16 * eb, &w4, stream);
      if (st.ok()) st = s2d_stem(pb, a, b, x4, w4, q.hp, q.wp, q.r, q.s, stream, o.s2d_one != 0);
      if (st.ok()) st = run_ws(q, w, o, x4, w4, seed, out, ep, stream);
      return st;
    }
  }
  if (needs_k7(pb)) {
    // K7: channel runs too thin for TMA (the C=3 stem).  Materialise
    // zero-padded im2col rows + weights and run them as a GEMM.
    int kp = 0;
    const Problem g = k7_gemm(pb, &kp);
    const int e = pb.f16 ? 2 : 1;
    void* wa = nullptr;
    void* wb = nullptr;
    st = workspace(1, (size_t)pb.m * kp * e, &wa, stream);
    if (st.ok()) st = workspace(2, (size_t)pb.ngemm * kp * e, &wb, stream);
    if (st.ok()) st = im2col_pad(pb, a, wa, kp, stream);
    if (st.ok()) st = weight_pad(pb, b, wb, kp, stream);
    if (!st.ok()) return st;
    st = run_problem(g, o, wa, wb, seed, out, ep, stream);
    if (st.ok()) g_last_launch.kernel = 4;  // the thin-channel GEMM rewrite
    return st;
  }
  tzc_plan plan;
  st = plan_problem(pb, o, &plan);
  if (!st.ok()) return st;
  const int e = pb.f16 ? 2 : 1;
  const int KE = plan.bk_bytes / e;
  const CUtensorMapDataType dt = pb.f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_UINT8;

  ConvKernelParams p;
  std::memset(&p, 0, sizeof(p));
#ifdef TZC_TRACE
  p.debug_flags = ::g_debug_flags;
#endif
  p.pol_a = (o.l2_hints & 1) ? tzcdev::kL2EvictFirst : 0;
  p.pol_b = (o.l2_hints & 2) ? tzcdev::kL2EvictLast : 0;
  p.producers = o.producers;
  // ---- A operand
  if (pb.a_mode == tzcdev::A_TILED) {
    cuuint64_t dims[2] = {(cuuint64_t)pb.a_kdim, (cuuint64_t)pb.a_rows};
    cuuint64_t strides[1] = {(cuuint64_t)pb.a_row_stride * e};
    cuuint32_t box[2] = {(cuuint32_t)KE, 128};
    cuuint32_t es[2] = {1, 1};
    st = enc_check(p_encode_tiled(&p.tmA, dt, 2, const_cast<void*>(a), dims, strides, box, es,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz(plan.bk_bytes),
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
                   "cuTensorMapEncodeTiled(A)");
  } else {
    cuuint64_t dims[4] = {(cuuint64_t)pb.c, (cuuint64_t)pb.wp, (cuuint64_t)pb.hp, (cuuint64_t)pb.n};
    cuuint64_t strides[3] = {(cuuint64_t)pb.c * e, (cuuint64_t)pb.wp * pb.c * e, (cuuint64_t)pb.hp * pb.wp * pb.c * e};
    int lower[2] = {0, 0};
    int upper[2] = {-(pb.s - 1), -(pb.r - 1)};
    cuuint32_t es[4] = {1, (cuuint32_t)pb.stride, (cuuint32_t)pb.stride, 1};
    st = enc_check(p_encode_im2col(&p.tmA, dt, 4, const_cast<void*>(a), dims, strides, lower, upper, (cuuint32_t)KE,
                                   128, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz(plan.bk_bytes),
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
                   "cuTensorMapEncodeIm2col(A)");
    // Driver <= 13.1 mis-encodes small im2col maps (< 128 KiB): the same
    // workaround CUTLASS applies (copy_traits_sm90_im2col.hpp).
    if (st.ok() && g_driver_version <= 13010 && (int64_t)pb.n * pb.hp * pb.wp * pb.c * e < 131072)
      reinterpret_cast<uint64_t*>(&p.tmA)[1] &= ~(1ull << 21);
  }
  if (!st.ok()) return st;
  // ---- B operand
  if (pb.b_kn) {
    cuuint64_t dims[2] = {(cuuint64_t)pb.ngemm, (cuuint64_t)pb.a_kdim};
    cuuint64_t strides[1] = {(cuuint64_t)pb.ngemm * e};
    cuuint32_t box[2] = {64, (cuuint32_t)KE};
    cuuint32_t es[2] = {1, 1};
    st = enc_check(p_encode_tiled(&p.tmB, dt, 2, const_cast<void*>(b), dims, strides, box, es,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
                   "cuTensorMapEncodeTiled(B[K,N])");
  } else {
    // dims (c, k_out, tap); stride of a unit tap dim only needs to be legal.
    const int64_t sk = pb.w_stride_k * e;
    const int64_t stap = pb.taps > 1 ? pb.w_stride_tap * e : sk * pb.ngemm;
    cuuint64_t dims[3] = {(cuuint64_t)pb.c, (cuuint64_t)pb.ngemm, (cuuint64_t)pb.taps};
    cuuint64_t strides[2] = {(cuuint64_t)sk, (cuuint64_t)stap};
    cuuint32_t box[3] = {(cuuint32_t)KE, (cuuint32_t)plan.bn, 1};
    cuuint32_t es[3] = {1, 1, 1};
    st = enc_check(p_encode_tiled(&p.tmB, dt, 3, const_cast<void*>(b), dims, strides, box, es,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz(plan.bk_bytes),
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
                   "cuTensorMapEncodeTiled(B)");
  }
  if (!st.ok()) return st;

  p.M = (int32_t)pb.m;
  p.Ngemm = pb.ngemm;
  p.c_blocks = (int32_t)(((int64_t)pb.c * e + plan.bk_bytes - 1) / plan.bk_bytes);
  p.num_kb = p.c_blocks * pb.taps;
  p.S = pb.s;
  p.OW = pb.ow;
  p.OHOW = pb.oh * pb.ow;
  p.stride = pb.stride;
  p.tiles_m = plan.tiles_m;
  p.tiles_n = plan.tiles_n;
  p.num_tiles = plan.tiles_m * plan.tiles_n;
  p.splits = plan.splits;
  {
    const WorkSplit wsplit = work_split(p.num_tiles, plan.tiles_n, p.num_kb, num_sms(), pb.ngemm % 16 == 0,
                                        pb.forced_splits ? pb.forced_splits : o.splits, o);
    p.full_units = wsplit.full;
    p.red_m0 = (int32_t)((wsplit.full / plan.tiles_n) * 128);
    p.red_rows = (int32_t)(pb.m - p.red_m0);
  }
  p.stages = plan.stages;
  p.epi_groups = epi_groups_for(p.num_kb / plan.splits, o);
  p.fd_splits = make_fdiv(plan.splits);
  p.fd_tiles_n = make_fdiv(plan.tiles_n);
  p.fd_ohow = make_fdiv(std::max<int64_t>(1, (int64_t)pb.oh * pb.ow));
  p.fd_ow = make_fdiv(std::max(1, pb.ow));
  p.fd_cblocks = make_fdiv(std::max(1, p.c_blocks));
  p.fd_s = make_fdiv(std::max(1, pb.s));
  fill_epilogue(&p, pb, o, seed, out, ep);
  // A evict-first only while the output fits L2 beside the streams: then the
  // output stays resident and the read-once activations make room for it
  // (c2_1x1_256_64 38.4 vs 45.1 us without the hint); a larger output is
  // written back during the kernel anyway and the hint only hurts
  // (c3_1x1_256_128, 103 MB out: 55.4 vs 49.3 us).  Sweep: profiles/r02c_sweep*.md
  if (o.l2_a_max_out_mb > 0 && p.out_bytes > ((int64_t)o.l2_a_max_out_mb << 20)) p.pol_a = 0;
  if (ep.kind == tzcdev::EP_REQUANT_I8 && p.full_units > 0 && p.vec_ok && pb.out.nb == pb.ngemm &&
      pb.out.stride_m == pb.ngemm && pb.ngemm % plan.bn == 0 &&
      (o.tma_store == 1 || (o.tma_store == 2 && (int64_t)p.num_kb * plan.bk_bytes <= o.tma_store_k))) {
    // int8 output as a [M, Ngemm] map; one box = 32 rows x min(BN, 128) bytes
    const int rb = std::min(plan.bn, 128);
    cuuint64_t dims[2] = {(cuuint64_t)pb.ngemm, (cuuint64_t)pb.m};
    cuuint64_t strides[1] = {(cuuint64_t)pb.out.stride_m};
    cuuint32_t box[2] = {(cuuint32_t)rb, 32};
    cuuint32_t es[2] = {1, 1};
    st = enc_check(p_encode_tiled(&p.tmO, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, out, dims, strides, box, es,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE,
                                  rb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
                   "cuTensorMapEncodeTiled(out)");
    if (!st.ok()) return st;
    p.tma_store = 1;
  }
  // without the TMA-store staging tiles the ring gets their SMEM
  if (!p.tma_store) p.stages = ring_stages(plan.bn, plan.bk_bytes, 0);
  if (o.pair && ep.kind == tzcdev::EP_REQUANT_I8 && p.vec_ok && pb.ngemm % plan.bn == 0 && !pb.f16 && !pb.b_kn &&
      plan.splits == 1 && p.full_units == p.num_tiles && p.num_kb >= o.pair_min_kb && plan.bn >= o.pair_bn &&
      (int64_t)((plan.tiles_m + 1) / 2) * plan.tiles_n >= (int64_t)o.pair_min_round * (num_sms() / 2) &&
      p.epi_groups == 1 && plan.bk_bytes == 128 && (plan.bn == 128 || plan.bn == 256) &&
      (pb.a_mode == tzcdev::A_TILED || pb.a_mode == tzcdev::A_IM2COL) && num_sms() >= 2) {
    // CTA pairs: 256-row tiles, each CTA loads its A rows and half the B rows
    const int64_t sk = pb.w_stride_k;
    const int64_t stap = pb.taps > 1 ? pb.w_stride_tap : sk * pb.ngemm;
    cuuint64_t dims[3] = {(cuuint64_t)pb.c, (cuuint64_t)pb.ngemm, (cuuint64_t)pb.taps};
    cuuint64_t strides[2] = {(cuuint64_t)sk, (cuuint64_t)stap};
    cuuint32_t box[3] = {(cuuint32_t)KE, (cuuint32_t)(plan.bn / 2), 1};
    cuuint32_t es[3] = {1, 1, 1};
    st = enc_check(p_encode_tiled(&p.tmB, dt, 3, const_cast<void*>(b), dims, strides, box, es,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz(plan.bk_bytes),
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
                   "cuTensorMapEncodeTiled(B half)");
    if (!st.ok()) return st;
    const int pairs_m = (plan.tiles_m + 1) / 2;
    p.num_tiles = pairs_m * plan.tiles_n;
    p.full_units = p.num_tiles;
    p.stages = pair_stages(plan.bn);
    const int sms = num_sms() & ~1;
    const int grid = (int)std::min<int64_t>(sms, 2 * (int64_t)p.num_tiles);
    return launch_pair_any(p, plan.bn, pb.a_mode, grid, stream);
  }
  if (plan.splits > 1) {
    p.partial_bytes = plan.workspace_bytes;
    st = workspace(0, (size_t)plan.workspace_bytes, &p.partial, stream);
    if (!st.ok()) return st;
    if (o.splitk_inkernel) {
      void* cnt = nullptr;
      st = workspace(3, (size_t)p.num_tiles * 16 * sizeof(int32_t), &cnt, stream);
      if (!st.ok()) return st;
      p.splitk_cnt = static_cast<int32_t*>(cnt);
    }
  }
  // Weight-stationary CTAs ("b_res"): when every unit of a CTA has the same
  // N tile (grid a multiple of tiles_n) and the whole B tile fits beside a
  // >= 4-deep A ring, B is loaded once per CTA instead of once per tile.
  p.b_res = 0;
  if ((o.b_res == 1 || (o.b_res == 2 && pb.taps == 1)) && plan.splits == 1 && p.full_units == p.num_tiles &&
      plan.grid % plan.tiles_n == 0 &&
      p.num_tiles >= 2 * plan.grid) {
    const int st = bres_stages(plan.bn, plan.bk_bytes, p.tma_store ? p.epi_groups : 0, p.num_kb, kStaticSmem);
    if (st) {
      p.b_res = 1;
      p.stages = st;
    }
  }
  const Entry* ent = find_entry(plan.bn, plan.bk_bytes, pb.f16, pb.a_mode, pb.b_kn);
  return ent->fn(p, plan.grid, stream);
}

}  // namespace tzcb200

#ifdef TZC_TRACE
extern "C" void tzc_debug_flags(int f) { g_debug_flags = f; }
extern "C" void tzc_trace_cta(unsigned long long* out /* [2][1024] */) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, tzcdev::g_cta_t, sizeof(unsigned long long) * 2048);
}
extern "C" void tzc_trace_dump(unsigned long long* out) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, tzcdev::g_trace, sizeof(unsigned long long) * 128);
}
#endif
