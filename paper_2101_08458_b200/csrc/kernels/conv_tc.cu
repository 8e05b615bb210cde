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
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../tzc_b200_internal.hpp"
#include "conv_tc.cuh"

namespace tzcb200 {

using tzcdev::ConvCfg;
using tzcdev::ConvKernelParams;

std::atomic<uint64_t> g_launches{0};

namespace {

PFN_cuTensorMapEncodeTiled_v12000 p_encode_tiled = nullptr;
PFN_cuTensorMapEncodeIm2col_v12000 p_encode_im2col = nullptr;
std::once_flag g_driver_once;
int g_driver_version = 0;
int g_num_sms = 0;
int g_dev_ok = -1;

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

int device_ok() {
  if (g_dev_ok >= 0) return g_dev_ok;
  int dev = 0;
  cudaDeviceProp prop;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaGetDeviceProperties(&prop, dev) != cudaSuccess) {
    cudaGetLastError();
    g_dev_ok = 0;
    return 0;
  }
  g_num_sms = prop.multiProcessorCount;
  g_dev_ok = (prop.major == 10 && prop.minor == 0) ? 1 : 0;
  return g_dev_ok;
}

int num_sms() {
  device_ok();
  return g_num_sms > 0 ? g_num_sms : 148;
}

namespace {

template <int BN, int KB, bool F16, int AM, bool BMN>
Status launch_impl(const ConvKernelParams& p, int grid, cudaStream_t stream) {
  using Cfg = ConvCfg<BN, KB>;
  auto kern = tzcdev::conv_tc_kernel<BN, KB, F16, AM, BMN>;
  static bool attr_done = false;  // per instantiation
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
    if (e != cudaSuccess) return Status(TZC_E_DEVICE, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    attr_done = true;
  }
  ConvKernelParams pk = p;
  if (p.splits > 1) pk.ep_kind = tzcdev::EP_PARTIAL;  // raw partials; fix-up applies the epilogue
  kern<<<grid, 256, Cfg::SMEM_BYTES, stream>>>(pk);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return Status(TZC_E_DEVICE, std::string("conv_tc launch: ") + cudaGetErrorString(e));
  if (p.splits > 1) {
    int64_t groups = (int64_t)p.M * (p.Ngemm / 16);
    int blocks = (int)std::min<int64_t>((groups + 255) / 256, 4 * 148);
    tzcdev::splitk_reduce_kernel<F16><<<blocks, 256, 0, stream>>>(p);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    e = cudaGetLastError();
    if (e != cudaSuccess) return Status(TZC_E_DEVICE, std::string("split-K reduce launch: ") + cudaGetErrorString(e));
  }
  return Status();
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
    TZC_E_BN(128, 1, 0, 1),
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

// Split-K workspace, cached per process (grown outside timed loops).
std::mutex g_ws_mu;
void* g_ws = nullptr;
size_t g_ws_bytes = 0;
int g_forced_splits = 0;

Status workspace(size_t bytes, void** out) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  if (bytes > g_ws_bytes) {
    if (g_ws) cudaFree(g_ws);
    g_ws = nullptr;
    g_ws_bytes = 0;
    cudaError_t e = cudaMalloc(&g_ws, bytes);
    if (e != cudaSuccess) return Status(TZC_E_DEVICE, std::string("split-K workspace: ") + cudaGetErrorString(e));
    g_ws_bytes = bytes;
  }
  *out = g_ws;
  return Status();
}

}  // namespace

void set_forced_splits(int s) { g_forced_splits = s; }

// ---- planning ----------------------------------------------------------------
Status plan_problem(const Problem& pb, tzc_plan* plan) {
  const int e = pb.f16 ? 2 : 1;
  const int64_t krow_bytes = (int64_t)pb.c * e;  // contiguous K run per tap
  int kb;
  if (krow_bytes % 128 == 0)
    kb = 128;
  else if (krow_bytes % 64 == 0)
    kb = 64;
  else
    return Status(TZC_E_INJECT, "reduction run of " + std::to_string(krow_bytes) +
                                    " bytes is not a multiple of 64 (TMA/UMMA K block); pad channels or use the layout adapter");
  if (pb.b_kn && kb != 128) return Status(TZC_E_INJECT, "fp16 [K,N] operand needs K*2 % 128 == 0");
  if (pb.ngemm % 16 != 0) return Status(TZC_E_INJECT, "output channels must be a multiple of 16");
  const int64_t M = pb.m;
  if (M <= 0 || M > INT32_MAX) return Status(TZC_E_SHAPE, "GEMM M out of range");
  int bn = pb.ngemm % 256 == 0 ? 256 : (pb.ngemm % 128 == 0 ? 128 : 64);
  if (pb.b_kn) bn = pb.ngemm % 128 == 0 ? 128 : 64;  // MN-major path instantiated for 64/128
  const int sms = num_sms();
  const int tiles_m = (int)((M + 127) / 128);
  // Prefer a narrower N tile when it fills the machine and the wide one does not.
  while (bn > 64 && (int64_t)tiles_m * ((pb.ngemm + bn - 1) / bn) < sms && !pb.b_kn) bn /= 2;
  const int tiles_n = (pb.ngemm + bn - 1) / bn;
  const int num_kb = (int)(pb.taps * (krow_bytes / kb));
  const int tiles = tiles_m * tiles_n;
  int splits = 1;
  if (g_forced_splits > 0) {
    splits = std::min(g_forced_splits, num_kb);
  } else if (tiles < sms && num_kb >= 8) {
    splits = std::min((sms + tiles - 1) / tiles, num_kb / 4);
    if (splits < 2) splits = 1;
  }
  const Entry* ent = find_entry(bn, kb, pb.f16, pb.a_mode, pb.b_kn);
  if (!ent) return Status(TZC_E_INTERNAL, "no kernel instantiation for this plan");
  plan->bm = 128;
  plan->bn = bn;
  plan->bk_bytes = kb;
  plan->stages = ent->stages;
  plan->a_mode = pb.a_mode;
  plan->splits = splits;
  plan->tiles_m = tiles_m;
  plan->tiles_n = tiles_n;
  plan->grid = std::min(tiles * splits, sms);
  plan->smem_bytes = ent->smem;
  plan->workspace_bytes = splits > 1 ? (int64_t)splits * M * pb.ngemm * 4 : 0;
  return Status();
}

// ---- launch --------------------------------------------------------------------
Status run_problem(const Problem& pb, const void* a, const void* b, const void* seed, void* out,
                   const tzc_epilogue& ep, cudaStream_t stream) {
  if (!device_ok()) return Status(TZC_E_DEVICE, "no usable sm_100 (B200) device");
  Status st = load_driver();
  if (!st.ok()) return st;
  tzc_plan plan;
  st = plan_problem(pb, &plan);
  if (!st.ok()) return st;
  const int e = pb.f16 ? 2 : 1;
  const int KE = plan.bk_bytes / e;
  const CUtensorMapDataType dt = pb.f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_UINT8;

  ConvKernelParams p;
  std::memset(&p, 0, sizeof(p));
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
  p.c_blocks = (int32_t)((int64_t)pb.c * e / plan.bk_bytes);
  p.num_kb = p.c_blocks * pb.taps;
  p.S = pb.s;
  p.OW = pb.ow;
  p.OHOW = pb.oh * pb.ow;
  p.stride = pb.stride;
  p.tiles_m = plan.tiles_m;
  p.tiles_n = plan.tiles_n;
  p.num_tiles = plan.tiles_m * plan.tiles_n;
  p.splits = plan.splits;
  p.out = out;
  p.seed = seed;
  p.out_nb = pb.out.nb;
  p.out_stride_m = pb.out.stride_m;
  p.out_stride_blk = pb.out.stride_blk;
  p.ep_kind = ep.kind;
  p.scale = ep.scale;
  if (plan.splits > 1) {
    st = workspace((size_t)plan.workspace_bytes, &p.partial);
    if (!st.ok()) return st;
  }
  const Entry* ent = find_entry(plan.bn, plan.bk_bytes, pb.f16, pb.a_mode, pb.b_kn);
  return ent->fn(p, plan.grid, stream);
}

}  // namespace tzcb200
