// tzc host library, part 4: device lowering and execution.
//
// tile_and_reorder keeps the reference's meaning (split each mapped loop by
// its instruction extent, reorder outer-dp / outer-red / pragma, emit the
// pragma; /root/reference/proj/src/rewriter.cpp:245-303) and adds what the
// sm_100a kernel needs: a KernelPlan derived from the affine index forms of
// the bound accesses (inject_intrinsic's split_linear step,
// rewriter.cpp:845-874, turned into TMA geometry).  run_tensorized plays the
// role eval_tir plays on the reference VM (vm.cpp:510-516): execute the
// tensorized body — here one tcgen05 kernel launch instead of a nest of
// interpreted intrinsic calls.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <random>
#include <sstream>

#include "../tzc_b200_internal.hpp"
#include "tzc/tzc.hpp"

namespace tzc {

// ============================ values =====================================
TensorValue TensorValue::zeros(DType t, std::vector<int64_t> shape) {
  TensorValue v;
  v.dtype = t.scalar();
  v.shape = std::move(shape);
  if (v.is_float())
    v.fdata.assign(v.size(), 0.0);
  else
    v.idata.assign(v.size(), 0);
  return v;
}
int64_t TensorValue::size() const {
  int64_t n = 1;
  for (int64_t d : shape) n *= d;
  return n;
}

// Same stream as the reference's random_tensor (vm.cpp:38-57): mt19937_64,
// integers lo + rng() % span over the full width, floats (rng()>>11)*2^-53
// rounded to the format.
TensorValue random_tensor(const TensorDecl& d, uint64_t seed) {
  TensorValue v = TensorValue::zeros(d.dtype, d.shape);
  std::mt19937_64 g(seed);
  if (v.is_float()) {
    for (auto& x : v.fdata) {
      const double u = static_cast<double>(g() >> 11) * 0x1.0p-53;
      x = d.dtype.bits == 16 ? round_f16(u) : round_f32(u);
    }
  } else {
    const uint64_t span = d.dtype.bits >= 64 ? 0 : (uint64_t{1} << d.dtype.bits);
    const int64_t lo = d.dtype.is_signed() ? -(int64_t{1} << (d.dtype.bits - 1)) : 0;
    for (auto& x : v.idata) x = lo + static_cast<int64_t>(span ? g() % span : g());
  }
  return v;
}

Inputs random_inputs(const ComputeOp& op, uint64_t seed) {
  Inputs in;
  uint64_t k = 0;
  for (const auto& t : op.tensors) {
    if (t.role == Role::Input || (t.name == op.out && op.update)) in.emplace(t.name, random_tensor(t, seed + k));
    ++k;
  }
  return in;
}

Deviation compare(const TensorValue& ref, const TensorValue& got, double rtol) {
  if (ref.dtype != got.dtype || ref.shape != got.shape) throw ShapeError("compared tensors differ in dtype or shape");
  Deviation d;
  for (int64_t i = 0; i < ref.size(); ++i) {
    const double a = ref.is_float() ? ref.fdata[i] : static_cast<double>(ref.idata[i]);
    const double b = got.is_float() ? got.fdata[i] : static_cast<double>(got.idata[i]);
    if (a != b) d.bitexact = false;
    const double rel = std::abs(a - b) / std::max(std::abs(a), 1.0);
    d.max_rel = std::max(d.max_rel, rel);
    if (rel > rtol) ++d.mismatches;
  }
  return d;
}

// ============================ planning ===================================
std::string KernelPlan::describe() const {
  std::ostringstream os;
  const char* fam = family == Family::Matmul        ? "matmul"
                    : family == Family::ConvNHWC    ? "conv_nhwc"
                    : family == Family::ConvBlocked ? "conv_blocked"
                                                    : "conv3d_blocked";
  os << fam << (f16 ? " f16" : " u8i8") << " n=" << n << " hp=" << hp << " wp=" << wp << " c=" << c << " k=" << k
     << (family == Family::ConvBlocked3D ? " dp=" + std::to_string(dp) + " kd=" + std::to_string(kd) : std::string())
     << " r=" << r << " s=" << s << " stride=" << stride << " m=" << m << (b_kn ? " b_kn" : "") << " out(nb=" << out_nb
     << ",sm=" << out_stride_m << ",sb=" << out_stride_blk << ") tile=m" << tile_m << "n" << tile_n;
  return os.str();
}

namespace {

struct Term {
  std::string var;
  int64_t coeff;
};
// Affine index as (terms, constant); InjectError when not affine.
std::pair<std::vector<Term>, int64_t> terms_of(const ExprPtr& e) {
  auto a = linearize(e);
  if (!a) throw InjectError("non-affine index '" + expr_to_string(e) + "'");
  std::vector<Term> t;
  for (const auto& [v, c] : a->coeff) t.push_back({v, c});
  return {t, a->constant};
}

int64_t ext(const ComputeOp& op, const std::string& v) { return op.find_loop(v)->extent; }

bool in(const std::vector<std::string>& s, const std::string& v) { return std::find(s.begin(), s.end(), v) != s.end(); }

// Row-major element strides of a declared tensor.
std::vector<int64_t> strides_of(const TensorDecl& t) {
  std::vector<int64_t> s(t.shape.size(), 1);
  for (int i = (int)t.shape.size() - 2; i >= 0; --i) s[i] = s[i + 1] * t.shape[i + 1];
  return s;
}

KernelPlan plan_for(const ComputeOp& op, const Intrinsic& intr, const LoopMapping& map, const BindMap& bind) {
  // registers: first two inputs of the instruction semantics are the A (M x K)
  // and B operands, the output is D
  std::vector<std::string> regs;
  for (const auto& t : intr.semantics.tensors)
    if (t.role == Role::Input) regs.push_back(t.name);
  if (regs.size() != 2 || intr.semantics.loops.size() != 3)
    throw InjectError("instruction '" + intr.name + "' is not a tcgen05 matrix description");
  const std::string& mn = intr.target_mnemonic;
  if (mn.rfind("tcgen05.mma", 0) != 0) throw InjectError("instruction '" + intr.name + "' has no sm_100a kernel (mnemonic '" + mn + "')");
  auto bound = [&](const std::string& r) {
    auto it = bind.reg_to_op.find(r);
    if (it == bind.reg_to_op.end() || it->second->kind != Expr::Kind::Load)
      throw InjectError("register '" + r + "' is not bound to a tensor access");
    return it->second;
  };
  const ExprPtr A = bound(regs[0]), B = bound(regs[1]);
  const auto& il = intr.semantics.loops;  // m (dp), n (dp), k (red)
  std::vector<std::string> Mv, Nv;
  std::string Kv;
  for (const auto& [o, i] : map.f) {
    std::vector<std::string>* grp = i == il[0].name ? &Mv : i == il[1].name ? &Nv : nullptr;
    if (grp) {
      auto f = map.fused.find(i);
      if (f != map.fused.end()) grp->insert(grp->end(), f->second.begin(), f->second.end());
      grp->push_back(o);
    } else {
      Kv = o;
    }
  }
  std::vector<std::string> taps;  // reduction loops other than the channel loop
  for (const auto& l : op.loops)
    if (l.kind == LoopKind::Reduction && l.name != Kv) taps.push_back(l.name);
  std::vector<std::string> unmapped_dp;
  for (const auto& l : op.loops)
    if (l.kind == LoopKind::DataParallel && !in(Mv, l.name) && !in(Nv, l.name)) unmapped_dp.push_back(l.name);
  if (!unmapped_dp.empty()) throw InjectError("data-parallel loop '" + unmapped_dp[0] + "' is not covered by the M/N tiles");

  KernelPlan p;
  p.f16 = mn.find("kind::f16") != std::string::npos;
  p.tile_m = il[0].extent;
  p.tile_n = il[1].extent;
  p.data = A->name;
  p.weight = B->name;
  p.out = op.out;
  const TensorDecl& td = *op.find_tensor(A->name);
  const TensorDecl& tw = *op.find_tensor(B->name);
  const TensorDecl& to = op.output();
  if ((p.f16 && (td.dtype != kF16 || tw.dtype != kF16)) || (!p.f16 && (td.dtype != kU8 || tw.dtype != kI8)))
    throw InjectError("operand dtypes do not match the instruction kind");

  // ---- output: every index a single dp loop with unit coefficient
  std::vector<std::string> odims;
  for (const auto& e : op.indices) {
    auto [t, c] = terms_of(e);
    if (t.size() != 1 || t[0].coeff != 1 || c != 0) throw InjectError("output index '" + expr_to_string(e) + "' is not a plain loop");
    odims.push_back(t[0].var);
  }
  const std::vector<int64_t> ost = strides_of(to);
  auto ostride = [&](const std::string& v) {
    for (size_t i = 0; i < odims.size(); ++i)
      if (odims[i] == v) return ost[i];
    throw InjectError("loop '" + v + "' does not index the output");
  };
  // M group: the pixel index p = fused (Mv...) must address the output linearly
  int64_t Mext = 1;
  for (const auto& v : Mv) Mext *= ext(op, v);
  int64_t sm = ostride(Mv.back());
  for (int i = (int)Mv.size() - 1; i > 0; --i)
    if (ostride(Mv[i - 1]) != ostride(Mv[i]) * ext(op, Mv[i])) throw InjectError("fused pixel axis is not linear in the output");
  // N group: (outer block, inner lanes) or a single loop with unit stride
  if (Nv.empty() || Nv.size() > 2) throw InjectError("unsupported output-channel structure");
  const std::string nin = Nv.back();
  if (ostride(nin) != 1) throw InjectError("output channels must be innermost");
  p.k = 1;
  for (const auto& v : Nv) p.k *= ext(op, v);
  p.out_stride_m = sm;
  if (Nv.size() == 2) {
    p.out_nb = ext(op, nin);
    p.out_stride_blk = ostride(Nv[0]);
  } else {
    p.out_nb = p.k;
    p.out_stride_blk = 0;
  }

  // ---- data (A operand)
  std::vector<std::pair<std::vector<Term>, int64_t>> dd;
  for (const auto& e : A->args) dd.push_back(terms_of(e));
  for (const auto& [t, c] : dd)
    if (c != 0) throw InjectError("constant offsets in operand indices are not supported");
  auto single = [&](size_t i) { return dd[i].first.size() == 1 ? dd[i].first[0] : Term{"", 0}; };
  const size_t nd = dd.size();
  const Term last = single(nd - 1);
  const bool blocked = Nv.size() == 2;
  if (!blocked) {
    if (last.var != Kv || last.coeff != 1) throw InjectError("the reduction channel must be the innermost, contiguous operand dimension");
    p.c = ext(op, Kv);
    if (td.shape.back() != p.c) throw InjectError("partial channel range");
  }
  // GEMM-like: all leading dims are plain M loops in output order with full extents
  bool gemm_like = !blocked && taps.empty();
  if (gemm_like) {
    std::vector<std::string> lead;
    for (size_t i = 0; i + 1 < nd; ++i) {
      const Term t = single(i);
      if (t.var.empty() || t.coeff != 1 || !in(Mv, t.var) || td.shape[i] != ext(op, t.var)) {
        gemm_like = false;
        break;
      }
      lead.push_back(t.var);
    }
    if (gemm_like && lead != Mv) gemm_like = false;
  }
  if (gemm_like) {
    // matmul / 1x1 unit-stride conv: A rows = fused pixels
    p.family = nd == 2 && Mv.size() == 1 ? KernelPlan::Family::Matmul : KernelPlan::Family::ConvNHWC;
    p.n = 1;
    p.hp = 1;
    p.wp = Mext;
    p.m = Mext;
    p.r = p.s = p.stride = 1;
    // B: [N..., K] (K-major) or fp16 [K, N] (MN-major)
    std::vector<std::string> wd;
    for (const auto& e : B->args) {
      auto [t, c] = terms_of(e);
      if (t.size() != 1 || t[0].coeff != 1 || c != 0) throw InjectError("weight index is not a plain loop");
      wd.push_back(t[0].var);
    }
    const std::vector<int64_t> wst = strides_of(tw);
    if (Nv.size() != 1) throw InjectError("unsupported weight structure");
    if (wd.size() == 2 && wd[0] == Nv[0] && wd[1] == Kv) {
      p.w_stride_k = wst[0];
      p.w_stride_tap = wst[0];
    } else if (wd.size() == 2 && wd[0] == Kv && wd[1] == Nv[0] && p.f16) {
      p.b_kn = true;
    } else {
      throw InjectError("weight layout has no kernel (need [N,K], or [K,N] for fp16)");
    }
    if (tw.shape[wd[0] == Kv ? 0 : 1] != p.c || tw.shape[wd[0] == Kv ? 1 : 0] != p.k)
      throw InjectError("partial weight range");
    if (p.family == KernelPlan::Family::ConvNHWC) {
      p.n = 1;
      p.hp = 1;
      p.wp = Mext;
    }
    return p;
  }

  // ---- convolution: [batch?] [h*st + r] [w*st + s] [channel]
  int di = 0;
  std::string vb, vh, vw, vr, vs;
  int64_t sth = 1, stw = 1;
  if (nd == 4 || (blocked && nd == 4)) {
    if (!blocked) {
      const Term t = single(0);
      if (t.var.empty() || t.coeff != 1 || !in(Mv, t.var)) throw InjectError("unsupported batch dimension");
      vb = t.var;
    }
    di = 1;
  } else if (nd != 3 && !(blocked && nd == 5)) {
    throw InjectError("unsupported operand rank for a convolution");
  }
  auto spatial = [&](size_t i, std::string* vm, std::string* vt, int64_t* st) {
    for (const auto& t : dd[i].first) {
      if (in(Mv, t.var)) {
        *vm = t.var;
        *st = t.coeff;
      } else if (in(taps, t.var) && t.coeff == 1) {
        *vt = t.var;
      } else {
        throw InjectError("unsupported spatial index '" + expr_to_string(A->args[i]) + "'");
      }
    }
    if (vm->empty()) throw InjectError("spatial index without an output-pixel loop");
  };
  auto weight_dims = [&]() {
    std::vector<std::string> wd;
    for (const auto& e : B->args) {
      auto [t, c] = terms_of(e);
      if (t.size() != 1 || t[0].coeff != 1 || c != 0) throw InjectError("weight index is not a plain loop");
      wd.push_back(t[0].var);
    }
    return wd;
  };
  if (nd == 5) {
    // conv3d_tdsl (proj/src/workloads.cpp:94-121): data[co, d*st+rd, h*st+rh, w*st+rw, ci],
    // kernel[ko, co, rd, rh, rw, ki, ci], out[ko, od, oh, ow, ki].  Executed as kd
    // batched 2-D convs (one per depth tap) over the od output depth slices,
    // accumulated through the int32 / fp32 C-seed (run_tensorized_packed).
    std::string vd, vrd, vh3, vr3, vw3, vs3;
    int64_t sd = 1, sh = 1, sw = 1;
    spatial(1, &vd, &vrd, &sd);
    spatial(2, &vh3, &vr3, &sh);
    spatial(3, &vw3, &vs3, &sw);
    if (sd != sh || sh != sw) throw InjectError("anisotropic strides are not supported");
    if (Mv != std::vector<std::string>{vd, vh3, vw3}) throw InjectError("pixel loops must be fused in (od, oh, ow) order");
    const Term tco = single(0), tci = single(4);
    if (tco.var.empty() || tci.var != Kv || !in(taps, tco.var)) throw InjectError("blocked data must be [co, d, h, w, ci]");
    const std::vector<std::string> wd = weight_dims();
    if (vrd.empty() || vr3.empty() || vs3.empty() || wd.size() != 7 || wd[0] != Nv[0] || wd[1] != tco.var ||
        wd[2] != vrd || wd[3] != vr3 || wd[4] != vs3 || wd[5] != Nv[1] || wd[6] != Kv)
      throw InjectError("blocked 3-D kernel must be [ko, co, rd, rh, rw, ki, ci]");
    p.family = KernelPlan::Family::ConvBlocked3D;
    p.stride = sd;
    p.kd = ext(op, vrd);
    p.r = ext(op, vr3);
    p.s = ext(op, vs3);
    p.dp = td.shape[1];
    p.hp = td.shape[2];
    p.wp = td.shape[3];
    p.od = ext(op, vd);
    if ((p.dp - p.kd) / p.stride + 1 != p.od || (p.hp - p.r) / p.stride + 1 != ext(op, vh3) ||
        (p.wp - p.s) / p.stride + 1 != ext(op, vw3))
      throw InjectError("output window does not cover the input exactly");
    p.n = p.od;
    p.m = p.od * ext(op, vh3) * ext(op, vw3);
    p.cb = ext(op, Kv);
    p.kb = ext(op, Nv[1]);
    p.c = ext(op, tco.var) * p.cb;
    p.w_stride_k = p.kd * p.r * p.s * p.c;  // after the K5 adapter: [K, kd, R, S, C]
    p.w_stride_tap = p.c;
    return p;
  }
  spatial(di, &vh, &vr, &sth);
  spatial(di + 1, &vw, &vs, &stw);
  if (sth != stw) throw InjectError("anisotropic strides are not supported");
  p.stride = sth;
  p.r = vr.empty() ? 1 : ext(op, vr);
  p.s = vs.empty() ? 1 : ext(op, vs);
  p.hp = td.shape[di];
  p.wp = td.shape[di + 1];
  p.n = vb.empty() ? 1 : ext(op, vb);
  const int64_t oh = ext(op, vh), ow = ext(op, vw);
  if ((p.hp - p.r) / p.stride + 1 != oh || (p.wp - p.s) / p.stride + 1 != ow)
    throw InjectError("output window does not cover the (pre-padded) input exactly");
  std::vector<std::string> want_m;
  if (!vb.empty()) want_m.push_back(vb);
  want_m.push_back(vh);
  want_m.push_back(vw);
  if (want_m != Mv) throw InjectError("pixel loops must be fused in (n, oh, ow) order");
  p.m = p.n * oh * ow;
  for (const auto& t : taps)
    if (t != vr && t != vs && !(blocked && single(0).var == t)) throw InjectError("reduction loop '" + t + "' has no kernel role");

  std::vector<std::string> wd;
  for (const auto& e : B->args) {
    auto [t, c] = terms_of(e);
    if (t.size() != 1 || t[0].coeff != 1 || c != 0) throw InjectError("weight index is not a plain loop");
    wd.push_back(t[0].var);
  }
  const std::vector<int64_t> wst = strides_of(tw);
  auto wpos = [&](const std::string& v) -> int {
    for (size_t i = 0; i < wd.size(); ++i)
      if (wd[i] == v) return (int)i;
    return -1;
  };
  if (!blocked) {
    p.family = KernelPlan::Family::ConvNHWC;
    // weights: element (k, r, s, c) at k*wsk + (r*S+s)*wst + c, c contiguous
    if (wd.back() != Kv) throw InjectError("weight channel must be innermost");
    const int pk = wpos(Nv[0]), pr = vr.empty() ? -1 : wpos(vr), ps = vs.empty() ? -1 : wpos(vs);
    if (pk < 0 || (!vr.empty() && pr < 0) || (!vs.empty() && ps < 0) || (int)wd.size() != 2 + (pr >= 0) + (ps >= 0))
      throw InjectError("weight indices do not match the convolution loops");
    p.w_stride_k = wst[pk];
    const int64_t rs = pr >= 0 ? wst[pr] : (ps >= 0 ? wst[ps] * p.s : p.c);
    const int64_t ss = ps >= 0 ? wst[ps] : p.c;
    if (rs != ss * p.s) throw InjectError("filter taps are not laid out as (r, s) rows");
    p.w_stride_tap = ss;
    return p;
  }
  // conv2d_tdsl channel-blocked family: data[co, h, w, ci], kernel[ko, co, r, s, ki, ci], out[ko, oh, ow, ki]
  p.family = KernelPlan::Family::ConvBlocked;
  const Term tco = single(0), tci = single(3);
  if (tco.var.empty() || tci.var.empty() || !in(taps, tco.var) || tci.var != Kv)
    throw InjectError("blocked data must be [co, h, w, ci]");
  if (wd.size() != 6 || wd[0] != Nv[0] || wd[1] != tco.var || wd[2] != vr || wd[3] != vs || wd[4] != Nv[1] || wd[5] != Kv)
    throw InjectError("blocked kernel must be [ko, co, r, s, ki, ci]");
  p.cb = ext(op, Kv);
  p.kb = ext(op, Nv[1]);
  p.c = ext(op, tco.var) * p.cb;
  p.w_stride_k = (int64_t)p.r * p.s * p.c;  // after the K5 adapter: [K, R, S, C]
  p.w_stride_tap = p.c;
  return p;
}

}  // namespace

static bool is_tcgen05(const Intrinsic& intr) { return intr.target_mnemonic.rfind("tcgen05.", 0) == 0; }

// The reference's tensorize tiling (proj/include/tzc/rewriter.hpp:56-69):
// pads (if allowed), one split per mapped loop by its instruction extent,
// then a reorder putting the outer pieces (declaration order, data-parallel
// before reduction) above the inner pieces (instruction loop order), which
// the pragma tags.  Backend additions: a fused pixel group (F6) is fused
// into one axis before its split; for tcgen05 instructions a non-dividing
// extent is not padded in the op but clipped on the device (TMA
// out-of-bounds zero fill / masked stores), and the kernel plan is derived.
TensorizedOp tile_and_reorder(const ComputeOp& op, const Intrinsic& intr, const LoopMapping& mapping, bool allow_pad) {
  const bool device = is_tcgen05(intr);
  TensorizedOp t;
  t.original = op;
  t.mapping = mapping;
  ComputeOp cur = op;
  // the fused group (outermost first) ending in each mapped op loop
  auto group_of = [&](const std::string& o, const std::string& i) {
    std::vector<std::string> g;
    auto f = mapping.fused.find(i);
    if (f != mapping.fused.end()) g = f->second;
    g.push_back(o);
    return g;
  };
  for (const auto& [o, i] : mapping.f) {
    const LoopVar* il = intr.semantics.find_loop(i);
    const LoopVar* ol = op.find_loop(o);
    if (!il || !ol) throw ScheduleError("mapping names an unknown loop (" + o + " -> " + i + ")");
    int64_t extent = 1;
    for (const auto& g : group_of(o, i)) extent *= op.find_loop(g)->extent;
    if (extent % il->extent == 0) continue;
    if (!allow_pad)
      throw DivisibilityError("loop '" + o + "' covers " + std::to_string(extent) + " iterations, not a multiple of " +
                              intr.name + "'s '" + i + "' extent " + std::to_string(il->extent) +
                              " (allow padding to proceed)");
    if (device || group_of(o, i).size() > 1) continue;  // the device clips the tail
    Transform pad;
    pad.kind = Transform::Kind::Pad;
    pad.a = o;
    pad.factor = il->extent;
    t.schedule.push_back(pad);
    cur = pad_to_multiple(cur, o, il->extent);
  }
  // fused groups: members must be adjacent (declaration order), so reorder
  // them together first when the op declares them apart (conv2d_tdsl's ko..ki)
  std::map<std::string, std::string> axis_of;  // op loop -> the axis it becomes before the split
  std::vector<std::string> order;
  bool moved = false;
  {
    std::set<std::string> placed;
    for (const auto& l : cur.loops) {
      if (placed.count(l.name)) continue;
      std::vector<std::string> grp{l.name};
      for (const auto& [o, i] : mapping.f) {
        const auto g = group_of(o, i);
        if (g.size() > 1 && std::count(g.begin(), g.end(), l.name)) grp = g;
      }
      for (const auto& g : grp) {
        moved = moved || order.size() >= cur.loops.size() || cur.loops[order.size()].name != g;
        order.push_back(g);
        placed.insert(g);
      }
    }
  }
  if (moved) {
    Transform ro;
    ro.kind = Transform::Kind::Reorder;
    ro.names = order;
    t.schedule.push_back(ro);
  }
  for (const auto& [o, i] : mapping.f) {
    const auto g = group_of(o, i);
    std::string axis = g.back();
    for (size_t k = g.size() - 1; k-- > 0;) {  // fuse outward: (oh, ow) -> oh.ow.fused, then (n, ...)
      Transform fu;
      fu.kind = Transform::Kind::Fuse;
      fu.a = g[k];
      fu.b = axis;
      t.schedule.push_back(fu);
      axis = g[k] + "." + axis + ".fused";
    }
    for (const auto& x : g) axis_of[x] = axis;
    Transform sp;
    sp.kind = Transform::Kind::Split;
    sp.a = axis;
    sp.factor = intr.semantics.find_loop(i)->extent;
    t.schedule.push_back(sp);
    t.pragma_axes.push_back(axis + ".i");
  }
  {
    std::set<std::string> done;
    for (const auto& name : order) {
      const LoopVar* l = cur.find_loop(name);
      auto it = axis_of.find(name);
      const std::string n = it == axis_of.end() ? name : it->second + ".o";
      if (!done.insert(n).second) continue;  // a fused group's axis appears once
      (l->kind == LoopKind::DataParallel ? t.outer_dp : t.outer_red).push_back(n);
    }
  }
  Transform ro;
  ro.kind = Transform::Kind::Reorder;
  ro.names = t.outer_dp;
  ro.names.insert(ro.names.end(), t.outer_red.begin(), t.outer_red.end());
  ro.names.insert(ro.names.end(), t.pragma_axes.begin(), t.pragma_axes.end());
  t.schedule.push_back(ro);
  Transform pg;
  pg.kind = Transform::Kind::Pragma;
  pg.names = t.pragma_axes;
  t.schedule.push_back(pg);
  t.op = std::move(cur);
  if (device) {
    MatchResult mr = match_operation(op, intr);
    if (!mr.ok) throw InjectError("no structural match: " + mr.reason);
    t.plan = plan_for(op, intr, mapping, mr.bind);
    t.has_plan = true;
  }
  return t;
}

TensorizedOp tensorize(const ComputeOp& op, const Intrinsic& intr) {
  MatchResult mr = match_operation(op, intr);
  if (!mr.ok) throw InjectError("no structural match: " + mr.reason);
  if (!is_tcgen05(intr))
    throw NoFeasibleMapping("no mapping of '" + intr.name + "' has an sm_100a kernel (mnemonic '" +
                            intr.target_mnemonic + "'; this backend executes tcgen05 descriptions)");
  std::string last;
  for (const auto& m : enumerate_group_mappings(op, intr, mr.bind)) {
    try {
      return tile_and_reorder(op, intr, m, true);
    } catch (const InjectError& e) {
      last = e.what();
    }
  }
  throw NoFeasibleMapping("no mapping of '" + intr.name + "' has an sm_100a kernel" + (last.empty() ? "" : " (" + last + ")"));
}

// ============================ execution ==================================
namespace {

// Per host thread: device staging buffers and streams, so concurrent
// run_op calls from different threads (independent ops) overlap their
// copies and kernels instead of serialising on one buffer set.
struct DeviceBuf {
  void* p = nullptr;
  size_t bytes = 0;
};
thread_local DeviceBuf t_pool[9];

void* pool(int slot, size_t bytes) {
  DeviceBuf& b = t_pool[slot];
  if (bytes > b.bytes) {
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    if (cudaMalloc(&b.p, bytes) != cudaSuccess) {
      cudaGetLastError();
      throw DeviceError("device allocation of " + std::to_string(bytes) + " bytes failed");
    }
    b.bytes = bytes;
  }
  return b.p;
}

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

int elem_bytes(const DType& t) { return t.bits / 8; }

struct Epi {
  int kind = TZC_EP_I32;
  float scale = 1.0f;
  DType out_dtype;
};

// The reference-expressible epilogues:
//   Q[i..] = cast<i8>(cast<fp32>(C[i..]) * s)      H[i..] = cast<fp16>(C[i..])
Epi epilogue_of(const ComputeOp& main, const ComputeOp* ep) {
  Epi r;
  r.kind = main.output().dtype.is_float() ? TZC_EP_F32 : TZC_EP_I32;
  r.out_dtype = main.output().dtype;
  if (!ep) return r;
  const ComputeOp e = infer_types(*ep);
  const TensorDecl* src = e.find_tensor(main.out);
  if (!src || src->role != Role::Input || src->shape != main.output().shape || src->dtype != main.output().dtype)
    throw InjectError("epilogue op must read the main op's output '" + main.out + "' with its shape and dtype");
  if (e.output().shape != main.output().shape || e.update || !e.loops_of_kind(LoopKind::Reduction).empty())
    throw InjectError("epilogue op must be an elementwise map of the output");
  // the loaded index must be the store index
  const ExprPtr& v = e.value;
  auto is_src = [&](const ExprPtr& x) {
    if (x->kind != Expr::Kind::Load || x->name != main.out || x->args.size() != e.indices.size()) return false;
    for (size_t i = 0; i < e.indices.size(); ++i)
      if (!expr_equal(x->args[i], e.indices[i], false)) return false;
    return true;
  };
  r.out_dtype = e.output().dtype;
  if (e.output().dtype == kI8 && v->kind == Expr::Kind::Cast && v->args[0]->kind == Expr::Kind::Mul) {
    const ExprPtr& m = v->args[0];
    const ExprPtr& a = m->args[0];
    const ExprPtr& s = m->args[1];
    if (m->dtype == kF32 && a->kind == Expr::Kind::Cast && a->dtype == kF32 && is_src(a->args[0]) &&
        s->kind == Expr::Kind::FloatImm && s->dtype == kF32 && !main.output().dtype.is_float()) {
      r.kind = TZC_EP_REQUANT_I8;
      r.scale = static_cast<float>(round_f32(s->fval));
      return r;
    }
  }
  if (e.output().dtype == kF16 && v->kind == Expr::Kind::Cast && is_src(v->args[0]) && main.output().dtype == kF32) {
    r.kind = TZC_EP_CAST_F16;
    return r;
  }
  throw InjectError("epilogue op is neither cast<i8>(cast<fp32>(C) * s) nor cast<fp16>(C)");
}

}  // namespace

// The instruction's tile binds the launch: N = the instruction's N when it
// divides the output channels (the printed TensorIR's 64-wide calls run as
// 64-wide N tiles), M = 256 (cta_group::2) selects the CTA-pair kernel.
tzcb200::Options instruction_options(const KernelPlan& p, tzcb200::Options o) {
  const bool flat = p.family == KernelPlan::Family::Matmul || p.family == KernelPlan::Family::ConvNHWC;
  if (flat && p.tile_n > 0 && p.k % p.tile_n == 0 && (p.tile_n == 64 || p.tile_n == 128 || p.tile_n == 256))
    o.bn = (int)p.tile_n;
  if (p.tile_m == 256) {
    o.pair = 1;
    o.pair_min_kb = 0;
    o.pair_bn = 0;
    o.pair_min_round = 0;
    o.shifted_window = 0;
  } else {
    o.pair = 0;  // an M = 128 description is a cta_group::1 MMA
  }
  return o;
}

void run_tensorized_packed(const TensorizedOp& t, const std::map<std::string, const void*>& host, void* host_out,
                           int64_t out_bytes, const ComputeOp* epilogue_op) {
  using namespace tzcb200;
  if (!t.has_plan)
    throw InjectError("no sm_100a kernel for this tensorized op (only tcgen05 descriptions execute on the B200)");
  const KernelPlan& p = t.plan;
  const ComputeOp& op = t.op;
  const Epi ep = epilogue_of(op, epilogue_op);
  const TensorDecl& td = *op.find_tensor(p.data);
  const TensorDecl& tw = *op.find_tensor(p.weight);
  const TensorDecl& to = op.output();
  if (out_bytes != to.size() * elem_bytes(ep.out_dtype))
    throw ShapeError("output buffer holds " + std::to_string(out_bytes) + " bytes, need " +
                     std::to_string(to.size() * elem_bytes(ep.out_dtype)));
  auto need = [&](const std::string& n) {
    auto it = host.find(n);
    if (it == host.end() || !it->second) throw MissingInput("missing input tensor '" + n + "'");
    return it->second;
  };
  const void* hx = need(p.data);
  const void* hw = need(p.weight);
  const void* hs = nullptr;
  if (op.update) {
    auto it = host.find(op.out);
    hs = it == host.end() ? nullptr : it->second;  // absent initial image => zeros
  }
  const size_t xb = td.size() * elem_bytes(td.dtype), wb = tw.size() * elem_bytes(tw.dtype);
  const size_t sb = to.size() * elem_bytes(to.dtype);
  void* dx = pool(0, xb);
  void* dw = pool(1, wb);
  void* ds = hs ? pool(2, sb) : nullptr;
  void* dout = pool(3, (size_t)out_bytes);
  tzc_out_layout ol{};
  ol.nb = (int32_t)p.out_nb;
  ol.stride_m = p.out_stride_m;
  ol.stride_blk = p.out_stride_blk;
  const tzc_epilogue e{ep.kind, ep.scale};
  const Options opts = instruction_options(p, options_for(""));  // one plan-option snapshot for every launch of this call
  auto fail = [](const Status& s) {
    if (s.code == TZC_E_DEVICE) throw DeviceError(s.msg);
    throw InjectError(s.msg);
  };
  // Problem of `rows` leading units (images for a conv, rows for a GEMM)
  auto problem = [&](int64_t rows) {
    Problem pb;
    Status s;
    if (p.family == KernelPlan::Family::Matmul) {
      tzc_gemm_desc g{};
      g.profile = p.f16 ? TZC_PROFILE_F16 : TZC_PROFILE_U8I8;
      g.m = (int32_t)rows;
      g.n = (int32_t)p.k;
      g.k = (int32_t)p.c;
      g.b_kn = p.b_kn ? 1 : 0;
      g.out = ol;
      s = problem_from_gemm(g, &pb);
    } else {
      tzc_conv_desc c{};
      c.profile = p.f16 ? TZC_PROFILE_F16 : TZC_PROFILE_U8I8;
      c.n = (int32_t)rows;
      c.hp = (int32_t)p.hp;
      c.wp = (int32_t)p.wp;
      c.c = (int32_t)p.c;
      c.k = (int32_t)p.k;
      c.r = (int32_t)p.r;
      c.s = (int32_t)p.s;
      c.stride = (int32_t)p.stride;
      c.w_stride_k = p.w_stride_k;
      c.w_stride_tap = p.w_stride_tap;
      c.out = ol;
      s = problem_from_conv(c, &pb);
    }
    if (!s.ok()) throw InjectError(s.msg);
    pb.forced_splits = (int)p.splits;
    return pb;
  };

  // Batched NHWC conv / row-major GEMM with a dense output: the leading unit
  // (image / row block) is outermost in data, accumulator image and output,
  // so the op splits into independent chunks.  Chunk i's H2D, kernel and D2H
  // go on stream i % 3: the H2D of chunk i+1 and the D2H of chunk i-1 run on
  // the two copy engines while chunk i computes, and the op costs about
  // max(H2D, D2H) instead of H2D + kernel + D2H.
  const bool conv = p.family == KernelPlan::Family::ConvNHWC;
  const int64_t units = p.family == KernelPlan::Family::Matmul ? p.m : (conv ? p.n : 1);
  const bool dense_out = ol.nb == (int32_t)p.k && ol.stride_m == p.k;
  const int64_t per_unit_x = p.family == KernelPlan::Family::Matmul ? p.c : p.hp * p.wp * p.c;
  const int64_t oh = (p.hp - p.r) / p.stride + 1, ow = (p.wp - p.s) / p.stride + 1;
  const int64_t per_unit_o = p.family == KernelPlan::Family::Matmul ? p.k : oh * ow * p.k;
  int64_t chunk = units;
  if ((conv || p.family == KernelPlan::Family::Matmul) && dense_out && units >= 2) {
    const int64_t target = p.family == KernelPlan::Family::Matmul ? 8 : std::min<int64_t>(8, units);
    chunk = (units + target - 1) / target;
    if (p.family == KernelPlan::Family::Matmul) chunk = std::max<int64_t>(128, (chunk + 127) / 128 * 128);
  }
  if (chunk < units) {
    thread_local cudaStream_t S[3] = {nullptr, nullptr, nullptr};
    thread_local cudaEvent_t ev_w = nullptr;
    if (!S[0]) {
      for (auto& x : S) cuda_ok(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking), "stream");
      cuda_ok(cudaEventCreateWithFlags(&ev_w, cudaEventDisableTiming), "event");
    }
    const int eb_x = elem_bytes(td.dtype), eb_s = elem_bytes(to.dtype), eb_o = elem_bytes(ep.out_dtype);
    cuda_ok(cudaMemcpyAsync(dw, hw, wb, cudaMemcpyHostToDevice, S[0]), "H2D weight");
    cuda_ok(cudaEventRecord(ev_w, S[0]), "event");
    int i = 0;
    for (int64_t u0 = 0; u0 < units; u0 += chunk, ++i) {
      const int64_t nu = std::min(chunk, units - u0);
      cudaStream_t st = S[i % 3];
      cuda_ok(cudaStreamWaitEvent(st, ev_w, 0), "wait weights");
      uint8_t* cx = static_cast<uint8_t*>(dx) + u0 * per_unit_x * eb_x;
      cuda_ok(cudaMemcpyAsync(cx, static_cast<const uint8_t*>(hx) + u0 * per_unit_x * eb_x, nu * per_unit_x * eb_x,
                              cudaMemcpyHostToDevice, st),
              "H2D data");
      uint8_t* cs = nullptr;
      if (hs) {
        cs = static_cast<uint8_t*>(ds) + u0 * per_unit_o * eb_s;
        cuda_ok(cudaMemcpyAsync(cs, static_cast<const uint8_t*>(hs) + u0 * per_unit_o * eb_s, nu * per_unit_o * eb_s,
                                cudaMemcpyHostToDevice, st),
                "H2D accumulator image");
      }
      uint8_t* co = static_cast<uint8_t*>(dout) + u0 * per_unit_o * eb_o;
      const Status s = run_problem(problem(nu), opts, cx, dw, cs, co, e, st);
      if (!s.ok()) fail(s);
      cuda_ok(cudaMemcpyAsync(static_cast<uint8_t*>(host_out) + u0 * per_unit_o * eb_o, co, nu * per_unit_o * eb_o,
                              cudaMemcpyDeviceToHost, st),
              "D2H output");
    }
    for (auto& x : S) cuda_ok(cudaStreamSynchronize(x), "tensorized op");
    return;
  }

  thread_local cudaStream_t st = nullptr;  // non-blocking: no implicit sync with other threads' streams
  if (!st) cuda_ok(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
  cuda_ok(cudaMemcpyAsync(dx, hx, xb, cudaMemcpyHostToDevice, st), "H2D data");
  cuda_ok(cudaMemcpyAsync(dw, hw, wb, cudaMemcpyHostToDevice, st), "H2D weight");
  if (hs) cuda_ok(cudaMemcpyAsync(ds, hs, sb, cudaMemcpyHostToDevice, st), "H2D accumulator image");
  const void* a = dx;
  const void* b = dw;
  if (p.family == KernelPlan::Family::ConvBlocked) {
    // K5: channel-blocked data / kernel -> NHWC / [K,R,S,C]
    const int eb = p.f16 ? 2 : 1;
    void* ux = pool(4, xb);
    void* uw = pool(5, wb);
    Status s1 = unblock_data(dx, ux, (int)p.c, (int)p.hp, (int)p.wp, (int)p.cb, eb, st);
    if (!s1.ok()) throw DeviceError(s1.msg);
    s1 = unblock_kernel(dw, uw, (int)p.k, (int)p.c, (int)p.r, (int)p.s, (int)p.kb, (int)p.cb, eb, st);
    if (!s1.ok()) throw DeviceError(s1.msg);
    a = ux;
    b = uw;
  }
  if (p.family == KernelPlan::Family::ConvBlocked3D) {
    // one batched 2-D conv per depth tap rd over the od output slices (input
    // slices rd, rd+st, ...), chained through the C-seed: ping-pong int32 /
    // fp32 accumulators, the caller's epilogue on the last tap only.  The sum
    // order per element is rd-major, exact for integers (wrap-add, F8).
    const int eb = p.f16 ? 2 : 1;
    void* ux = pool(4, xb);
    void* uw = pool(5, wb);
    Status s1 = unblock_data(dx, ux, (int)p.c, (int)(p.dp * p.hp), (int)p.wp, (int)p.cb, eb, st);
    if (!s1.ok()) throw DeviceError(s1.msg);
    s1 = unblock_kernel(dw, uw, (int)p.k, (int)p.c, (int)(p.kd * p.r), (int)p.s, (int)p.kb, (int)p.cb, eb, st);
    if (!s1.ok()) throw DeviceError(s1.msg);
    const size_t slice = (size_t)(p.hp * p.wp * p.c) * eb;
    const size_t acc_bytes = (size_t)to.size() * 4;
    void* acc[2] = {pool(6, acc_bytes), pool(7, acc_bytes)};
    void* gathered = p.stride > 1 ? pool(8, slice * p.od) : nullptr;
    const tzc_epilogue mid{p.f16 ? TZC_EP_F32 : TZC_EP_I32, 1.0f};
    const void* seed = ds;
    for (int64_t rd = 0; rd < p.kd; ++rd) {
      const uint8_t* src = static_cast<const uint8_t*>(ux) + rd * slice;
      const void* a3 = src;
      if (p.stride > 1) {
        cuda_ok(cudaMemcpy2DAsync(gathered, slice, src, slice * p.stride, slice, p.od, cudaMemcpyDeviceToDevice, st),
                "depth-slice gather");
        a3 = gathered;
      }
      const void* b3 = static_cast<const uint8_t*>(uw) + rd * (size_t)(p.r * p.s * p.c) * eb;
      const bool last = rd == p.kd - 1;
      void* o3 = last ? dout : acc[rd & 1];
      const Status s = run_problem(problem(p.n), opts, a3, b3, seed, o3, last ? e : mid, st);
      if (!s.ok()) fail(s);
      seed = o3;
    }
    cuda_ok(cudaMemcpyAsync(host_out, dout, (size_t)out_bytes, cudaMemcpyDeviceToHost, st), "D2H output");
    cuda_ok(cudaStreamSynchronize(st), "tensorized op");
    return;
  }
  const Status s = run_problem(problem(p.family == KernelPlan::Family::Matmul ? p.m : p.n), opts, a, b, ds, dout, e, st);
  if (!s.ok()) fail(s);
  cuda_ok(cudaMemcpyAsync(host_out, dout, (size_t)out_bytes, cudaMemcpyDeviceToHost, st), "D2H output");
  cuda_ok(cudaStreamSynchronize(st), "tensorized op");
}

namespace {

// TensorValues packed at their declared element widths (the C ABI's buffers).
std::map<std::string, std::vector<uint8_t>> pack_inputs(const ComputeOp& op, const Inputs& inputs) {
  std::map<std::string, std::vector<uint8_t>> packed;
  for (const auto& [name, v] : inputs) {
    const TensorDecl* d = op.find_tensor(name);
    if (!d) throw MissingInput("no tensor named '" + name + "'");
    if (v.dtype != d->dtype || v.shape != d->shape) throw ShapeError("input '" + name + "' does not match its declaration");
    std::vector<uint8_t> buf(v.size() * elem_bytes(d->dtype));
    for (int64_t i = 0; i < v.size(); ++i) {
      if (d->dtype == kF16) {
        const uint16_t h = f64_to_f16_bits(v.fdata[i]);
        std::memcpy(&buf[i * 2], &h, 2);
      } else if (d->dtype == kF32) {
        const float f = static_cast<float>(v.fdata[i]);
        std::memcpy(&buf[i * 4], &f, 4);
      } else {
        const uint64_t u = static_cast<uint64_t>(v.idata[i]);
        std::memcpy(&buf[i * elem_bytes(d->dtype)], &u, elem_bytes(d->dtype));
      }
    }
    packed[name] = std::move(buf);
  }
  return packed;
}

}  // namespace

std::string tune_tensorized(const TensorizedOp& t, const Inputs& inputs, int reps) {
  using namespace tzcb200;
  const KernelPlan& p = t.plan;
  if (p.family != KernelPlan::Family::Matmul && p.family != KernelPlan::Family::ConvNHWC)
    throw InjectError("tune times matmul / NHWC-conv plans; blocked layouts run those after the K5 adapters");
  auto packed = pack_inputs(t.op, inputs);
  auto dev = [&](int slot, const std::string& name) -> void* {
    auto it = packed.find(name);
    if (it == packed.end()) return nullptr;
    void* d = pool(slot, it->second.size());
    cuda_ok(cudaMemcpy(d, it->second.data(), it->second.size(), cudaMemcpyHostToDevice), "H2D");
    return d;
  };
  void* dx = dev(0, p.data);
  void* dw = dev(1, p.weight);
  if (!dx || !dw) throw MissingInput("tune needs the data and weight tensors");
  void* ds = t.op.update ? dev(2, t.op.out) : nullptr;
  const TensorDecl& to = t.op.output();
  void* dout = pool(3, (size_t)to.size() * elem_bytes(to.dtype));
  tzc_out_layout ol{};
  ol.nb = (int32_t)p.out_nb;
  ol.stride_m = p.out_stride_m;
  ol.stride_blk = p.out_stride_blk;
  const tzc_epilogue e{p.f16 ? TZC_EP_F32 : TZC_EP_I32, 1.0f};
  char log[1 << 14];
  log[0] = 0;
  int rc;
  if (p.family == KernelPlan::Family::Matmul) {
    tzc_gemm_desc g{};
    g.profile = p.f16 ? TZC_PROFILE_F16 : TZC_PROFILE_U8I8;
    g.m = (int32_t)p.m;
    g.n = (int32_t)p.k;
    g.k = (int32_t)p.c;
    g.b_kn = p.b_kn ? 1 : 0;
    g.out = ol;
    rc = tzc_b200_tune_gemm(&g, dx, dw, ds, dout, &e, reps, 1, log, sizeof log, nullptr);
  } else {
    tzc_conv_desc c{};
    c.profile = p.f16 ? TZC_PROFILE_F16 : TZC_PROFILE_U8I8;
    c.n = (int32_t)p.n;
    c.hp = (int32_t)p.hp;
    c.wp = (int32_t)p.wp;
    c.c = (int32_t)p.c;
    c.k = (int32_t)p.k;
    c.r = (int32_t)p.r;
    c.s = (int32_t)p.s;
    c.stride = (int32_t)p.stride;
    c.w_stride_k = p.w_stride_k;
    c.w_stride_tap = p.w_stride_tap;
    c.out = ol;
    rc = tzc_b200_tune_conv(&c, dx, dw, ds, dout, &e, reps, 1, log, sizeof log, nullptr);
  }
  if (rc < 0) {
    const std::string msg = tzc_b200_last_error();
    if (rc == TZC_E_DEVICE) throw DeviceError(msg);
    throw InjectError(msg);
  }
  return log;
}

TensorValue run_tensorized(const TensorizedOp& t, const Inputs& inputs, const ComputeOp* epilogue_op) {
  // pack TensorValues at their declared widths, run, unpack
  const std::map<std::string, std::vector<uint8_t>> packed = pack_inputs(t.op, inputs);
  std::map<std::string, const void*> ptrs;
  for (const auto& [name, buf] : packed) ptrs[name] = buf.data();
  const Epi ep = epilogue_of(t.op, epilogue_op);
  const std::vector<int64_t>& shape = t.op.output().shape;
  TensorValue out = TensorValue::zeros(ep.out_dtype, shape);
  std::vector<uint8_t> raw(out.size() * elem_bytes(ep.out_dtype));
  run_tensorized_packed(t, ptrs, raw.data(), (int64_t)raw.size(), epilogue_op);
  for (int64_t i = 0; i < out.size(); ++i) {
    if (ep.out_dtype == kF16) {
      uint16_t h;
      std::memcpy(&h, &raw[i * 2], 2);
      out.fdata[i] = f16_bits_to_f64(h);
    } else if (ep.out_dtype == kF32) {
      float f;
      std::memcpy(&f, &raw[i * 4], 4);
      out.fdata[i] = f;
    } else {
      uint64_t u = 0;
      std::memcpy(&u, &raw[i * elem_bytes(ep.out_dtype)], elem_bytes(ep.out_dtype));
      out.idata[i] = wrap_int(static_cast<int64_t>(u), ep.out_dtype);
    }
  }
  return out;
}

}  // namespace tzc
