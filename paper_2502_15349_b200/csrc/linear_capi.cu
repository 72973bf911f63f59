// C-ABI entry points of the linear (recurrent) template: K4 forward and the K5 backward built from
// three runs of the same chunked kernel plus the per-step gradient scan for the decay factors.
#include "host_common.h"
#include "linear_chunk.cuh"
#include "linear_wide.cuh"

namespace af {
namespace {

// Scratch of the decay scan shared by every template pass of one call.
struct ScanBufs {
  float* lcum = nullptr;
  float* ucum = nullptr;
  int* cflag = nullptr;
};

size_t scan_bytes(const af_linear_desc* d) {
  const size_t units = static_cast<size_t>(d->batch) * d->heads * ((d->seq + 127) / 128);
  const size_t vec = units * kLinChunk * sizeof(float);
  return (2 * vec + units * sizeof(int) + 255) / 256 * 256;
}

ScanBufs scan_layout(const af_linear_desc* d, void* base) {
  const size_t units = static_cast<size_t>(d->batch) * d->heads * ((d->seq + 127) / 128);
  ScanBufs s;
  s.lcum = static_cast<float*>(base);
  s.ucum = d->key_gate != nullptr ? s.lcum + units * kLinChunk : nullptr;
  s.cflag = reinterpret_cast<int*>(s.lcum + 2 * units * kLinChunk);
  return s;
}

struct LaArgs {
  const void* q;
  const void* k;
  const void* v;
  const int64_t* q_st;
  const int64_t* k_st;
  const int64_t* v_st;
  int dqk, dvv;  // query/key dim, value dim of this run
  void* o;
  const int64_t* o_st;
  float out_scale;
  bool u_gate;       // key/value side scaled by the key gate
  bool row_gate;     // output rows scaled by the key gate
  const void* dot_x;
  const int64_t* x_st;
  float* dot;
  bool reverse;
  float* final_state = nullptr;
  ScanBufs scan{};
  const void* dot2_x = nullptr;  // second dot (same strides as dot_x)
  float* dot2 = nullptr;
};

StepTensor step_tensor(const float* ptr, const int64_t* st) {
  StepTensor t{};
  t.ptr = ptr;
  if (ptr != nullptr) {
    t.sb = st[0];
    t.sh = st[1];
    t.ss = st[2];
  }
  return t;
}

LinearParams base_params(const af_linear_desc* d) {
  LinearParams p{};
  p.batch = d->batch;
  p.heads = d->heads;
  p.seq = d->seq;
  p.log_const = d->log_decay_const;
  p.nfac = d->n_decay_factors;
  for (int f = 0; f < d->n_decay_factors; ++f)
    p.fac[f] = step_tensor(d->decay_factor[f], d->decay_factor_stride[f]);
  return p;
}

template <int DK, bool kRev, bool kFac>
int launch_la(const af_linear_desc* d, const LaArgs& a, cudaStream_t s) {
  using L = LinSmem<DK>;
  CUtensorMap tq, tk, tv;
  if (!make_tmap_4d(&tq, a.q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.dqk, d->seq, d->heads,
                    d->batch, a.q_st, 64, kLinChunk, true) ||
      !make_tmap_4d(&tk, a.k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.dqk, d->seq, d->heads,
                    d->batch, a.k_st, 64, kLinChunk, true) ||
      !make_tmap_4d(&tv, a.v, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.dvv, d->seq, d->heads,
                    d->batch, a.v_st, 64, kLinChunk, true))
    return AF_ERR_INPUT;
  LinearParams p = base_params(d);
  p.dqk = a.dqk;
  p.dv = a.dvv;
  p.out_scale = a.out_scale;
  if (a.u_gate) p.u_scale = step_tensor(d->key_gate, d->key_gate_stride);
  if (a.row_gate) p.o_rowscale = step_tensor(d->key_gate, d->key_gate_stride);
  p.o = a.o;
  p.o_sb = a.o_st[0];
  p.o_sh = a.o_st[1];
  p.o_ss = a.o_st[2];
  p.dot_x = a.dot_x;
  if (a.dot_x != nullptr) {
    p.x_sb = a.x_st[0];
    p.x_sh = a.x_st[1];
    p.x_ss = a.x_st[2];
  }
  p.dot = a.dot;
  p.dot2_x = a.dot2_x;
  p.dot2 = a.dot2;
  p.final_state = a.final_state;
  p.lcum = a.scan.lcum;
  p.ucum = a.u_gate ? a.scan.ucum : nullptr;  // the pass's own key/value-side scale
  p.cflag = a.scan.cflag;
  auto kern = linear_chunk_kernel<DK, kRev, kFac>;
  AF_SMEM_ATTR(kern, L::kTotal);
  dim3 grid(d->batch * d->heads * (a.dvv / kLinVB));
  ::af::note_launch();
  kern<<<grid, lin_threads(DK), L::kTotal, s>>>(tq, tk, tv, p);
  AF_CUDA_CHECK(cudaGetLastError());
  return AF_OK;
}

// Dk = Dv = 128: one CTA per (b, h) over the whole value dimension (linear_wide.cuh).
#ifndef AF_LIN_WIDE
#define AF_LIN_WIDE 1
#endif
template <bool kRev>
int launch_wide(const af_linear_desc* d, const LaArgs& a, cudaStream_t s) {
  using L = LinWideSmem;
  CUtensorMap tq, tk, tv;
  if (!make_tmap_4d(&tq, a.q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.dqk, d->seq, d->heads,
                    d->batch, a.q_st, 64, kLinChunk, true) ||
      !make_tmap_4d(&tk, a.k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.dqk, d->seq, d->heads,
                    d->batch, a.k_st, 64, kLinChunk, true) ||
      !make_tmap_4d(&tv, a.v, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.dvv, d->seq, d->heads,
                    d->batch, a.v_st, 64, kLinChunk, true))
    return AF_ERR_INPUT;
  LinearParams p = base_params(d);
  p.dqk = a.dqk;
  p.dv = a.dvv;
  p.out_scale = a.out_scale;
  if (a.u_gate) p.u_scale = step_tensor(d->key_gate, d->key_gate_stride);
  if (a.row_gate) p.o_rowscale = step_tensor(d->key_gate, d->key_gate_stride);
  p.o = a.o;
  p.o_sb = a.o_st[0];
  p.o_sh = a.o_st[1];
  p.o_ss = a.o_st[2];
  p.dot_x = a.dot_x;
  if (a.dot_x != nullptr) {
    p.x_sb = a.x_st[0];
    p.x_sh = a.x_st[1];
    p.x_ss = a.x_st[2];
  }
  p.dot = a.dot;
  p.dot2_x = a.dot2_x;
  p.dot2 = a.dot2;
  p.final_state = a.final_state;
  p.lcum = a.scan.lcum;
  p.ucum = a.u_gate ? a.scan.ucum : nullptr;
  p.cflag = a.scan.cflag;
  auto kern = linear_wide_kernel<kRev>;
  AF_SMEM_ATTR(kern, L::kTotal);
  ::af::note_launch();
  kern<<<d->batch * d->heads, kLinWideThreads, L::kTotal, s>>>(tq, tk, tv, p);
  AF_CUDA_CHECK(cudaGetLastError());
  return AF_OK;
}

int run_la(const af_linear_desc* d, const LaArgs& a, cudaStream_t s) {
  if (AF_LIN_WIDE && a.dqk == 128 && a.dvv == 128)
    return a.reverse ? launch_wide<true>(d, a, s) : launch_wide<false>(d, a, s);
  if (a.dvv % kLinVB != 0) {
    set_error("linear template: value dim %d is not a multiple of %d", a.dvv, kLinVB);
    return AF_ERR_UNSUPPORTED;
  }
  // decay factorisation is decided per 32-key group at run time (desc->decay_hint is advisory)
  if (a.dqk == 128)
    return a.reverse ? launch_la<128, true, true>(d, a, s) : launch_la<128, false, true>(d, a, s);
  if (a.dqk == 256)
    return a.reverse ? launch_la<256, true, true>(d, a, s) : launch_la<256, false, true>(d, a, s);
  set_error("linear template: key dim %d not instantiated (128, 256)", a.dqk);
  return AF_ERR_UNSUPPORTED;
}

int run_scan(const af_linear_desc* d, const ScanBufs& sb, cudaStream_t s) {
  LinearParams p = base_params(d);
  p.u_scale = step_tensor(d->key_gate, d->key_gate_stride);
  const int64_t warps = static_cast<int64_t>(d->batch) * d->heads * ((d->seq + 127) / 128);
  ::af::note_launch();
  linear_decay_scan_kernel<<<static_cast<unsigned>((warps + 7) / 8), 256, 0, s>>>(
      p, sb.lcum, sb.ucum, sb.cflag);
  AF_CUDA_CHECK(cudaGetLastError());
  return AF_OK;
}

int validate_linear(const af_linear_desc* d) {
  AF_REQUIRE(d != nullptr, AF_ERR_INPUT, "null descriptor");
  AF_REQUIRE(d->batch >= 1 && d->heads >= 1 && d->seq >= 1 && d->d_k >= 1 && d->d_v >= 1,
             AF_ERR_INPUT, "dims must be >= 1");
  AF_REQUIRE(d->n_decay_factors >= 0 && d->n_decay_factors <= 2, AF_ERR_UNSUPPORTED,
             "at most two per-step decay factors are supported (got %d)", d->n_decay_factors);
  AF_REQUIRE(d->q_stride[3] == 1 && d->k_stride[3] == 1 && d->v_stride[3] == 1 &&
                 d->o_stride[3] == 1,
             AF_ERR_INPUT, "feature stride must be 1");
  return AF_OK;
}

}  // namespace
}  // namespace af

extern "C" size_t af_linear_fwd_workspace(const af_linear_desc* d) {
  return d == nullptr ? 0 : af::scan_bytes(d);
}

extern "C" int af_linear_fwd(const af_linear_desc* d, const void* q, const void* k, const void* v,
                             void* o, float* final_state, void* workspace,
                             size_t workspace_bytes, void* stream) {
  using namespace af;
  int st = validate_linear(d);
  if (st != AF_OK) return st;
  AF_REQUIRE(workspace != nullptr && workspace_bytes >= scan_bytes(d), AF_ERR_INPUT,
             "workspace too small (%zu < %zu)", workspace_bytes, scan_bytes(d));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const ScanBufs sb = scan_layout(d, workspace);
  if ((st = run_scan(d, sb, s)) != AF_OK) return st;
  LaArgs a{q, k, v, d->q_stride, d->k_stride, d->v_stride, d->d_k, d->d_v, o, d->o_stride,
           d->q_scale, true, false, nullptr, nullptr, nullptr, false, final_state, sb};
  return run_la(d, a, s);
}

extern "C" size_t af_linear_bwd_workspace(const af_linear_desc* d) {
  if (d == nullptr) return 0;
  const size_t rows = static_cast<size_t>(d->batch) * d->heads * d->seq;
  const size_t slots = static_cast<size_t>(d->d_k) / 32;  // dot partials per 32-column slot
  // dot partials (q.dQm, Km.dKm, raw k.dKm), then d log a and dk_dot per step; the bf16 Km copy
  // starts 256-byte aligned
  size_t bytes = (rows * (3 * slots + 2) * sizeof(float) + 255) / 256 * 256;
  if (d->key_gate != nullptr) bytes += rows * static_cast<size_t>(d->d_k) * 2;  // bf16 Km
  bytes = (bytes + 255) / 256 * 256;
  return bytes + af::scan_bytes(d);
}

extern "C" int af_linear_bwd(const af_linear_desc* d, const void* q, const void* k, const void* v,
                             const void* dout, void* dq, void* dk, void* dv,
                             float* const* d_decay_factor, float* d_key_gate, void* workspace,
                             size_t workspace_bytes, void* stream) {
  using namespace af;
  int st = validate_linear(d);
  if (st != AF_OK) return st;
  AF_REQUIRE(workspace_bytes >= af_linear_bwd_workspace(d), AF_ERR_INPUT, "workspace too small");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t n = static_cast<int64_t>(d->batch) * d->heads * d->seq;
  const int slots = d->d_k / 32;
  float* dq_dot = static_cast<float*>(workspace);
  float* dk_dot = dq_dot + n * slots;
  float* kdot_raw = dk_dot + n * slots;
  float* step_dloga = kdot_raw + n * slots;
  float* step_dkdot = step_dloga + n;
  // (every dot partial slot of every live step is stored exactly once: no clearing needed)
  // Gated keys, materialised once (see gate_keys_kernel)
  const void* km = k;
  const int64_t* km_st = d->k_stride;
  int64_t km_contig[4] = {static_cast<int64_t>(d->heads) * d->seq * d->d_k,
                          static_cast<int64_t>(d->seq) * d->d_k, d->d_k, 1};
  if (d->key_gate != nullptr) {
    __nv_bfloat16* kmb = reinterpret_cast<__nv_bfloat16*>(
        static_cast<char*>(workspace) +
        (static_cast<size_t>(n) * (3 * slots + 2) * sizeof(float) + 255) / 256 * 256);
    const int64_t thr = n * (d->d_k >= 8 * kGkVec ? d->d_k / (8 * kGkVec) : 1);
    ::af::note_launch();
    gate_keys_kernel<<<static_cast<unsigned>((thr + 255) / 256), 256, 0, s>>>(
        static_cast<const __nv_bfloat16*>(k), d->k_stride[0], d->k_stride[1], d->k_stride[2],
        step_tensor(d->key_gate, d->key_gate_stride), d->heads, d->seq, d->d_k, kmb, n);
    AF_CUDA_CHECK(cudaGetLastError());
    km = kmb;
    km_st = km_contig;
  }
  size_t scan_off = (static_cast<size_t>(n) * (3 * slots + 2) * sizeof(float) + 255) / 256 * 256;
  if (d->key_gate != nullptr)
    scan_off = (scan_off + static_cast<size_t>(n) * d->d_k * 2 + 255) / 256 * 256;
  const ScanBufs sb = scan_layout(d, static_cast<char*>(workspace) + scan_off);
  if ((st = run_scan(d, sb, s)) != AF_OK) return st;
  const bool want_fac = d_decay_factor != nullptr &&
                        ((d->n_decay_factors > 0 && d_decay_factor[0] != nullptr) ||
                         (d->n_decay_factors > 1 && d_decay_factor[1] != nullptr));
  // the per-step dot products feed only the decay / gate gradients: skipped (no re-read of q
  // and Km) when none is requested
  const bool want_dots = want_fac || d_key_gate != nullptr;
  // dq = q_scale * LA_fwd(q=dO, k=V, v=Km)                 dq_dot = q . dq   (= Qm . dQm)
  LaArgs a1{dout, v, km, d->o_stride, d->v_stride, km_st, d->d_v, d->d_k, dq, d->q_stride,
            d->q_scale, false, false, want_dots ? q : nullptr, d->q_stride, dq_dot, false, nullptr,
            sb};
  if ((st = run_la(d, a1, s)) != AF_OK) return st;
  // dKm = q_scale * LA_rev(q=V, k=dO, v=Q); dk = gate*dKm   dk_dot = Km . dKm, and with a gate
  // gradient requested kdot_raw = k . dKm (raw keys; Km shares k's layout when materialised)
  LaArgs a2{v, dout, q, d->v_stride, d->o_stride, d->q_stride, d->d_v, d->d_k, dk, d->k_stride,
            d->q_scale, false, true, want_dots ? km : nullptr, km_st, dk_dot, true, nullptr, sb};
  // A pure key gate's gradient is k . dKm over the raw keys (a second dot in this pass; finite at
  // gate = 0).  A gate that is also a decay factor (Mamba2's dt) takes Km . dKm / gate instead:
  // its decay part d log a / gate has no finite value at 0 either way, and the division path
  // saves re-reading k.
  bool gate_is_factor = false;
  for (int f = 0; f < d->n_decay_factors; ++f)
    gate_is_factor |= d->decay_factor[f] == d->key_gate;
  const bool raw_gate_dot = d_key_gate != nullptr && !gate_is_factor;
  if (raw_gate_dot) {
    AF_REQUIRE(km_st[0] == d->k_stride[0] && km_st[1] == d->k_stride[1] &&
                   km_st[2] == d->k_stride[2],
               AF_ERR_INPUT, "gate gradient needs contiguous keys");
    a2.dot2_x = k;
    a2.dot2 = kdot_raw;
  }
  if ((st = run_la(d, a2, s)) != AF_OK) return st;
  // dV = q_scale * LA_rev(q=Km, k=Q, v=dO)
  LaArgs a3{km, q, dout, km_st, d->q_stride, d->o_stride, d->d_k, d->d_v, dv, d->v_stride,
            d->q_scale, false, false, nullptr, nullptr, nullptr, true, nullptr, sb};
  if ((st = run_la(d, a3, s)) != AF_OK) return st;
  if (want_fac || d_key_gate != nullptr) {
    LinearParams p = base_params(d);
    p.u_scale = step_tensor(d->key_gate, d->key_gate_stride);
    if (d_key_gate != nullptr)
      AF_REQUIRE(d->key_gate != nullptr, AF_ERR_INPUT, "d_key_gate without a key gate");
    ::af::note_launch();
    linear_step_grads_kernel<<<d->batch * d->heads, kStepGradThreads, 0, s>>>(
        dq_dot, dk_dot, raw_gate_dot ? kdot_raw : nullptr, slots, p, step_dloga,
        d_key_gate != nullptr ? step_dkdot : nullptr);
    AF_CUDA_CHECK(cudaGetLastError());
    // the per-step reductions: decay factors, then the gate (one launch when their outputs share
    // a broadcast pattern)
    StepReduceJobs jobs{};
    for (int f = 0; f < d->n_decay_factors; ++f)
      if (d_decay_factor != nullptr && d_decay_factor[f] != nullptr)
        jobs.job[jobs.n++] = {step_dloga, p.fac[f],
                              step_tensor(d_decay_factor[f], d->decay_factor_stride[f])};
    if (d_key_gate != nullptr)
      jobs.job[jobs.n++] = {step_dkdot,
                            raw_gate_dot ? StepTensor{nullptr, 0, 0, 0} : p.u_scale,
                            step_tensor(d_key_gate, d->key_gate_stride)};
    bool same = true;
    for (int j = 1; j < jobs.n; ++j)
      same &= (jobs.job[j].out.sb == 0) == (jobs.job[0].out.sb == 0) &&
              (jobs.job[j].out.sh == 0) == (jobs.job[0].out.sh == 0);
    for (int j0 = 0; j0 < jobs.n;) {
      StepReduceJobs one{};
      const int cnt = same ? jobs.n : 1;
      for (int j = 0; j < cnt; ++j) one.job[j] = jobs.job[j0 + j];
      one.n = cnt;
      const StepTensor& o = one.job[0].out;
      const int nb = o.sb == 0 ? 1 : d->batch, nh = o.sh == 0 ? 1 : d->heads;
      const int64_t total = static_cast<int64_t>(nb) * nh * d->seq;
      ::af::note_launch();
      step_grad_reduce_multi_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, s>>>(
          one, d->batch, d->heads, d->seq);
      AF_CUDA_CHECK(cudaGetLastError());
      j0 += cnt;
    }
  }
  return AF_OK;
}

#ifdef AF_TRACE
extern "C" int af_debug_lin_trace_read(void* host) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, af::g_lin_trace, sizeof(af::g_lin_trace)));
}
#endif
