// pgti_dcrnn_step, precision = 1: bf16 operands on the 5th-gen tensor cores (tcgen05, fp32 TMEM
// accumulation).  Differences from the fp32 path (dcrnn.cu):
//  * the diffusion blocks of H and r*H are bf16 (tensor-core A operands, forward SpMM
//    operands); an fp32 copy of H carries the recurrence; weights are re-tiled to bf16 per step;
//  * layer 0's F-channel input part stays fp32 (FFMA in the GEMM epilogue; skinny wgrad rows);
//  * backward "diffuse-then-GEMM": dZ = sum_m (P^m)^T dG W_m^T = sum_m ((P^m)^T dG) W_m^T, so
//    the gate gradient (2H wide, bf16) is diffused with the transposed operators and ONE
//    multi-block tcgen05 GEMM accumulates dZ straight into the fp32 BPTT accumulators;
//  * layer pipelining: layer l runs on its own stream; (l+1, t) depends only on (l, t) and
//    (l+1, t-1), so layer l at t+1 overlaps layer l+1 at t (and the reverse wavefront in BPTT).
//    Cross-layer gradients use per-layer, time-parity double buffers (dHup) so no two streams
//    ever write the same accumulator.  Captured into one CUDA graph this is a DAG, not a chain.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <vector>

#include "dcrnn_common.cuh"
#include "tc_gemm.cuh"

namespace pgti {
namespace detail {
namespace {

using bf16 = __nv_bfloat16;

// ------------------------------------------------------------------ streams / events
struct StreamPool {
  std::vector<cudaStream_t> side;
  std::vector<cudaEvent_t> ev;
  size_t next = 0;
};

// One pool per (host thread, device, caller stream): side streams for layers 1.., a ring of
// events.  Steps issued on different caller streams get different side streams, so they stay
// independent (no false ordering between their layer chains, also under graph capture).
StreamPool *pool(int nside, cudaStream_t caller, cudaError_t *err) {
  thread_local std::map<std::pair<int, cudaStream_t>, StreamPool> pools;
  int dev = 0;
  *err = cudaGetDevice(&dev);
  if (*err != cudaSuccess) return nullptr;
  StreamPool &p = pools[{dev, caller}];
  while (int(p.side.size()) < nside) {
    cudaStream_t st;
    *err = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    if (*err != cudaSuccess) return nullptr;
    p.side.push_back(st);
  }
  while (p.ev.size() < 1024) {
    cudaEvent_t e;
    *err = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    if (*err != cudaSuccess) return nullptr;
    p.ev.push_back(e);
  }
  return &p;
}

// `to` waits for all work enqueued so far on `from`.
cudaError_t depend(StreamPool *p, cudaStream_t from, cudaStream_t to) {
  if (from == to) return cudaSuccess;
  cudaEvent_t e = p->ev[p->next++ % p->ev.size()];
  cudaError_t r = cudaEventRecord(e, from);
  if (r != cudaSuccess) return r;
  return cudaStreamWaitEvent(to, e, 0);
}

cudaError_t record(StreamPool *p, cudaStream_t st, cudaEvent_t *out) {
  *out = p->ev[p->next++ % p->ev.size()];
  return cudaEventRecord(*out, st);
}

// ------------------------------------------------------------------ workspace
struct LayoutTC {
  size_t Dx, Dy, Xb, yhat, dyhat, lossp, total;
  std::vector<size_t> DHb, DrHb, H32, Rg, Ug, Cg, dGb, dCb, Wf_ru, Wf_c, Wd_ru, Wd_c;
  std::vector<size_t> Q, wpart, spart, dHrec0, dHrec1, dHup0, dHup1;
  size_t wpart_floats, spart_floats;
};

// forward B k-blocks per layer: layer 0 = the M hidden blocks + one x k-block (the layer-0
// input channels folded into the MMA); layer > 0 = M x (input, hidden)
int nkb_total(const Dims &d, int l) { return l == 0 ? d.M + 1 : 2 * d.M; }
int vrows(const Dims &d, int l) { return l == 0 ? d.M * 64 : d.M * (d.H + d.H); }

LayoutTC make_layout_tc(const Dims &d) {
  LayoutTC L{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += round_up(int64_t(bytes), 1024);
    return o;
  };
  const size_t R = size_t(d.R), H = size_t(d.H), M = size_t(d.M), T = size_t(d.T_in);
  const size_t TT = size_t(d.steps());  // hidden-state steps (encoder + decoder for model 1)
  L.Dx = take(M * T * R * d.F * 4);
  L.Dy = take(d.model ? size_t(d.T_out) * M * R * d.F_out * 4 : 0);
  L.Xb = take(T * R * 64 * 2);  // layer-0 input channels as one bf16 k-block per row
  const int Tmax = std::max(d.T_in, d.model ? d.T_out : 0);
  const size_t spf = std::max(small_wgrad_partial_floats(Tmax, int(d.R), 2 * d.H),
                              small_wgrad_partial_floats(d.T_out, int(d.R), d.H));
  L.spart_floats = spf;
  size_t wp = spf;
  for (int l = 0; l < d.L; ++l)  // layer 0: + the packed input rows' chunk (x fold)
    wp = std::max(wp, tc_wgrad_partial_floats(vrows(d, l) + (l == 0 ? 64 : 0), 2 * d.H, Tmax,
                                              int(d.R)));
  L.wpart_floats = wp;
  for (int ll = 0; ll < d.L * (d.model ? 2 : 1); ++ll) {  // bf16 weight tiles per layer set
    const int l = ll % d.L;
    L.Wf_ru.push_back(take(size_t(nkb_total(d, l)) * 2 * H * 64 * 2));
    L.Wf_c.push_back(take(size_t(nkb_total(d, l)) * H * 64 * 2));
    L.Wd_ru.push_back(take(size_t(vrows(d, l)) * 2 * H * 2));
    L.Wd_c.push_back(take(size_t(vrows(d, l)) * H * 2));
  }
  for (int l = 0; l < d.L; ++l) {
    L.DHb.push_back(take(TT * M * R * H * 2));
    L.DrHb.push_back(take(TT * M * R * H * 2));
    L.H32.push_back(take(TT * R * H * 4));
    L.Rg.push_back(take(TT * R * H * 2));  // r, c: bf16 (backward-only operands)
    L.Ug.push_back(take(TT * R * H * 4));
    L.Cg.push_back(take(TT * R * H * 2));
    L.dGb.push_back(take(TT * R * 2 * H * 2));  // bf16 only: dgrad / wgrad operands and the
    L.dCb.push_back(take(TT * R * H * 2));      // skinny bias / input-row reductions
    // per-layer (= per-stream) scratch
    L.Q.push_back(take(M * R * 2 * H * 2));
    L.wpart.push_back(take(wp * 4));
    L.spart.push_back(take(spf * 4));  // the skinny reductions' own partials (aux stream)
    L.dHrec0.push_back(take(R * H * 4));
    L.dHrec1.push_back(take(R * H * 4));
    L.dHup0.push_back(take(R * H * 4));
    L.dHup1.push_back(take(R * H * 4));
  }
  L.yhat = take(size_t(d.T_out) * R * d.F_out * 4);
  L.dyhat = take(size_t(d.T_out) * R * d.F_out * 4);
  L.lossp = take(size_t(kLossBlocks) * 8);
  L.total = off;
  return L;
}

}  // namespace

size_t workspace_tc(const Dims &d) { return make_layout_tc(d).total; }

pgti_status run_step_tc(const pgti_dcrnn_desc &g, const Dims &d, const float *params,
                        float *grads, const WindowSrc &x, const WindowSrc &y, float *loss_dev,
                        char *ws, float *act_dump, cudaStream_t s) {
  const LayoutTC Ly = make_layout_tc(d);
  const ParamOffsets P = param_offsets(d);
  auto Fp = [&](size_t off) { return reinterpret_cast<float *>(ws + off); };
  auto Bp = [&](size_t off) { return reinterpret_cast<bf16 *>(ws + off); };
  const int64_t R = d.R, H = d.H, M = d.M, RH = R * H, MRH = M * RH;
  const int T = d.T_in, L = d.L, TT = d.steps();
  float *Dx = Fp(Ly.Dx), *Dy = Fp(Ly.Dy);
  const int64_t RF = R * d.F, RFo = R * d.F_out;
  // encoder-decoder bookkeeping (model 1, reading c24): decoder steps t >= T use layer set L + l,
  // a readout every decoder step, and a layer-0 input diffused per step (Dy)
  auto is_dec = [&](int t) { return d.model == 1 && t >= T; };
  auto pset = [&](int t, int l) { return is_dec(t) ? L + l : l; };
  auto out_slot = [&](int t) {
    return d.model == 1 ? (t >= T ? t - T : -1) : (t >= T - d.T_out ? t - (T - d.T_out) : -1);
  };
  unsigned *err = device_error_flag();
  PGTI_REQUIRE(err, PGTI_ERR_CUDA, "device error flag unavailable");
  cudaError_t perr = cudaSuccess;
  StreamPool *sp = pool(2 * L - 1, s, &perr);  // L - 1 layer streams + L weight-gradient aux
  CU(perr);
  std::vector<cudaStream_t> st(L);
  st[0] = s;
  for (int l = 1; l < L; ++l) st[l] = sp->side[l - 1];

  // ------------------------------------------------------------------ prologue on s
  {
    WeightJob jobs[32];
    int nj = 0;
    for (int ll = 0; ll < L * (d.model ? 2 : 1); ++ll) {
      const int l = ll % L, Fin = l > 0 ? d.H : (ll < L ? d.F : d.F_out), C = Fin + d.H;
      jobs[nj++] = WeightJob{params + P.Wru[ll], 2 * d.H, C, d.M, Fin, l == 0, Bp(Ly.Wf_ru[ll]),
                             Bp(Ly.Wd_ru[ll])};
      jobs[nj++] = WeightJob{params + P.Wc[ll], d.H, C, d.M, Fin, l == 0, Bp(Ly.Wf_c[ll]),
                             Bp(Ly.Wd_c[ll])};
    }
    for (int i = 0; i < nj; i += 8) CU(launch_convert_weights(jobs + i, std::min(8, nj - i), s));
  }
  CU(launch_x_prep(x, d.B, T, d.ld, d.N, d.F, Dx, err, s));
  CU(diffuse_fwd(g, d, Dx, int64_t(T) * RF, T, RF, int64_t(d.B) * d.F, s));
  // the encoder's layer-0 input part goes through the MMA: all M F diffused input channels of a
  // row packed into one bf16 k-block (the decoder's per-step input keeps the FFMA epilogue)
  bf16 *Xb = Bp(Ly.Xb);
  const bool xfold = !std::getenv("PGTI_NO_XFOLD");
  if (xfold) CU(launch_xpack(Dx, int64_t(T) * RF, T, R, d.F, d.M, Xb, s));
  for (int l = 1; l < L; ++l) CU(depend(sp, s, st[l]));  // fork

  // ------------------------------------------------------------------ forward
  std::vector<std::vector<cudaEvent_t>> fdone(L, std::vector<cudaEvent_t>(TT));
  for (int t = 0; t < TT; ++t) {
    if (is_dec(t)) {  // decoder layer-0 input on layer 0's stream: GO, previous prediction/target
      float *blk = Dy + int64_t(t - T) * M * RFo;
      if (t == T) {
        CU(cudaMemsetAsync(blk, 0, size_t(M * RFo) * 4, st[0]));
      } else {
        if (d.fed_truth(t - T)) {
          CU(launch_dec_input(y, t - T - 1, d.B, d.T_out, d.ld, d.N, d.F, d.F_out, blk, st[0]));
        } else {
          if (L > 1) CU(cudaStreamWaitEvent(st[0], fdone[L - 1][t - 1], 0));
          CU(cudaMemcpyAsync(blk, Fp(Ly.yhat) + int64_t(t - T - 1) * RFo, size_t(RFo) * 4,
                             cudaMemcpyDeviceToDevice, st[0]));
        }
        CU(diffuse_fwd(g, d, blk, RFo, 1, 0, int64_t(d.B) * d.F_out, st[0]));
      }
    }
    for (int l = 0; l < L; ++l) {
      cudaStream_t ss = st[l];
      if (l > 0) CU(cudaStreamWaitEvent(ss, fdone[l - 1][t], 0));
      const int Fin = l > 0 ? d.H : (is_dec(t) ? d.F_out : d.F), C = Fin + d.H, ps = pset(t, l);
      float *Xin = is_dec(t) ? Dy + int64_t(t - T) * M * RFo : Dx + t * RF;
      const int64_t x_ms = is_dec(t) ? RFo : int64_t(T) * RF;
      const bf16 *Ain = l == 0 ? nullptr : Bp(Ly.DHb[l - 1]) + t * MRH;
      const bf16 *DHp = t > 0 ? Bp(Ly.DHb[l]) + (t - 1) * MRH : nullptr;
      bf16 *DHt = Bp(Ly.DHb[l]) + t * MRH, *DrHt = Bp(Ly.DrHb[l]) + t * MRH;
      const float *Hp32 = t > 0 ? Fp(Ly.H32[l]) + (t - 1) * RH : nullptr;
      bf16 *r = Bp(Ly.Rg[l]) + t * RH, *c = Bp(Ly.Cg[l]) + t * RH;
      float *u = Fp(Ly.Ug[l]) + t * RH;
      // k-blocks: (input block m: map A0) and (hidden block m: map A1), B = Wf[kb] tiles
      const bool fold = l == 0 && xfold && !is_dec(t);
      auto fill_kb = [&](TcFwd &f, const bf16 *Ah, int Nout) {
        f.A0 = Ain, f.A1 = Ah, f.CA = 64, f.M0 = d.M, f.M1 = d.M;
        f.bX = 64, f.bY = Nout, f.bZ = nkb_total(d, l);
        f.nkb = 0;
        if (fold) {  // the x k-block: A0 = this step's packed input rows, B k-block M
          f.A0 = Xb + int64_t(t) * R * 64, f.M0 = 1;
          f.kb_as[f.nkb] = 0, f.kb_am[f.nkb] = 0, f.kb_ac[f.nkb] = 0;
          f.kb_bx[f.nkb] = 0, f.kb_by[f.nkb] = 0, f.kb_bz[f.nkb] = d.M, ++f.nkb;
        }
        for (int m = 0; m < d.M; ++m) {
          if (l > 0) {
            f.kb_as[f.nkb] = 0, f.kb_am[f.nkb] = m, f.kb_ac[f.nkb] = 0;
            f.kb_bx[f.nkb] = 0, f.kb_by[f.nkb] = 0, f.kb_bz[f.nkb] = 2 * m, ++f.nkb;
          }
          if (Ah) {
            f.kb_as[f.nkb] = 1, f.kb_am[f.nkb] = m, f.kb_ac[f.nkb] = 0;
            f.kb_bx[f.nkb] = 0, f.kb_by[f.nkb] = 0, f.kb_bz[f.nkb] = l > 0 ? 2 * m + 1 : m, ++f.nkb;
          }
        }
      };
      TcFwd gate{};
      gate.R = int(R), gate.H = d.H, gate.Nout = 2 * d.H, gate.mode = kEpiGate, gate.ntiles = 2;
      fill_kb(gate, DHp, 2 * d.H);
      gate.Bw = Bp(Ly.Wf_ru[ps]);
      gate.bias = params + P.bru[ps];
      if (l == 0 && !fold)
        gate.Dx = Xin, gate.dx_mstride = x_ms, gate.F = Fin, gate.C_in = C, gate.M = d.M,
        gate.Wx = params + P.Wru[ps];
      gate.Hprev = Hp32;
      gate.out_r = r, gate.out_u = u, gate.out_rH = DrHt;
      CU(launch_tc_fwd(gate, ss));
      CU(diffuse_fwd(g, d, reinterpret_cast<float *>(DrHt), RH, 1, 0, int64_t(d.B) * d.H, ss, 1));

      TcFwd cand{};
      cand.R = int(R), cand.H = d.H, cand.Nout = d.H, cand.mode = kEpiCand, cand.ntiles = 1;
      fill_kb(cand, t > 0 ? DrHt : nullptr, d.H);
      cand.Bw = Bp(Ly.Wf_c[ps]);
      cand.bias = params + P.bc[ps];
      if (l == 0 && !fold)
        cand.Dx = Xin, cand.dx_mstride = x_ms, cand.F = Fin, cand.C_in = C, cand.M = d.M,
        cand.Wx = params + P.Wc[ps];
      cand.Hprev = Hp32, cand.u_in = u, cand.out_c = c;
      cand.out_H = Fp(Ly.H32[l]) + t * RH, cand.out_Hb = DHt;
      if (l == L - 1 && out_slot(t) >= 0) {
        cand.Wout = params + P.Wout, cand.bout = params + P.bout, cand.F_out = d.F_out;
        cand.yhat = Fp(Ly.yhat) + int64_t(out_slot(t)) * RFo;
      }
      CU(launch_tc_fwd(cand, ss));
      if (!(l == L - 1 && t == TT - 1))
        CU(diffuse_fwd(g, d, reinterpret_cast<float *>(DHt), RH, 1, 0, int64_t(d.B) * d.H, ss, 1));
      if (l + 1 < L || d.model == 1) CU(record(sp, ss, &fdone[l][t]));
    }
  }
  cudaStream_t top = st[L - 1];
  CU(launch_loss(Fp(Ly.yhat), y, d.T_out, d.N, d.B, d.F, d.F_out, d.ld, Fp(Ly.dyhat),
                 reinterpret_cast<double *>(ws + Ly.lossp), loss_dev, err, top));
  if (!grads) {  // pgti_dcrnn_loss: forward and loss only
    for (int l = 1; l < L; ++l) CU(depend(sp, st[l], s));  // join
    return PGTI_OK;
  }

  // ------------------------------------------------------------------ backward (BPTT)
  // dZ = sum_m Q_m W_m^T, Q_0 = gradient itself (map A0), Q_{m>0} = (P^m)^T grad (map A1)
  struct GateFuse {
    const float *Hprev;
    const bf16 *r;
    float *dG;
    bf16 *dGb;
    float *dHprev;
  };
  auto bwd_gemm = [&](int l, const bf16 *grad, int NG, const bf16 *Wd, bf16 *Q, bool need_in,
                      bool need_h, float *dst_in, int acc_in, float *dst_h, int acc_h,
                      const GateFuse *fuse, cudaStream_t ss) -> pgti_status {
    const int vseg = l == 0 ? 64 : 2 * d.H;
    TcFwd b{};
    b.R = int(R), b.H = d.H, b.Nout = NG, b.mode = kEpiBwd;
    b.A0 = grad, b.A1 = Q, b.CA = NG, b.M0 = 1, b.M1 = d.M;
    b.Bw = Wd, b.bX = NG, b.bY = vrows(d, l), b.bZ = 1;
    b.nkb = 0;
    for (int m = 0; m < d.M; ++m)
      for (int jb = 0; jb < NG / 64; ++jb) {
        b.kb_as[b.nkb] = m > 0, b.kb_am[b.nkb] = m, b.kb_ac[b.nkb] = jb * 64;
        b.kb_bx[b.nkb] = jb * 64, b.kb_by[b.nkb] = m * vseg, b.kb_bz[b.nkb] = 0, ++b.nkb;
      }
    // column tiles: l > 0 -> [input (64), hidden (64)]; l = 0 -> [hidden]
    int nt = 0;
    if (need_in) b.dst[nt] = dst_in, b.dst_acc[nt] = acc_in, ++nt;
    if (need_h) {
      if (fuse) {
        b.fuse_tile = nt, b.Hprev = fuse->Hprev, b.g_r = fuse->r, b.g_dG = fuse->dG;
        b.g_dGb = fuse->dGb, b.g_dHprev = fuse->dHprev;
      }
      b.dst[nt] = dst_h, b.dst_acc[nt] = acc_h, ++nt;
    }
    if (nt == 0) return PGTI_OK;
    if (l > 0 && !need_in)  // skip the input tile: shift B rows by one 64-column tile
      for (int k = 0; k < b.nkb; ++k) b.kb_by[k] += 64;
    b.ntiles = nt;
    CU(launch_tc_fwd(b, ss));
    return PGTI_OK;
  };
  std::vector<std::vector<cudaEvent_t>> bdone(L, std::vector<cudaEvent_t>(TT));
  auto rec_buf = [&](int l, int t) { return Fp((t & 1) ? Ly.dHrec1[l] : Ly.dHrec0[l]); };
  auto up_buf = [&](int l, int t) { return Fp((t & 1) ? Ly.dHup1[l] : Ly.dHup0[l]); };
  for (int t = TT - 1; t >= 0; --t) {
    for (int l = L - 1; l >= 0; --l) {
      cudaStream_t ss = st[l];
      // d(H^l_t) from above is ready; the parity buffer this step writes (for layer l-1) was
      // last read by (l-1, t+2)
      if (l + 1 < L) CU(cudaStreamWaitEvent(ss, bdone[l + 1][t], 0));
      if (l > 0 && t + 2 < TT) CU(cudaStreamWaitEvent(ss, bdone[l - 1][t + 2], 0));
      // own-prediction decoder: the next step's layer 0 added its input gradient to this step's
      // dyhat
      const bool fed_back = d.model == 1 && t + 1 < TT && t + 1 > T && !d.fed_truth(t + 1 - T);
      if (l == L - 1 && fed_back && L > 1) CU(cudaStreamWaitEvent(ss, bdone[0][t + 1], 0));
      const bool feed = l == 0 && d.model == 1 && t > T && !d.fed_truth(t - T);  // yhat_{t-1}
      const bool need_in = l > 0, need_h = t > 0;
      const int ps = pset(t, l), C0 = (is_dec(t) ? d.F_out : d.F) + d.H;
      const float *Hprev = t > 0 ? Fp(Ly.H32[l]) + (t - 1) * RH : nullptr;
      const bf16 *r = Bp(Ly.Rg[l]) + t * RH, *c = Bp(Ly.Cg[l]) + t * RH;
      const float *u = Fp(Ly.Ug[l]) + t * RH;
      float *dC = nullptr, *dG = nullptr;
      bf16 *dCb = Bp(Ly.dCb[l]) + t * RH, *dGb = Bp(Ly.dGb[l]) + t * 2 * RH;
      const float *dy = (l == L - 1 && out_slot(t) >= 0)
                            ? Fp(Ly.dyhat) + int64_t(out_slot(t)) * RFo
                            : nullptr;
      float *dfeed = feed ? Fp(Ly.dyhat) + int64_t(out_slot(t) - 1) * RFo : nullptr;
      const float *dH_rec = t + 1 < TT ? rec_buf(l, t) : nullptr;  // from (l, t+1)
      const float *dH_up = l + 1 < L ? up_buf(l, t) : nullptr;     // from (l+1, t)
      float *dH_prev = need_h ? rec_buf(l, t - 1) : nullptr;       // to (l, t-1)
      float *dIn = need_in ? up_buf(l - 1, t) : nullptr;           // to (l-1, t)
      bf16 *Q = Bp(Ly.Q[l]);
      // candidate backward (+ dG_u, and dG_r = 0 at t = 0)
      CU(launch_cand_bwd_tc(RH, d.H, dH_rec, dH_up, dy, params + P.Wout, d.F_out, u, c, Hprev,
                            dC, dCb, dH_prev, dG, dGb, ss));
      if (need_in || need_h || feed) {
        // d[in, r*H] = sum_m ((P^m)^T dC) W_c[m]^T; the hidden tile's epilogue runs the gate
        // backward (dG_r, dH_{t-1} += d(rH) r) in place of storing d(rH)
        CU(diffuse_fwd(g, d, reinterpret_cast<float *>(Q), RH, 1, 0, int64_t(d.B) * d.H, ss, 1, 1,
                       dCb));
        const GateFuse fz{Hprev, r, dG, dGb, dH_prev};
        PGTI_STATUS_TRY(bwd_gemm(l, dCb, d.H, Bp(Ly.Wd_c[ps]), Q, need_in, need_h, dIn, 0,
                                 nullptr, 0, &fz, ss));
        if (feed)  // the decoder input's F_out channels: into the previous prediction's dyhat
          CU(launch_xpart_dgrad(dCb, Q, RH, d.M, d.H, params + P.Wc[ps], C0, d.F_out, R, dfeed,
                                ss));
        // d[in, H] += sum_m ((P^m)^T dG) W_ru[m]^T
        CU(diffuse_fwd(g, d, reinterpret_cast<float *>(Q), 2 * RH, 1, 0, int64_t(d.B) * 2 * d.H,
                       ss, 1, 1, dGb));
        PGTI_STATUS_TRY(bwd_gemm(l, dGb, 2 * d.H, Bp(Ly.Wd_ru[ps]), Q, need_in, need_h, dIn, 1,
                                 dH_prev, 1, nullptr, ss));
        if (feed)
          CU(launch_xpart_dgrad(dGb, Q, 2 * RH, d.M, 2 * d.H, params + P.Wru[ps], C0, d.F_out, R,
                                dfeed, ss));
      }
      CU(record(sp, ss, &bdone[l][t]));
    }
  }

  // ------------------------------------------------------------------ weight gradients
  for (int ll = 0; ll < L * (d.model ? 2 : 1); ++ll) {  // (encoder) stack, then the decoder
    const int l = ll % L, dec = ll >= L, t0 = dec ? T : 0, nt = dec ? d.T_out : T;
    cudaStream_t ss = st[l];  // layer l's backward is complete in stream order
    cudaStream_t as = sp->side[L - 1 + l];
    CU(depend(sp, ss, as));
    const int Fin = l > 0 ? d.H : (dec ? d.F_out : d.F), C = Fin + d.H;
    const int V = vrows(d, l), vseg = l == 0 ? 64 : 2 * d.H, coff = l == 0 ? Fin : 0;
    const bf16 *Ain = l == 0 ? nullptr : Bp(Ly.DHb[l - 1]) + t0 * MRH;
    float *wpart = Fp(Ly.wpart[l]);
    // gate: Z_t = [in_t, H_{t-1}] (the decoder's first step reads the encoder's last state)
    TcWgrad tw{Ain, dec ? Bp(Ly.DHb[l]) + (t0 - 1) * MRH : Bp(Ly.DHb[l]), dec ? 0 : -1, nt,
               d.M, int(R), Bp(Ly.dGb[l]) + int64_t(t0) * 2 * RH, 2 * d.H, V, vseg, coff, C,
               wpart, int64_t(Ly.wpart_floats), grads + P.Wru[ll]};
    // the encoder's layer-0 input rows (x fold): the packed rows Xb are chunk M of the v range
    // (they fill the otherwise empty half of the last 128-row tile), not a skinny reduction
    const bool xw = l == 0 && !dec && xfold;
    // (+ the bias rows from Xb's ones channel when there is room for it)
    const bool xb = xw && d.M * d.F < 64;
    if (xw) tw.A_in = Xb, tw.V = V + 64, tw.x_F = d.F, tw.x_bias = xb ? 1 : 0;
    CU(launch_tc_wgrad(tw, ss));
    tw.A_h = Bp(Ly.DrHb[l]) + t0 * MRH, tw.h_toff = 0, tw.G = Bp(Ly.dCb[l]) + int64_t(t0) * RH;
    tw.Nout = d.H, tw.out = grads + P.Wc[ll];
    CU(launch_tc_wgrad(tw, ss));
    // input rows of layer 0 (fp32 x part) and the bias rows: skinny reduction over nt*R rows,
    // on the layer's aux stream (own partials; disjoint output rows) next to the tcgen05 wgrads
    SmallWgrad sw{};
    sw.mode = kSmallBiasX, sw.T = nt, sw.R = int(R);
    if (l == 0 && !dec && !xw) sw.Dx = Dx, sw.dx_mstride = int64_t(T) * RF, sw.dx_tstride = RF;
    if (l == 0 && dec) sw.Dx = Dy, sw.dx_mstride = RFo, sw.dx_tstride = M * RFo;
    sw.M = d.M, sw.F = Fin, sw.C_in = C;
    sw.partial = Fp(Ly.spart[l]), sw.partial_cap = int64_t(Ly.spart_floats);
    sw.Gb = Bp(Ly.dGb[l]) + int64_t(t0) * 2 * RH, sw.g_tstride = 2 * RH, sw.NG = 2 * d.H;
    sw.out = grads + P.Wru[ll];
    if (!xb) CU(launch_small_wgrad(sw, as));
    sw.Gb = Bp(Ly.dCb[l]) + int64_t(t0) * RH, sw.g_tstride = RH, sw.NG = d.H;
    sw.out = grads + P.Wc[ll];
    if (!xb) CU(launch_small_wgrad(sw, as));
  }
  for (int l = 0; l < L; ++l) CU(depend(sp, sp->side[L - 1 + l], s));  // join the aux streams
  SmallWgrad rw{};
  rw.mode = kSmallReadout, rw.T = d.T_out, rw.R = int(R);
  rw.dy = Fp(Ly.dyhat), rw.F_out = d.F_out;
  rw.G = Fp(Ly.H32[L - 1]) + int64_t(TT - d.T_out) * RH, rw.g_tstride = RH, rw.NG = d.H;
  rw.partial = Fp(Ly.wpart[L - 1]), rw.partial_cap = int64_t(Ly.wpart_floats);
  rw.out = grads + P.Wout;
  CU(launch_small_wgrad(rw, top));
  for (int l = 1; l < L; ++l) CU(depend(sp, st[l], s));  // join

  if (act_dump) {
    for (int t = 0; t < TT; ++t)
      for (int l = 0; l < L; ++l) {
        float *dst = act_dump + (int64_t(t) * L + l) * 4 * RH;
        CU(cudaMemcpyAsync(dst, Fp(Ly.H32[l]) + t * RH, size_t(RH) * 4, cudaMemcpyDeviceToDevice,
                           s));
        CU(launch_bf16_to_f32(Bp(Ly.Rg[l]) + t * RH, dst + RH, RH, s));
        CU(cudaMemcpyAsync(dst + 2 * RH, Fp(Ly.Ug[l]) + t * RH, size_t(RH) * 4,
                           cudaMemcpyDeviceToDevice, s));
        CU(launch_bf16_to_f32(Bp(Ly.Cg[l]) + t * RH, dst + 3 * RH, RH, s));
      }
    CU(cudaMemcpyAsync(act_dump + int64_t(TT) * L * 4 * RH, Fp(Ly.yhat),
                       size_t(d.T_out) * R * d.F_out * 4, cudaMemcpyDeviceToDevice, s));
  }
  return PGTI_OK;
}

}  // namespace detail
}  // namespace pgti
