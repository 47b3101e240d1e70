// pgti_dcrnn_step: one forward + BPTT pass of the stepwise stacked DCGRU over one gathered
// batch, plus the diffusion test hooks.  Orchestration only: every arithmetic step runs in the
// kernels of spmm.cu (K2), gemm_simt.cu / tc_gemm.cu (K3/K3'/K4/K5), small_wgrad.cu and
// elementwise.cu.  This file holds the fp32 parity path (precision 0) and the C ABI; the bf16
// tcgen05 path (precision 1) is dcrnn_tc.cu.
//
// Workspace of the fp32 path (all device, caller-owned; R = N*B rows ordered n*B + b;
// M = 2K+1):
//   Dx        [M][T_in][R*F]        diffusion blocks of every x_t (layer-0 input)
//   DH[l]     [T_in][M][R*H]        diffusion blocks of H^l_t (block 0 = H^l_t itself)
//   DrH[l]    [T_in][M][R*H]        diffusion blocks of r*H^l_{t-1}
//   Rg/Ug/Cg  [l][T_in][R*H]        saved gates r, u and candidate c
//   dG[l]     [T_in][R*2H], dC[l] [T_in][R*H]   gate / candidate pre-activation grads (wgrad)
//   yhat, dyhat [T_out][R*F_out]; loss partials; BPTT accumulators and temporaries;
//   split-K partial sums of the weight gradients.
// "Only new columns are diffused": T(Z) = [T(in), T(H)] is column-separable,
// so each H^l_t is diffused once when produced and reused by layer l+1 at t and layer l at t+1.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "dcrnn_common.cuh"

namespace pgti {
namespace detail {

ParamOffsets param_offsets(const Dims &d) {
  ParamOffsets o;
  size_t off = 0;
  for (int ll = 0; ll < d.L * (d.model ? 2 : 1); ++ll) {
    const int l = ll % d.L, f0 = ll < d.L ? d.F : d.F_out;
    const size_t C = size_t((l == 0 ? f0 : d.H) + d.H);
    o.Wru.push_back(off), off += size_t(d.M) * C * 2 * d.H;
    o.bru.push_back(off), off += 2 * d.H;
    o.Wc.push_back(off), off += size_t(d.M) * C * d.H;
    o.bc.push_back(off), off += d.H;
  }
  o.Wout = off, off += size_t(d.H) * d.F_out;
  o.bout = off, off += d.F_out;
  o.total = off;
  return o;
}

pgti_status check_desc(const pgti_dcrnn_desc *desc, Dims *out) {
  PGTI_REQUIRE(desc, PGTI_ERR_INVALID_ARG, "null pgti_dcrnn_desc");
  const pgti_dcrnn_desc &g = *desc;
  PGTI_REQUIRE(g.N > 0 && g.F > 0 && g.L > 0 && g.K >= 0 && g.T_in > 0 && g.B > 0,
               PGTI_ERR_SHAPE, "desc: N=%d F=%d L=%d K=%d T_in=%d B=%d", g.N, g.F, g.L, g.K,
               g.T_in, g.B);
  PGTI_REQUIRE(g.cheb == 0 || g.cheb == 1, PGTI_ERR_INVALID_ARG, "desc: cheb=%d", g.cheb);
  PGTI_REQUIRE(g.model == 0 || g.model == 1, PGTI_ERR_INVALID_ARG,
               "desc: model=%d (0 = stepwise, 1 = encoder-decoder)", g.model);
  PGTI_REQUIRE(g.teacher_forcing == 0 ||
                   (g.model == 1 && g.teacher_forcing > 0 && g.T_out <= 31 &&
                    (g.teacher_forcing >> (g.T_out > 1 ? g.T_out - 1 : 0)) == 0),
               PGTI_ERR_INVALID_ARG,
               "desc: teacher_forcing=0x%x must be a mask of decoder steps 1..T_out-1 (model 1)",
               unsigned(g.teacher_forcing));
  PGTI_REQUIRE(g.T_out >= 1 && (g.model == 1 || g.T_out <= g.T_in), PGTI_ERR_SHAPE,
               "desc: need 1 <= T_out=%d <= T_in=%d (stepwise readout, reading c6)", g.T_out,
               g.T_in);
  PGTI_REQUIRE(g.F_out >= 1 && g.F_out <= g.F && g.F_out <= 4, PGTI_ERR_SHAPE,
               "desc: F_out=%d must be in [1, min(F, 4)]", g.F_out);
  PGTI_REQUIRE(g.H == 16 || g.H == 32 || g.H == 64, PGTI_ERR_UNSUPPORTED,
               "desc: H=%d (this build supports 16, 32, 64)", g.H);
  PGTI_REQUIRE(g.ld >= int64_t(g.N) * g.F && g.ld % 4 == 0, PGTI_ERR_ALIGNMENT,
               "desc: ld=%lld must be >= N*F and a multiple of 4", (long long)g.ld);
  PGTI_REQUIRE(g.precision == 0 || g.precision == 1, PGTI_ERR_UNSUPPORTED,
               "desc: precision=%d (0 = fp32 SIMT, 1 = bf16 tcgen05)", g.precision);
  PGTI_REQUIRE(g.precision == 0 || (g.H == 64 && g.F * (2 * g.K + 1) <= 11 && 2 * g.K + 1 <= 8 &&
                                    g.L <= 8),
               PGTI_ERR_UNSUPPORTED,
               "desc: the bf16 tcgen05 path needs H = 64, F*(2K+1) <= 11, K <= 3, L <= 8 "
               "(H=%d F=%d K=%d L=%d)",
               g.H, g.F, g.K, g.L);
  PGTI_REQUIRE(int64_t(g.N) * g.B * 2 * g.H < (int64_t(1) << 31), PGTI_ERR_SHAPE,
               "desc: N*B*2H exceeds int32 row indexing");
  if (g.K > 0)
    PGTI_REQUIRE(g.a_rowptr && g.a_col && g.Pf_val && g.PbT_val && g.at_rowptr && g.at_col &&
                     g.Pb_val && g.PfT_val && g.nnz >= 0,
                 PGTI_ERR_INVALID_ARG, "desc: CSR pointers must be set when K > 0");
  if (g.K > 0 && g.win_rows != 0)
    PGTI_REQUIRE(g.win_rows >= 1 && g.win_rows <= 64 && g.win_max >= 0 && g.a_win_ptr &&
                     g.a_win_nodes && g.a_lcol && g.at_win_ptr && g.at_win_nodes && g.at_lcol,
                 PGTI_ERR_INVALID_ARG,
                 "desc: SpMM window plan needs win_rows in [1,64], win_max >= 0 and all six "
                 "plan pointers (win_rows=%d)",
                 g.win_rows);
  Dims d{g.N, g.F, g.F_out, g.L, g.H, g.K, g.T_in, g.T_out, g.B, 2 * g.K + 1,
         int64_t(g.N) * g.B, g.ld, g.precision, g.model, g.teacher_forcing, g.cheb};
  *out = d;
  return PGTI_OK;
}

namespace {
// term t of a job: pattern(A) (pat 0) or pattern(A^T) (pat 1) with values val, operand X
void set_term(SpmmJob &j, int t, const pgti_dcrnn_desc &g, int pat, const float *val,
              const float *X) {
  // pat: 0 = pattern(A), 1 = pattern(A^T)
  j.rowptr[t] = pat ? g.at_rowptr : g.a_rowptr;
  j.col[t] = pat ? g.at_col : g.a_col;
  j.val[t] = val;
  j.X[t] = X;
  j.nnz[t] = g.nnz;
  j.win_ptr[t] = pat ? g.at_win_ptr : g.a_win_ptr;
  j.win_nodes[t] = pat ? g.at_win_nodes : g.a_win_nodes;
  j.lcol[t] = pat ? g.at_lcol : g.a_lcol;
  j.win_rows = g.win_rows, j.win_max = g.win_max;
}
}  // namespace

cudaError_t diffuse_fwd(const pgti_dcrnn_desc &g, const Dims &d, float *base, int64_t mstride,
                        int G, int64_t gstride, int64_t W, cudaStream_t s, int bf16,
                        int transposed, const void *src0) {
  const int es = bf16 ? 2 : 4;
  char *b = reinterpret_cast<char *>(base);
  const char *z = src0 ? static_cast<const char *>(src0) : b;
  auto blk = [&](int m) { return b + int64_t(m) * mstride * es; };
  for (int k = 1; k <= d.K; ++k) {
    SpmmJob j[2] = {};
    const float *xf = reinterpret_cast<const float *>(k == 1 ? z : blk(k - 1));
    const float *xb = reinterpret_cast<const float *>(k == 1 ? z : blk(d.K + k - 1));
    if (!transposed) {
      set_term(j[0], 0, g, 0, g.Pf_val, xf);
      set_term(j[1], 0, g, 1, g.Pb_val, xb);
    } else {
      set_term(j[0], 0, g, 1, g.PfT_val, xf);
      set_term(j[1], 0, g, 0, g.PbT_val, xb);
    }
    j[0].Y = reinterpret_cast<float *>(blk(k));
    j[1].Y = reinterpret_cast<float *>(blk(d.K + k));
    for (auto &jb : j) jb.nterms = 1, jb.W = W, jb.G = G, jb.gstride = gstride, jb.bf16 = bf16;
    if (d.cheb && k >= 2) {  // T_k = 2 P T_{k-1} - T_{k-2}
      j[0].alpha = j[1].alpha = 2.f, j[0].beta = j[1].beta = -1.f;
      j[0].add = reinterpret_cast<const float *>(k == 2 ? z : blk(k - 2));
      j[1].add = reinterpret_cast<const float *>(k == 2 ? z : blk(d.K + k - 2));
    }
    cudaError_t e = launch_spmm(j, 2, d.N, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t diffuse_adj(const pgti_dcrnn_desc &g, const Dims &d, AdjChain *ch, int nch,
                        cudaStream_t s) {
  if (nch == 0) return cudaSuccess;
  const int K = d.K;
  SpmmJob jobs[kMaxSpmmJobs];
  if (K == 0) {
    for (int c = 0; c < nch; ++c) {
      jobs[c] = SpmmJob{};
      jobs[c].nterms = 0, jobs[c].add = ch[c].dT, jobs[c].Y = ch[c].out;
      jobs[c].accumulate = ch[c].accumulate, jobs[c].W = ch[c].W, jobs[c].G = 1;
    }
    return launch_spmm(jobs, nch, d.N, s);
  }
  if (d.cheb && K >= 2) {
    // Chebyshev blocks (reading c25): dZ = d_0 + sum_dir sum_k T_k(A) d_k with A = P^T of the
    // direction, by Clenshaw's recurrence b_K = d_K, b_k = d_k + 2 A b_{k+1} - b_{k+2}, then
    // dZ = d_0 + sum_dir (A b_1 - b_2).  b_k overwrites b_{k+2} in place (read and written by the
    // same thread), so two temporaries per direction serve any K.
    std::vector<const float *> f1(nch), f2(nch, nullptr), b1(nch), b2(nch, nullptr);
    for (int c = 0; c < nch; ++c)
      f1[c] = ch[c].dT + K * ch[c].mstride, b1[c] = ch[c].dT + 2 * K * ch[c].mstride;
    int pp = 0;
    for (int k = K - 1; k >= 1; --k) {
      int nj = 0;
      for (int c = 0; c < nch; ++c) {
        SpmmJob f{}, b{};
        set_term(f, 0, g, 1, g.PfT_val, f1[c]);
        f.add = ch[c].dT + k * ch[c].mstride, f.add2 = f2[c], f.Y = ch[c].tf[pp];
        set_term(b, 0, g, 0, g.PbT_val, b1[c]);
        b.add = ch[c].dT + (K + k) * ch[c].mstride, b.add2 = b2[c], b.Y = ch[c].tb[pp];
        for (SpmmJob *jb : {&f, &b})
          jb->nterms = 1, jb->W = ch[c].W, jb->G = 1, jb->alpha = 2.f, jb->beta2 = -1.f;
        jobs[nj++] = f, jobs[nj++] = b;
        f2[c] = f1[c], f1[c] = ch[c].tf[pp], b2[c] = b1[c], b1[c] = ch[c].tb[pp];
      }
      cudaError_t e = launch_spmm(jobs, nj, d.N, s);
      if (e != cudaSuccess) return e;
      pp ^= 1;
    }
    for (int dir = 0; dir < 2; ++dir) {  // out (+)= d_0 + A_f b_1 - b_2, then += A_b b_1 - b_2
      for (int c = 0; c < nch; ++c) {
        SpmmJob j{};
        if (dir == 0)
          set_term(j, 0, g, 1, g.PfT_val, f1[c]), j.add = ch[c].dT, j.add2 = f2[c];
        else
          set_term(j, 0, g, 0, g.PbT_val, b1[c]), j.add2 = b2[c];
        j.nterms = 1, j.beta2 = -1.f, j.Y = ch[c].out;
        j.accumulate = dir == 1 || ch[c].accumulate, j.W = ch[c].W, j.G = 1;
        jobs[c] = j;
      }
      cudaError_t e = launch_spmm(jobs, nch, d.N, s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  std::vector<const float *> af(nch), ab(nch);
  for (int c = 0; c < nch; ++c)
    af[c] = ch[c].dT + K * ch[c].mstride, ab[c] = ch[c].dT + 2 * K * ch[c].mstride;
  int pp = 0;
  for (int k = K - 1; k >= 1; --k) {
    int nj = 0;
    for (int c = 0; c < nch; ++c) {
      SpmmJob f{}, b{};
      set_term(f, 0, g, 1, g.PfT_val, af[c]);
      f.add = ch[c].dT + k * ch[c].mstride, f.Y = ch[c].tf[pp];
      set_term(b, 0, g, 0, g.PbT_val, ab[c]);
      b.add = ch[c].dT + (K + k) * ch[c].mstride, b.Y = ch[c].tb[pp];
      for (SpmmJob *jb : {&f, &b}) jb->nterms = 1, jb->W = ch[c].W, jb->G = 1;
      jobs[nj++] = f, jobs[nj++] = b;
      af[c] = ch[c].tf[pp], ab[c] = ch[c].tb[pp];
    }
    cudaError_t e = launch_spmm(jobs, nj, d.N, s);
    if (e != cudaSuccess) return e;
    pp ^= 1;
  }
  for (int c = 0; c < nch; ++c) {
    SpmmJob j{};
    set_term(j, 0, g, 1, g.PfT_val, af[c]);
    set_term(j, 1, g, 0, g.PbT_val, ab[c]);
    j.nterms = 2, j.add = ch[c].dT, j.Y = ch[c].out, j.accumulate = ch[c].accumulate;
    j.W = ch[c].W, j.G = 1;
    jobs[c] = j;
  }
  return launch_spmm(jobs, nch, d.N, s);
}

namespace {

struct Layout {
  size_t Dx, Dy, yhat, dyhat, lossp, dU, drH, dTin, dTH, wpart, total;
  size_t tmp[8];
  std::vector<size_t> DH, DrH, Rg, Ug, Cg, dG, dC, dHa, dHb;
  size_t tmp_floats, wpart_floats;
};

Layout make_layout(const Dims &d) {
  Layout L{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += round_up(int64_t(bytes), 256);
    return o;
  };
  const size_t R = size_t(d.R), H = size_t(d.H), M = size_t(d.M), T = size_t(d.T_in);
  const size_t TT = size_t(d.steps());
  L.Dx = take(M * T * R * d.F * 4);
  // model 1: diffusion blocks of every decoder step's layer-0 input [T_out][M][R*F_out]
  L.Dy = take(d.model ? size_t(d.T_out) * M * R * d.F_out * 4 : 0);
  for (int l = 0; l < d.L; ++l) {
    L.DH.push_back(take(TT * M * R * H * 4));
    L.DrH.push_back(take(TT * M * R * H * 4));
    L.Rg.push_back(take(TT * R * H * 4));
    L.Ug.push_back(take(TT * R * H * 4));
    L.Cg.push_back(take(TT * R * H * 4));
    L.dG.push_back(take(TT * R * 2 * H * 4));
    L.dC.push_back(take(TT * R * H * 4));
    L.dHa.push_back(take(R * H * 4));
    L.dHb.push_back(take(R * H * 4));
  }
  L.yhat = take(size_t(d.T_out) * R * d.F_out * 4);
  L.dyhat = take(size_t(d.T_out) * R * d.F_out * 4);
  L.lossp = take(size_t(kLossBlocks) * 8);
  L.dU = take(R * H * 4);
  L.drH = take(R * H * 4);
  const size_t fin_max = std::max(d.L > 1 ? H : size_t(d.F), size_t(d.model ? d.F_out : 0));
  L.dTin = take(M * R * fin_max * 4);
  L.dTH = take(M * R * H * 4);
  L.tmp_floats = R * std::max(H, fin_max);
  for (int i = 0; i < 8; ++i) L.tmp[i] = take(L.tmp_floats * 4);
  size_t wp = small_wgrad_partial_floats(d.T_out, int(d.R), d.H);
  for (int ll = 0; ll < d.L * (d.model ? 2 : 1); ++ll) {
    const int l = ll % d.L, f0 = ll < d.L ? d.F : d.F_out;
    const int C = (l == 0 ? f0 : d.H) + d.H, T_set = ll < d.L ? d.T_in : d.T_out;
    wp = std::max(wp, wgrad_partial_floats(d.M, C, 2 * d.H, T_set, int(d.R)));
  }
  L.wpart_floats = wp;
  L.wpart = take(wp * 4);
  L.total = off;
  return L;
}

// The fp32 step.  Stepwise model (model 0): hidden-state steps t < T_in, readout on the last
// T_out.  Encoder-decoder (model 1, reading c24): steps t < T_in run the encoder stack (layer
// set l), steps T_in <= t < T_in + T_out the decoder stack (layer set L + l) on the same hidden
// chains, with a readout on every decoder step and the decoder's layer-0 input diffused per step
// from the GO symbol / the previous prediction / the previous target.
pgti_status run_step(const pgti_dcrnn_desc &g, const Dims &d, const float *params, float *grads,
                     const WindowSrc &x, const WindowSrc &y, float *loss_dev, char *ws,
                     float *act_dump,
                     cudaStream_t s) {
  const Layout Ly = make_layout(d);
  const ParamOffsets P = param_offsets(d);
  auto Fp = [&](size_t off) { return reinterpret_cast<float *>(ws + off); };
  const int64_t R = d.R, H = d.H, M = d.M, RH = R * H, MRH = M * RH;
  const int T = d.T_in, L = d.L, TT = d.steps();
  float *Dx = Fp(Ly.Dx), *Dy = Fp(Ly.Dy);
  const int64_t RF = R * d.F, RFo = R * d.F_out;
  unsigned *err = device_error_flag();
  PGTI_REQUIRE(err, PGTI_ERR_CUDA, "device error flag unavailable");
  // step t: decoder?  parameter set of layer l; readout slot (-1: none) of the top layer
  auto is_dec = [&](int t) { return d.model == 1 && t >= T; };
  auto pset = [&](int t, int l) { return is_dec(t) ? L + l : l; };
  auto out_slot = [&](int t) {
    return d.model == 1 ? (t >= T ? t - T : -1) : (t >= T - d.T_out ? t - (T - d.T_out) : -1);
  };
  auto fin_of = [&](int t, int l) { return l > 0 ? d.H : (is_dec(t) ? d.F_out : d.F); };
  // layer-0 input blocks of step t and their block stride
  auto in0 = [&](int t) { return is_dec(t) ? Dy + int64_t(t - T) * M * RFo : Dx + t * RF; };
  auto in0_ms = [&](int t) { return is_dec(t) ? RFo : int64_t(T) * RF; };

  // ------------------------------------------------------------------ forward
  CU(launch_x_prep(x, d.B, T, d.ld, d.N, d.F, Dx, err, s));
  CU(diffuse_fwd(g, d, Dx, int64_t(T) * RF, T, RF, int64_t(d.B) * d.F, s));
  for (int t = 0; t < TT; ++t) {
    if (is_dec(t)) {  // decoder layer-0 input: GO, previous prediction or previous target
      float *blk = Dy + int64_t(t - T) * M * RFo;
      if (t == T) {
        CU(cudaMemsetAsync(blk, 0, size_t(M * RFo) * 4, s));
      } else {
        if (d.fed_truth(t - T))
          CU(launch_dec_input(y, t - T - 1, d.B, d.T_out, d.ld, d.N, d.F, d.F_out, blk, s));
        else
          CU(cudaMemcpyAsync(blk, Fp(Ly.yhat) + int64_t(t - T - 1) * RFo, size_t(RFo) * 4,
                             cudaMemcpyDeviceToDevice, s));
        CU(diffuse_fwd(g, d, blk, RFo, 1, 0, int64_t(d.B) * d.F_out, s));
      }
    }
    for (int l = 0; l < L; ++l) {
      const int Fin = fin_of(t, l), ps = pset(t, l);
      const float *Din = l == 0 ? in0(t) : Fp(Ly.DH[l - 1]) + t * MRH;
      const int64_t din_ms = l == 0 ? in0_ms(t) : RH;
      float *DHt = Fp(Ly.DH[l]) + t * MRH;
      const float *DHp = t > 0 ? Fp(Ly.DH[l]) + (t - 1) * MRH : nullptr;
      float *DrHt = Fp(Ly.DrH[l]) + t * MRH;
      float *r = Fp(Ly.Rg[l]) + t * RH, *u = Fp(Ly.Ug[l]) + t * RH, *c = Fp(Ly.Cg[l]) + t * RH;

      GconvFwd gate{};
      gate.a = GconvA{Din, din_ms, DHp, RH, Fin, d.H, d.M};
      gate.R = int(R), gate.W = params + P.Wru[ps], gate.bias = params + P.bru[ps];
      gate.Nout = 2 * d.H, gate.mode = kEpiGate, gate.Hprev = DHp;
      gate.out_r = r, gate.out_u = u, gate.out_rH = DrHt;
      CU(launch_gconv_fwd(gate, s));
      CU(diffuse_fwd(g, d, DrHt, RH, 1, 0, int64_t(d.B) * d.H, s));

      GconvFwd cand{};
      cand.a = GconvA{Din, din_ms, DrHt, RH, Fin, d.H, d.M};
      cand.R = int(R), cand.W = params + P.Wc[ps], cand.bias = params + P.bc[ps];
      cand.Nout = d.H, cand.mode = kEpiCand, cand.Hprev = DHp;
      cand.u_in = u, cand.out_c = c, cand.out_H = DHt;
      if (l == L - 1 && out_slot(t) >= 0) {
        cand.Wout = params + P.Wout, cand.bout = params + P.bout, cand.F_out = d.F_out;
        cand.yhat = Fp(Ly.yhat) + int64_t(out_slot(t)) * RFo;
      }
      CU(launch_gconv_fwd(cand, s));
      if (!(l == L - 1 && t == TT - 1)) CU(diffuse_fwd(g, d, DHt, RH, 1, 0, int64_t(d.B) * d.H, s));
    }
  }
  CU(launch_loss(Fp(Ly.yhat), y, d.T_out, d.N, d.B, d.F, d.F_out, d.ld, Fp(Ly.dyhat),
                 reinterpret_cast<double *>(ws + Ly.lossp), loss_dev, err, s));
  if (!grads) return PGTI_OK;  // pgti_dcrnn_loss: forward and loss only

  // ------------------------------------------------------------------ backward (BPTT)
  std::vector<float *> dHcur(L), dHprev(L);
  for (int l = 0; l < L; ++l) {
    dHcur[l] = Fp(Ly.dHa[l]), dHprev[l] = Fp(Ly.dHb[l]);
    CU(cudaMemsetAsync(dHcur[l], 0, size_t(RH) * 4, s));
  }
  float *dU = Fp(Ly.dU), *drH = Fp(Ly.drH), *dTin = Fp(Ly.dTin), *dTH = Fp(Ly.dTH);
  float *tmp[8];
  for (int i = 0; i < 8; ++i) tmp[i] = Fp(Ly.tmp[i]);
  for (int t = TT - 1; t >= 0; --t) {
    for (int l = L - 1; l >= 0; --l) {
      const int Fin = fin_of(t, l), C = Fin + d.H, ps = pset(t, l);
      // the decoder's layer-0 input is the previous prediction: its gradient joins dyhat
      const bool feed = l == 0 && is_dec(t) && t > T && !d.fed_truth(t - T);
      const bool need_in = l > 0 || feed, need_h = t > 0;
      const float *Hprev = t > 0 ? Fp(Ly.DH[l]) + (t - 1) * MRH : nullptr;
      const float *r = Fp(Ly.Rg[l]) + t * RH, *u = Fp(Ly.Ug[l]) + t * RH, *c = Fp(Ly.Cg[l]) + t * RH;
      float *dC = Fp(Ly.dC[l]) + t * RH, *dG = Fp(Ly.dG[l]) + t * 2 * RH;
      const float *dy = (l == L - 1 && out_slot(t) >= 0)
                            ? Fp(Ly.dyhat) + int64_t(out_slot(t)) * RFo
                            : nullptr;
      CU(launch_cand_bwd(RH, d.H, dHcur[l], nullptr, dy, params + P.Wout, d.F_out, u, c, Hprev,
                         dU, dC, need_h ? dHprev[l] : nullptr, s));
      const int64_t tin_ms = R * Fin;
      if (need_in || need_h) {
        GconvDgrad dg{};
        dg.G = dC, dg.R = int(R), dg.Nout = d.H, dg.W = params + P.Wc[ps];
        dg.M = d.M, dg.Fin = Fin, dg.Hd = d.H;
        dg.c_lo = need_in ? 0 : Fin, dg.c_hi = need_h ? C : Fin;
        dg.Tin = dTin, dg.tin_mstride = tin_ms, dg.acc_in = 0, dg.Th = dTH, dg.th_mstride = RH;
        CU(launch_gconv_dgrad(dg, s));
      }
      if (need_h) {
        AdjChain ch{dTH, RH, int64_t(d.B) * d.H, drH, 0, {tmp[0], tmp[1]}, {tmp[2], tmp[3]}};
        CU(diffuse_adj(g, d, &ch, 1, s));
      }
      CU(launch_gate_bwd(RH, d.H, need_h ? drH : nullptr, Hprev, r, u, dU,
                         need_h ? dHprev[l] : nullptr, dG, s));
      if (need_in || need_h) {
        GconvDgrad dg{};
        dg.G = dG, dg.R = int(R), dg.Nout = 2 * d.H, dg.W = params + P.Wru[ps];
        dg.M = d.M, dg.Fin = Fin, dg.Hd = d.H;
        dg.c_lo = need_in ? 0 : Fin, dg.c_hi = need_h ? C : Fin;
        dg.Tin = dTin, dg.tin_mstride = tin_ms, dg.acc_in = 1, dg.Th = dTH, dg.th_mstride = RH;
        CU(launch_gconv_dgrad(dg, s));
        AdjChain ch[2];
        int nch = 0;
        if (need_h)
          ch[nch++] = AdjChain{dTH, RH, int64_t(d.B) * d.H, dHprev[l], 1, {tmp[0], tmp[1]},
                               {tmp[2], tmp[3]}};
        if (need_in)  // to the layer below, or (decoder layer 0) to the previous prediction
          ch[nch++] = AdjChain{dTin, tin_ms, int64_t(d.B) * Fin,
                               l > 0 ? dHcur[l - 1] : Fp(Ly.dyhat) + int64_t(out_slot(t) - 1) * RFo,
                               1, {tmp[4], tmp[5]}, {tmp[6], tmp[7]}};
        CU(diffuse_adj(g, d, ch, nch, s));
      }
      std::swap(dHcur[l], dHprev[l]);
    }
  }

  // ------------------------------------------------------------------ weight gradients
  for (int ll = 0; ll < L * (d.model ? 2 : 1); ++ll) {
    const int l = ll % L, dec = ll >= L;
    const int t0 = dec ? T : 0, nt = dec ? d.T_out : T;
    const int Fin = l > 0 ? d.H : (dec ? d.F_out : d.F);
    GconvWgrad w{};
    if (l == 0) {
      w.in = dec ? Dy : Dx;
      w.in_tstride = dec ? M * RFo : RF;
      w.in_mstride = dec ? RFo : int64_t(T) * RF;
    } else {
      w.in = Fp(Ly.DH[l - 1]) + t0 * MRH, w.in_tstride = MRH, w.in_mstride = RH;
    }
    w.Fin = Fin, w.Hd = d.H, w.M = d.M, w.T = nt, w.R = int(R);
    w.partial = Fp(Ly.wpart), w.partial_cap = int64_t(Ly.wpart_floats);
    // r|u gate: Z_t = [in_t, H_{t-1}] (the decoder's first step reads the encoder's last state)
    if (dec)
      w.h = Fp(Ly.DH[l]) + (t0 - 1) * MRH, w.h_toff = 0;
    else
      w.h = Fp(Ly.DH[l]), w.h_toff = -1;
    w.h_tstride = MRH, w.h_mstride = RH;
    w.G = Fp(Ly.dG[l]) + t0 * 2 * RH, w.g_tstride = 2 * RH, w.Nout = 2 * d.H;
    w.out = grads + P.Wru[ll];
    CU(launch_gconv_wgrad(w, s));
    // candidate: Z'_t = [in_t, r*H_{t-1}]
    w.h = Fp(Ly.DrH[l]) + t0 * MRH, w.h_toff = 0;
    w.G = Fp(Ly.dC[l]) + t0 * RH, w.g_tstride = RH, w.Nout = d.H, w.out = grads + P.Wc[ll];
    CU(launch_gconv_wgrad(w, s));
  }
  SmallWgrad rw{};
  rw.mode = kSmallReadout, rw.T = d.T_out, rw.R = int(R);
  rw.dy = Fp(Ly.dyhat), rw.F_out = d.F_out;
  rw.G = Fp(Ly.DH[L - 1]) + int64_t(TT - d.T_out) * MRH, rw.g_tstride = MRH, rw.NG = d.H;
  rw.partial = Fp(Ly.wpart), rw.partial_cap = int64_t(Ly.wpart_floats), rw.out = grads + P.Wout;
  CU(launch_small_wgrad(rw, s));

  // ------------------------------------------------------------------ test-only dump
  if (act_dump) {
    for (int t = 0; t < TT; ++t)
      for (int l = 0; l < L; ++l) {
        float *dst = act_dump + (int64_t(t) * L + l) * 4 * RH;
        const float *src[4] = {Fp(Ly.DH[l]) + t * MRH, Fp(Ly.Rg[l]) + t * RH,
                               Fp(Ly.Ug[l]) + t * RH, Fp(Ly.Cg[l]) + t * RH};
        for (int q = 0; q < 4; ++q)
          CU(cudaMemcpyAsync(dst + q * RH, src[q], size_t(RH) * 4, cudaMemcpyDeviceToDevice, s));
      }
    CU(cudaMemcpyAsync(act_dump + int64_t(TT) * L * 4 * RH, Fp(Ly.yhat),
                       size_t(d.T_out) * R * d.F_out * 4, cudaMemcpyDeviceToDevice, s));
  }
  return PGTI_OK;
}

size_t workspace_for(const Dims &d) {
  return d.precision == 1 ? workspace_tc(d) : make_layout(d).total;
}

}  // namespace
}  // namespace detail
}  // namespace pgti

using namespace pgti;
using namespace pgti::detail;

extern "C" size_t pgti_dcrnn_desc_size(void) { return sizeof(pgti_dcrnn_desc); }

extern "C" size_t pgti_dcrnn_num_params(const pgti_dcrnn_desc *desc) {
  Dims d;
  if (check_desc(desc, &d) != PGTI_OK) return 0;
  return param_offsets(d).total;
}

extern "C" size_t pgti_dcrnn_workspace_bytes(const pgti_dcrnn_desc *desc) {
  Dims d;
  if (check_desc(desc, &d) != PGTI_OK) return 0;
  return workspace_for(d);
}

extern "C" pgti_status pgti_dcrnn_loss(const pgti_dcrnn_desc *desc, const float *params,
                                       const float *x, const float *y, float *loss_dev,
                                       void *workspace, size_t ws_bytes, void *stream) {
  clear_error();
  Dims d;
  PGTI_STATUS_TRY(check_desc(desc, &d));
  PGTI_REQUIRE(params && x && y && loss_dev && workspace, PGTI_ERR_INVALID_ARG,
               "pgti_dcrnn_loss: null pointer");
  PGTI_REQUIRE(aligned16(params) && aligned16(workspace), PGTI_ERR_ALIGNMENT,
               "pgti_dcrnn_loss: params / workspace must be 16-byte aligned");
  const size_t need = workspace_for(d);
  PGTI_REQUIRE(ws_bytes >= need, PGTI_ERR_WORKSPACE,
               "pgti_dcrnn_loss: workspace %zu bytes < %zu needed", ws_bytes, need);
  const WindowSrc xs{x, nullptr, 0, 0, 0, 0}, ys{y, nullptr, 0, 0, 0, 0};
  if (d.precision == 1)
    return run_step_tc(*desc, d, params, nullptr, xs, ys, loss_dev, static_cast<char *>(workspace),
                       nullptr, as_stream(stream));
  return run_step(*desc, d, params, nullptr, xs, ys, loss_dev, static_cast<char *>(workspace),
                  nullptr, as_stream(stream));
}

extern "C" pgti_status pgti_dcrnn_step(const pgti_dcrnn_desc *desc, const float *params,
                                       float *grads, const float *x, const float *y,
                                       float *loss_dev, void *workspace, size_t ws_bytes,
                                       float *act_dump, void *stream) {
  clear_error();
  Dims d;
  PGTI_STATUS_TRY(check_desc(desc, &d));
  PGTI_REQUIRE(params && grads && x && y && loss_dev && workspace, PGTI_ERR_INVALID_ARG,
               "pgti_dcrnn_step: null pointer");
  PGTI_REQUIRE(aligned16(params) && aligned16(grads) && aligned16(workspace), PGTI_ERR_ALIGNMENT,
               "pgti_dcrnn_step: params / grads / workspace must be 16-byte aligned");
  const size_t need = workspace_for(d);
  PGTI_REQUIRE(ws_bytes >= need, PGTI_ERR_WORKSPACE,
               "pgti_dcrnn_step: workspace %zu bytes < %zu needed", ws_bytes, need);
  const WindowSrc xs{x, nullptr, 0, 0, 0, 0}, ys{y, nullptr, 0, 0, 0, 0};
  if (d.precision == 1)
    return run_step_tc(*desc, d, params, grads, xs, ys, loss_dev, static_cast<char *>(workspace),
                       act_dump, as_stream(stream));
  return run_step(*desc, d, params, grads, xs, ys, loss_dev, static_cast<char *>(workspace),
                  act_dump, as_stream(stream));
}

extern "C" pgti_status pgti_dcrnn_step_indexed(const pgti_dcrnn_desc *desc, const float *params,
                                               float *grads, const pgti_series *series,
                                               const int32_t *dev_idx, float *loss_dev,
                                               void *workspace, size_t ws_bytes, float *act_dump,
                                               void *stream) {
  clear_error();
  Dims d;
  PGTI_STATUS_TRY(check_desc(desc, &d));
  PGTI_REQUIRE(params && grads && series && dev_idx && loss_dev && workspace,
               PGTI_ERR_INVALID_ARG, "pgti_dcrnn_step_indexed: null pointer");
  PGTI_REQUIRE(aligned16(params) && aligned16(grads) && aligned16(workspace), PGTI_ERR_ALIGNMENT,
               "pgti_dcrnn_step_indexed: params / grads / workspace must be 16-byte aligned");
  const float *buf = nullptr;
  int64_t row0 = 0, nrows = 0, N = 0, F = 0, ld = 0;
  series_view(series, &buf, &row0, &nrows, &N, &F, &ld);
  PGTI_REQUIRE(N == d.N && F == d.F && ld == d.ld, PGTI_ERR_SHAPE,
               "pgti_dcrnn_step_indexed: series N=%lld F=%lld ld=%lld vs desc N=%d F=%d ld=%lld",
               (long long)N, (long long)F, (long long)ld, d.N, d.F, (long long)d.ld);
  const size_t need = workspace_for(d);
  PGTI_REQUIRE(ws_bytes >= need, PGTI_ERR_WORKSPACE,
               "pgti_dcrnn_step_indexed: workspace %zu bytes < %zu needed", ws_bytes, need);
  const int span = d.T_in + d.T_out;
  const WindowSrc xs{buf, dev_idx, row0, nrows, 0, span}, ys{buf, dev_idx, row0, nrows, d.T_in, span};
  if (d.precision == 1)
    return run_step_tc(*desc, d, params, grads, xs, ys, loss_dev, static_cast<char *>(workspace),
                       act_dump, as_stream(stream));
  return run_step(*desc, d, params, grads, xs, ys, loss_dev, static_cast<char *>(workspace),
                  act_dump, as_stream(stream));
}

extern "C" pgti_status pgti_diffuse(const pgti_dcrnn_desc *desc, const float *X, int64_t W,
                                    float *out, void *stream) {
  clear_error();
  Dims d;
  PGTI_STATUS_TRY(check_desc(desc, &d));
  PGTI_REQUIRE(X && out && W > 0, PGTI_ERR_INVALID_ARG, "pgti_diffuse: bad arguments");
  cudaStream_t s = as_stream(stream);
  const int64_t NW = int64_t(d.N) * W;
  CU(cudaMemcpyAsync(out, X, size_t(NW) * 4, cudaMemcpyDeviceToDevice, s));
  CU(diffuse_fwd(*desc, d, out, NW, 1, 0, W, s));
  return PGTI_OK;
}

extern "C" pgti_status pgti_diffuse_adjoint(const pgti_dcrnn_desc *desc, const float *dT,
                                            int64_t W, float *dZ, void *stream) {
  clear_error();
  Dims d;
  PGTI_STATUS_TRY(check_desc(desc, &d));
  PGTI_REQUIRE(dT && dZ && W > 0, PGTI_ERR_INVALID_ARG, "pgti_diffuse_adjoint: bad arguments");
  cudaStream_t s = as_stream(stream);
  const int64_t NW = int64_t(d.N) * W;
  float *tmp = nullptr;
  CU(cudaMallocAsync(reinterpret_cast<void **>(&tmp), size_t(4 * NW) * 4, s));
  AdjChain ch{dT, NW, W, dZ, 0, {tmp, tmp + NW}, {tmp + 2 * NW, tmp + 3 * NW}};
  cudaError_t e = diffuse_adj(*desc, d, &ch, 1, s);
  cudaError_t e2 = cudaFreeAsync(tmp, s);
  CU(e);
  CU(e2);
  return PGTI_OK;
}
