// DIC preconditioner kernels — included by kernels.cu
// (same translation unit: shares the grid barrier / reduction helpers).
//
// OpenFOAM's DICPreconditioner is three sequential face loops over the
// upper-triangular face order (include/lfoam.h, LF_PRECOND_DIC):
//   calcReciprocalD  rD[u] -= upper_f^2 / rD[l]           (f ascending)
//   forward          w[u]  -= rD[u] upper_f w[l]           (f ascending)
//   backward         w[l]  -= rD[l] upper_f w[u]           (f descending)
// A cell's value is final once all its lower (forward) / upper (backward)
// neighbours are, so the loops parallelise over LEVELS: level(c) = 0 without
// lower neighbours, else 1 + max level of them.  Cells of one level are
// independent; levels are separated by grid barriers inside one persistent
// launch.  Each cell gathers its neighbours' contributions in exactly the
// sequential order (lower neighbours ascending = ascending face id; upper
// neighbours descending), with explicit _rn operations (no FMA), so rD and
// the preconditioned vector are bitwise those of the face loops.
//
// Level 0 needs no forward pass: its forward value is rD_c r_c, which the
// forward passes of higher levels recompute at the neighbour (bit L0 of the
// row label) from the not-yet-updated r and q — so a solve with L levels
// costs 2L-2 grid barriers per preconditioner application plus one for the
// Amul phase: 3 per iteration on a 2-colour numbering (renumber = 2).
//
// Row layout: full-row ELL (DicDev / LduDev.symU), every access coalesced;
// coefficients written by the assembly kernel.

#ifndef LF_DIC_TAIL
#define LF_DIC_TAIL 0    // 1: level passes and the Amul phase spread the tail trip (r2e:
#endif                   // neutral at 200^3, -2% at 100^3 -> off)
#ifndef LF_REV_ALIGN
#define LF_REV_ALIGN 0
#endif
#ifndef LF_DIC_REVERSE
#define LF_DIC_REVERSE 1  // 1: the 2-level forward sweep in reverse trip order (L2 reuse);
#endif                    // 2: every pass reversed on alternate iterations
#ifndef LF_DIC_STASH
#define LF_DIC_STASH 1   // L2-resident DIC solve keeps {q, rD} on chip (see k_pcg_dic)
#endif
#ifndef LF_DIC_STASH_DIAG
#define LF_DIC_STASH_DIAG 0  // ... and diag (phase 1 reads it from the stash after iteration 0)
#endif
#ifndef LF_DIC_LPF
#define LF_DIC_LPF 0  // HBM-bound variant (two contiguous levels): next-trip L2 prefetch of the
#endif                // own-cell streams of the Amul phase and both sweeps when ws.l2pf.
                      // Measured r6l (forced on): 200^3 37.9 -> 42.0 ms/step, 400^3 585 -> 721 ms
                      // (the pair-mode passes' L2 working set cannot take another trip): off
#ifndef LF_DIC_PAIR
#define LF_DIC_PAIR 1    // phase 1 interleaves the two colours (thread t: cell t of each) in the
#endif                   // HBM-bound variant (r1x: 200^3 39.2 vs 39.9 ms/step; 100^3 3.37 vs 3.13)

// Grid-stride loop over [t0, t1) with the evenly spread tail trip of the
// persistent kernels (LF_TAIL): full trips while every thread has an index,
// then the leftover indices split into equal consecutive runs per block.
template <class F>
__device__ __forceinline__ void grid_range(int t0, int t1, F body) {
  const int S = gridDim.x * blockDim.x, len = t1 - t0;
  const int first = t0 + (int)(blockIdx.x * blockDim.x + threadIdx.x);
#if LF_TAIL && LF_DIC_TAIL
  const int nFull = len / S;
  for (int i = 0; i < nFull; ++i) body(first + i * S);
  const int R = len - nFull * S, per = (R + (int)gridDim.x - 1) / (int)gridDim.x;
  const int off = (int)blockIdx.x * per + (int)threadIdx.x;
  if ((int)threadIdx.x < per && off < R) body(t0 + nFull * S + off);
#else
  for (int t = first; t < t1; t += S) body(t);
#endif
}

// The same trips in reverse order (the last trip first): a pass that
// starts where the previous one ended finds that pass's lines still in L2.
template <class F>
__device__ __forceinline__ void grid_range_rev(int t0, int t1, F body) {
  const int S = gridDim.x * blockDim.x;
  const int first = t0 + (int)(blockIdx.x * blockDim.x + threadIdx.x);
#if LF_REV_ALIGN
  // the same trip index in every thread
  for (int i = (t1 - t0 + S - 1) / S - 1; i >= 0; --i) {
    const int t = first + i * S;
    if (t < t1) body(t);
  }
#else
  // each thread starts at its own last index (threads past the end of the
  // partial last trip start one trip lower)
  if (first >= t1) return;
  for (int t = first + ((t1 - 1 - first) / S) * S; t >= t0; t -= S) body(t);
#endif
}

template <int KS>
struct SymRow {
  int lab[KS];
  double u[KS];
};

template <int KS>
__device__ __forceinline__ void load_row(const DicDev &d, const LduDev &a, int c, SymRow<KS> &R) {
#pragma unroll
  for (int k = 0; k < KS; ++k) {
    R.lab[k] = __ldg(d.symN + k * d.ldS + c);
    R.u[k] = __ldg(a.symU + k * d.ldS + c);
  }
}

__device__ __forceinline__ int sym_cell(int lab) { return lab & (DIC_L0BIT - 1); }

// calcReciprocalD for a cell on level >= 1 (its lower neighbours are final)
template <int KS>
__device__ __forceinline__ double dic_factor_cell(const DicDev &d, const LduDev &a, int c) {
  SymRow<KS> R;
  load_row<KS>(d, a, c, R);
  double rdu = a.diag[c];
#pragma unroll
  for (int k = 0; k < KS; ++k) {
    const int lab = R.lab[k];
    if (lab >= 0 && sym_cell(lab) < c) {
      const int j = sym_cell(lab);
      const double dj = (lab & DIC_L0BIT) ? a.diag[j] : d.rDu[j];
      rdu = __dsub_rn(rdu, __ddiv_rn(__dmul_rn(R.u[k], R.u[k]), dj));
    }
  }
  d.rDu[c] = rdu;
  const double rd = __ddiv_rn(1.0, rdu);
  d.rD[c] = rd;
  return rd;
}

// r of a cell after this iteration's update (upd) — identical operation
// wherever it is evaluated
__device__ __forceinline__ double r_new(const double *r, const double *q, bool upd, double alpha, int j) {
  return upd ? fma(-alpha, q[j], r[j]) : r[j];
}

// Forward pass of a cell on level >= 1.  Writes r (upd) and the forward w;
// returns r_c.
template <int KS>
__device__ __forceinline__ double dic_forward_cell(const DicDev &d, const LduDev &a, int c, double *r,
                                                   const double *q, double *w, bool upd, double alpha,
                                                   double &wOut, const double2 *own = nullptr) {
  // own: {q_c, rD_c} from the shared-memory stash instead of global memory
  SymRow<KS> R;
  load_row<KS>(d, a, c, R);
  const double rc = own ? (upd ? fma(-alpha, own->x, r[c]) : r[c]) : r_new(r, q, upd, alpha, c);
  if (upd) r[c] = rc;
  const double rd = own ? own->y : d.rD[c];
  double wv = __dmul_rn(rd, rc);
#pragma unroll
  for (int k = 0; k < KS; ++k) {
    const int lab = R.lab[k];
    if (lab >= 0 && sym_cell(lab) < c) {
      const int j = sym_cell(lab);
      const double wj = (lab & DIC_L0BIT) ? __dmul_rn(d.rD[j], r_new(r, q, upd, alpha, j)) : w[j];
      wv = __dsub_rn(wv, __dmul_rn(__dmul_rn(rd, R.u[k]), wj));
    }
  }
  w[c] = wv;
  wOut = wv;
  return rc;
}

// Backward pass of a cell on level l (l == 0: r update and forward value
// here).  Writes the final w; returns r_c.
template <int KS>
__device__ __forceinline__ double dic_backward_cell(const DicDev &d, const LduDev &a, int c, bool level0,
                                                    double *r, const double *q, double *w, bool upd,
                                                    double alpha, double &wOut, const double2 *own = nullptr) {
  SymRow<KS> R;
  load_row<KS>(d, a, c, R);
  const double rd = own ? own->y : d.rD[c];
  double rc, wv;
  if (level0) {
    rc = own ? (upd ? fma(-alpha, own->x, r[c]) : r[c]) : r_new(r, q, upd, alpha, c);
    if (upd) r[c] = rc;
    wv = __dmul_rn(rd, rc);
  } else {
    rc = r[c];
    wv = w[c];
  }
#pragma unroll
  for (int k = KS - 1; k >= 0; --k) {
    const int lab = R.lab[k];
    if (lab >= 0 && sym_cell(lab) > c)
      wv = __dsub_rn(wv, __dmul_rn(__dmul_rn(rd, R.u[k]), w[sym_cell(lab)]));
  }
  w[c] = wv;
  wOut = wv;
  return rc;
}

__device__ __forceinline__ int level_cell(const DicDev &d, int t) { return d.contig ? t : __ldg(d.lvlCells + t); }

// One application of the preconditioner inside the persistent kernel (upd:
// fused r -= alpha q), ending in the reducing barrier that publishes
// {sum|r|, sum w.r} to out[0..1].  HALO: each final w of a cell with
// processor faces is stored into the neighbour ranks' recvW (peer memory),
// ordered before the reduction's cross-rank exchange; the factor and the
// sweeps themselves are processor-local, as OpenFOAM's DIC (reading A42).
template <int KS, bool HALO, class Idle = NoIdle>
__device__ __forceinline__ void dic_apply(const MeshDev &m, const DicDev &d, const LduDev &a, double *r,
                                          const double *q, double *w, bool upd, double alpha, unsigned *bar,
                                          double *partials, double *out, const P2PDev &pp,
                                          Idle idle = Idle(), bool odd = false, const double2 *stash = nullptr,
                                          int n = 0, const PfSet *pfs = nullptr) {
  const int L = d.L;
  double v[2] = {0.0, 0.0};
  if (stash) {
    // two contiguous levels, each thread's cells at the Amul-phase mapping
    // c = gtid + i*S with {q, rD} of trip i in stash[i*BS + tid]
    const int S = gridDim.x * blockDim.x, gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const int T = (n + S - 1) / S, n0 = __ldg(d.lvlStart + 1);
    for (int i = T - 1; i >= 0; --i) {  // forward sweep of level 1, backwards (L2 reuse)
      const int c = gtid + i * S;
      if (c >= n0 && c < n) {
        double wc;
        const double rc = dic_forward_cell<KS>(d, a, c, r, q, w, upd, alpha, wc, &stash[i * BS + threadIdx.x]);
        v[0] += fabs(rc);
        v[1] = fma(wc, rc, v[1]);
        if (HALO && pp.P > 0) push_halo<HALO_W>(m, pp, c, wc);
      }
    }
    grid_barrier(bar);
    for (int i = 0; i < T; ++i) {  // backward sweep of level 0
      const int c = gtid + i * S;
      if (c < n0) {
        double wc;
        const double rc = dic_backward_cell<KS>(d, a, c, true, r, q, w, upd, alpha, wc, &stash[i * BS + threadIdx.x]);
        v[0] += fabs(rc);
        v[1] = fma(wc, rc, v[1]);
        if (HALO && pp.P > 0) push_halo<HALO_W>(m, pp, c, wc);
      }
    }
    grid_reduce_sync<2, HALO>(v, partials, bar, out, pp LF_DBG_ARG(0), idle);
    return;
  }
  const int S = gridDim.x * blockDim.x, lane = threadIdx.x & 31;
  for (int l = 1; l < L; ++l) {
    const int t0 = __ldg(d.lvlStart + l), t1 = __ldg(d.lvlStart + l + 1);
    const bool rev = LF_DIC_REVERSE && L == 2 && !odd;
    auto fwd = [&](int t) {
      if (pfs) {  // the warp's run of the next trip (contiguous levels)
        const int nb = t - lane + (rev ? -S : S);
        if (nb >= t0 && nb < t1) pf_run(*pfs, nb);
      }
      const int c = level_cell(d, t);
      double wc;
      const double rc = dic_forward_cell<KS>(d, a, c, r, q, w, upd, alpha, wc);
      v[0] += fabs(rc);
      if (l == L - 1) {  // no upper neighbours: final
        v[1] = fma(wc, rc, v[1]);
        if (HALO && pp.P > 0) push_halo<HALO_W>(m, pp, c, wc);
      }
    };
    // two levels (LF_DIC_REVERSE): every pass starts where the previous one
    // ended — even iterations: Amul forwards, this pass backwards, the
    // backward pass forwards; odd iterations the mirror image
    if (rev)
      grid_range_rev(t0, t1, fwd);
    else
      grid_range(t0, t1, fwd);
    grid_barrier(bar);
  }
  for (int l = L >= 2 ? L - 2 : 0; l >= 0; --l) {
    const int t0 = __ldg(d.lvlStart + l), t1 = __ldg(d.lvlStart + l + 1);
    const bool rev = LF_DIC_REVERSE == 2 && L == 2 && odd;
    auto bwd = [&](int t) {
      if (pfs) {
        const int nb = t - lane + (rev ? -S : S);
        if (nb >= t0 && nb < t1) pf_run(*pfs, nb);
      }
      const int c = level_cell(d, t);
      double wc;
      const double rc = dic_backward_cell<KS>(d, a, c, l == 0, r, q, w, upd, alpha, wc);
      if (l == 0) v[0] += fabs(rc);
      v[1] = fma(wc, rc, v[1]);
      if (HALO && pp.P > 0) push_halo<HALO_W>(m, pp, c, wc);
    };
    if (rev)
      grid_range_rev(t0, t1, bwd);
    else
      grid_range(t0, t1, bwd);
    if (l > 0) grid_barrier(bar);
  }
  grid_reduce_sync<2, HALO>(v, partials, bar, out, pp LF_DBG_ARG(0), idle);
}

// Phase-1 work of one cell in the DIC solve: deferred psi update, p = w +
// beta p_old, q = A p over the full row (ascending neighbour label = the
// order of lduMatrix::Amul's face loop) minus the processor-interface term
// (HALO: halo p recomputed from the neighbour's w), partial sums {p.q, psi}.
template <int KS, bool HALO>
__device__ __forceinline__ void dic_amul_cell(const MeshDev &m, const LduDev &a, const DicDev &d,
                                              const Workspace &ws, int k, int c, bool first, bool cont,
                                              double alpha, double beta, double *psi, const double *w,
                                              const double *pold, double *pnew, double *q, double (&v1)[2],
                                              bool idleF, double *qOut = nullptr, bool writeQ = true,
                                              double *dSlot = nullptr) {
  if (idleF) {  // psi was updated in the previous beta-barrier wait
    if (first) v1[1] += psi[c];
  } else {
    double ps = psi[c];
    if (!first) {
      ps = fma(alpha, pold[c], ps);
      psi[c] = ps;
    }
    v1[1] += ps;
  }
  if (cont) {
    SymRow<KS> R;
    load_row<KS>(d, a, c, R);
    const double pc = first ? w[c] : fma(beta, pold[c], w[c]);
    pnew[c] = pc;
    double pn[KS];
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
      const int j = sym_cell(R.lab[kk]);
      pn[kk] = R.lab[kk] >= 0 ? (first ? w[j] : fma(beta, pold[j], w[j])) : 0.0;
    }
    double dc;
    if (dSlot) {  // stashed diag: global on the first iteration only
      if (first) *dSlot = a.diag[c];
      dc = *dSlot;
    } else {
      dc = a.diag[c];
    }
    double qc = dc * pc;
#pragma unroll
    for (int kk = 0; kk < KS; ++kk)
      if (R.lab[kk] >= 0) qc = fma(R.u[kk], pn[kk], qc);
    if (HALO) qc -= row_proc_p(m, a.bBnd, ws, first, beta, k, c);
    if (writeQ) q[c] = qc;
    if (qOut) *qOut = qc;
    v1[0] = fma(pc, qc, v1[0]);
  }
}

// ------------------------------------------------ persistent DIC PCG solve
// The diagonal persistent kernel's state machine (k_pcg_persistent) with
// the preconditioner application replaced by the level sweeps:
//   set-up:    DIC factor (L-1 passes), w = M^-1 r (2L-2 barriers), sum w.r
//   iteration: phase 1 (p, q = A p over full rows, sum p.q, deferred psi)
//              | r -= alpha q fused into the sweeps, w = M^-1 r, sum|r|, sum w.r
// HALO: processor patches through the peer-memory transport (halo w puts in
// the sweeps, halo p recomputed in the Amul phase, rank-ordered mailbox
// allreduce in the two reducing barriers), as k_pcg_persistent<.., true>.
template <int KS, bool HALO, bool IDLE = false>
__global__ void __launch_bounds__(BS, LF_MINB_P)
    k_pcg_dic(MeshDev m, LduDev a, DicDev d, Workspace ws, unsigned *bar) {
  PcgCtl *ctl = ws.ctl;
  if (ctl->stop) return;
  const P2PDev &pp = ws.p2p;  // P == 0 unless HALO with the peer-memory transport
  struct St {
    double nf, initRes, finRes, wArA, alpha, beta;
    int k, cont, singular;
  };
  __shared__ St st;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
  const int L = d.L;
  // two contiguous colours: interleave them in phase 1 (HBM-bound variant only)
  const bool pair = LF_DIC_PAIR && !IDLE && d.contig && L == 2;
  const bool idleF = IDLE;  // psi flush in the beta-barrier wait (Workspace.idleFlush)
  double psiSum = 0.0;
  double *psi = ctl->psi;
  double *r = ws.r, *w = ws.w, *q = ws.q;
  // L2-resident variant, two contiguous levels, <= LF_STASH_TRIPS trips per
  // thread (LF_DIC_STASH): {q, rD} of the thread's cells stay in shared
  // memory (slot = trip of the Amul-phase mapping c = gtid + i*S) — q of
  // level-1 cells is never written to global memory and the sweeps read
  // their own q and rD on chip
  extern __shared__ double2 lf_dstash[];
  double *lf_ddiag = reinterpret_cast<double *>(lf_dstash + LF_STASH_TRIPS * BS);  // LF_DIC_STASH_DIAG
  const int nTrips = (m.n + stride - 1) / stride;
  const bool stash = LF_DIC_STASH && IDLE && d.contig && L == 2 && nTrips <= LF_STASH_TRIPS;
  const int n0s = stash ? __ldg(d.lvlStart + 1) : 0;
  // next-trip L2 prefetch (HBM-bound variant, two contiguous levels)
  const bool dpf = LF_DIC_LPF && pair && ws.l2pf;
  __shared__ PfSet pfA, pfS;  // Amul phase (rebuilt per iteration: p_old), sweeps
  if (dpf && threadIdx.x == 0) {
    pfS.clear();
    for (int kk = 0; kk < KS; ++kk) pfS.addI(d.symN + kk * d.ldS);
    for (int kk = 0; kk < KS; ++kk) pfS.addD(a.symU + kk * d.ldS);
    pfS.addD(r);
    pfS.addD(q);
    pfS.addD(d.rD);
  }

  if (threadIdx.x == 0) {
    st.k = ctl->it;
    st.nf = ctl->normFactor;
    st.initRes = ctl->initRes;
    st.finRes = ctl->finRes;
    st.wArA = ctl->wArA;
    st.alpha = ctl->alpha;
    st.singular = 0;
    // OpenFOAM: iterate if minIter > 0 || !checkConvergence (set-up sums)
    st.nf = __ldcg(&ws.gsum->setup[0]) + 1e-20;
    st.initRes = __ldcg(&ws.gsum->setup[1]) / st.nf;
    st.finRes = st.initRes;
    st.cont = ctl->minIter > 0 || !conv(st.finRes, st.initRes, ctl);
  }
  __syncthreads();
  if (st.cont && stash) {
    // calcReciprocalD of both levels in one pass at the Amul-phase mapping
    // (level 1 reads only diag of its level-0 neighbours), rD stashed
    for (int i = 0; i < nTrips; ++i) {
      const int c = gtid + i * stride;
      if (c < m.n) {
        double rd;
        if (c < n0s) {
          rd = __ddiv_rn(1.0, a.diag[c]);
          d.rD[c] = rd;
        } else {
          rd = dic_factor_cell<KS>(d, a, c);
        }
        lf_dstash[i * BS + threadIdx.x].y = rd;
      }
    }
    grid_barrier(bar);
    dic_apply<KS, HALO>(m, d, a, r, q, w, false, 0.0, bar, ws.partials, ws.gsum->p2, pp, NoIdle(), false,
                        lf_dstash, m.n);  // set-up w (q unused)
  } else if (st.cont) {
    // ---- calcReciprocalD: levels 0 and 1 in one pass (level 1 reads only
    // diag of level-0 cells), then one pass per level
    for (int l = 0; l < L; ++l) {
      if (l >= 2) grid_barrier(bar);
      grid_range(__ldg(d.lvlStart + l), __ldg(d.lvlStart + l + 1), [&](int t) {
        const int c = level_cell(d, t);
        if (l == 0)
          d.rD[c] = __ddiv_rn(1.0, a.diag[c]);
        else
          dic_factor_cell<KS>(d, a, c);
      });
    }
    grid_barrier(bar);
    dic_apply<KS, HALO>(m, d, a, r, q, w, false, 0.0, bar, ws.partials, ws.gsum->p2, pp);  // set-up w
  }
  for (;;) {
    if (threadIdx.x == 0) {
      if (st.k == 0) {
        st.wArA = st.cont ? __ldcg(&ws.gsum->p2[1]) : 0.0;
        st.beta = 0.0;
      } else {
        st.finRes = __ldcg(&ws.gsum->p2[0]) / st.nf;
        st.cont = (st.k < ctl->maxIter && !conv(st.finRes, st.initRes, ctl)) || st.k < ctl->minIter;
        const double wn = __ldcg(&ws.gsum->p2[1]);
        st.beta = wn / st.wArA;
        st.wArA = wn;
      }
      if (dpf) {
        pfA.clear();
        for (int kk = 0; kk < KS; ++kk) pfA.addI(d.symN + kk * d.ldS);
        for (int kk = 0; kk < KS; ++kk) pfA.addD(a.symU + kk * d.ldS);
        pfA.addD(psi);
        pfA.addD(w);
        pfA.addD(a.diag);
        if (st.k > 0) pfA.addD((st.k & 1) ? ws.p[0] : ws.p[1]);  // p_old
      }
    }
    __syncthreads();
    const int k = st.k;
    const bool first = (k == 0), cont = st.cont != 0;
    const double beta = st.beta, alpha = st.alpha;
    const double *pold = (k & 1) ? ws.p[0] : ws.p[1];
    double *pnew = (k & 1) ? ws.p[1] : ws.p[0];
    // ---- phase 1: flush psi, p = w + beta p_old, q = A p (full rows), sums.
    // With two contiguous levels (multicolour numbering) thread t may handle
    // cell t of each colour together (LF_DIC_PAIR), so a cell's gathers hit
    // the lines its partner-colour neighbours just read.
    double v1[2] = {0.0, 0.0};
    if (idleF) v1[1] = psiSum;
    const bool odd = LF_DIC_REVERSE == 2 && L == 2 && (k & 1);  // walk backwards on odd iterations
    if (pair) {
      const int n0 = __ldg(d.lvlStart + 1), n1 = m.n - n0, nt = max(n0, n1);
      auto two = [&](int t) {
        if (t < n0)
          dic_amul_cell<KS, HALO>(m, a, d, ws, k, t, first, cont, alpha, beta, psi, w, pold, pnew, q, v1, false);
        if (t < n1)
          dic_amul_cell<KS, HALO>(m, a, d, ws, k, n0 + t, first, cont, alpha, beta, psi, w, pold, pnew, q, v1,
                                  false);
      };
      if (odd)
        grid_range_rev(0, nt, two);
      else
        for (int t = gtid; t < nt; t += stride) {
          if (dpf) {  // both colours' runs of the next trip
            const int nb = t - (int)(threadIdx.x & 31) + stride;
            if (nb < n0) pf_run(pfA, nb);
            if (nb < n1) pf_run(pfA, n0 + nb);
          }
          two(t);
        }
    } else if (stash) {
      for (int i = 0; i < nTrips; ++i) {
        const int c = gtid + i * stride;
        if (c < m.n) {
          double qc;
          dic_amul_cell<KS, HALO>(m, a, d, ws, k, c, first, cont, alpha, beta, psi, w, pold, pnew, q, v1, idleF,
                                  &qc, c < n0s,  // level-0 q is read by neighbours: global
                                  LF_DIC_STASH_DIAG ? lf_ddiag + i * BS + threadIdx.x : nullptr);
          if (cont) lf_dstash[i * BS + threadIdx.x].x = qc;
        }
      }
    } else {
      auto one = [&](int c) {
        dic_amul_cell<KS, HALO>(m, a, d, ws, k, c, first, cont, alpha, beta, psi, w, pold, pnew, q, v1, idleF);
      };
      if (odd)
        grid_range_rev(0, m.n, one);
      else
        grid_range(0, m.n, one);
    }
    grid_reduce_sync<2, HALO>(v1, ws.partials, bar, ws.gsum->p1, pp LF_DBG_ARG(0));
    if (!cont) break;
    if (threadIdx.x == 0) {
      const double pq = __ldcg(&ws.gsum->p1[0]);
      st.singular = fabs(pq) / st.nf < 1e-300;
      if (!st.singular) st.alpha = st.wArA / pq;
    }
    __syncthreads();
    if (st.singular) break;
    // ---- r -= alpha q, w = M^-1 r, sum|r|, sum w.r
    // idleF: psi += alpha_k p_k for this thread's phase-1 cells while the
    // block waits for beta (as k_pcg_persistent)
    psiSum = 0.0;
    const double alphaK = st.alpha;
    auto flush = [&]() {
      if (!idleF) return;
      grid_range(0, m.n, [&](int c) {
        const double ps = fma(alphaK, pnew[c], psi[c]);
        psi[c] = ps;
        psiSum += ps;
      });
    };
    dic_apply<KS, HALO>(m, d, a, r, q, w, true, alphaK, bar, ws.partials, ws.gsum->p2, pp, flush,
                        LF_DIC_REVERSE == 2 && L == 2 && (st.k & 1), stash ? lf_dstash : nullptr, m.n,
                        dpf ? &pfS : nullptr);
    if (threadIdx.x == 0) ++st.k;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctl->it = st.k;
    ctl->stop = 1;
    ctl->singular = st.singular;
    ctl->converged = conv(st.finRes, st.initRes, ctl) ? 1 : 0;
    ctl->normFactor = st.nf;
    ctl->initRes = st.initRes;
    ctl->finRes = st.finRes;
    ctl->wArA = st.wArA;
    ctl->alpha = st.alpha;
  }
}

template <bool HALO, bool IDLE = false>
static const void *dic_fn(int KS) {
  return KS <= 6 ? (const void *)k_pcg_dic<6, HALO, IDLE> : (const void *)k_pcg_dic<8, HALO, IDLE>;
}

static size_t dic_stash_bytes() {
  return stash_bytes() + (LF_DIC_STASH_DIAG ? (size_t)LF_STASH_TRIPS * BS * sizeof(double) : 0);
}

int dic_grid(int device, int KS) {
  int sms = 0, best = 1 << 30;
  LF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  for (const void *fn : {dic_fn<false>(KS), dic_fn<true>(KS), dic_fn<false, true>(KS), dic_fn<true, true>(KS)}) {
    int nb = 0;  // co-resident for all variants; the L2 ones carry the stash
    const size_t sm = (fn == dic_fn<false, true>(KS) || fn == dic_fn<true, true>(KS)) ? dic_stash_bytes() : 0;
    if (sm) LF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    LF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, BS, sm));
    best = std::min(best, nb);
  }
  return sms * (best < 1 ? 1 : best);
}

void launch_pcg_dic(cudaStream_t s, int grid, const MeshDev &m, const LduDev &a, const DicDev &d,
                    const Workspace &ws, unsigned *bar) {
  void *args[] = {(void *)&m, (void *)&a, (void *)&d, (void *)&ws, (void *)&bar};
  const bool halo = m.hasProc || ws.p2p.P > 0;
  const bool idle = LF_IDLE_FLUSH && ws.idleFlush;  // L2-resident variant, single rank or halo
  const void *fn = halo ? (idle ? dic_fn<true, true>(d.KS) : dic_fn<true>(d.KS))
                        : (idle ? dic_fn<false, true>(d.KS) : dic_fn<false>(d.KS));
  // the diag slots follow LF_STASH_TRIPS full {q, rD} rows: fit only without them
  const size_t smem = LF_DIC_STASH_DIAG ? dic_stash_bytes() : stash_fit(m.n, grid, sizeof(double2));
  LF_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(BS), args, idle ? smem : 0, s));
}

// ------------------------------------------- full-row coefficients (fill)
// symU from upper for a system assembled before the DIC rows existed (the
// assembly kernel writes them directly afterwards).  Slot order: the
// neighbour-side faces (losort order), then the owned faces.
__global__ void k_sym_fill(MeshDev m, LduDev a) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < m.n; c += gridDim.x * blockDim.x) {
    const int l0 = m.losortStart[c], l1 = m.losortStart[c + 1];
    const int o0 = m.ownerStart[c], o1 = m.ownerStart[c + 1];
    for (int j = l0; j < l1; ++j) a.symU[(j - l0) * a.ldS + c] = a.upper[m.losort[j]];
    for (int i = o0; i < o1; ++i) a.symU[((l1 - l0) + (i - o0)) * a.ldS + c] = a.upper[i];
  }
}

void launch_sym_fill(cudaStream_t s, const Launch &L, const MeshDev &m, const LduDev &a) {
  k_sym_fill<<<L.grid, BS, 0, s>>>(m, a);
}

// ------------------------------------------------ standalone level passes
template <int KS>
__global__ void k_dic_factor_level(LduDev a, DicDev d, int l) {
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
  const int lo = l, hi = l == 0 ? min(1, d.L - 1) : l;
  for (int ll = lo; ll <= hi; ++ll) {
    const int t1 = d.lvlStart[ll + 1];
    for (int t = d.lvlStart[ll] + gtid; t < t1; t += stride) {
      const int c = level_cell(d, t);
      if (ll == 0)
        d.rD[c] = __ddiv_rn(1.0, a.diag[c]);
      else
        dic_factor_cell<KS>(d, a, c);
    }
  }
}

template <int KS>
__global__ void k_dic_sweep_level(LduDev a, DicDev d, int l, int forward, const double *r, double *w) {
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
  const int t1 = d.lvlStart[l + 1];
  for (int t = d.lvlStart[l] + gtid; t < t1; t += stride) {
    const int c = level_cell(d, t);
    double wc;
    // r is read only (no update): the const_cast is never written through
    if (forward)
      dic_forward_cell<KS>(d, a, c, const_cast<double *>(r), nullptr, w, false, 0.0, wc);
    else
      dic_backward_cell<KS>(d, a, c, l == 0, const_cast<double *>(r), nullptr, w, false, 0.0, wc);
  }
}

void launch_dic_factor_level(cudaStream_t s, const Launch &L, const MeshDev &m, const LduDev &a,
                             const DicDev &d, int l) {
  (void)m;
  if (d.KS <= 6)
    k_dic_factor_level<6><<<L.grid, BS, 0, s>>>(a, d, l);
  else
    k_dic_factor_level<8><<<L.grid, BS, 0, s>>>(a, d, l);
}

void launch_dic_sweep_level(cudaStream_t s, const Launch &L, const MeshDev &m, const LduDev &a,
                            const DicDev &d, int l, bool forward, const double *r, double *w) {
  (void)m;
  if (d.KS <= 6)
    k_dic_sweep_level<6><<<L.grid, BS, 0, s>>>(a, d, l, forward ? 1 : 0, r, w);
  else
    k_dic_sweep_level<8><<<L.grid, BS, 0, s>>>(a, d, l, forward ? 1 : 0, r, w);
}

// diagonalPreconditioner: w = (1/diag) r (rD = 1/diag, then rD*r, as
// OpenFOAM); r == null: w = rD
__global__ void k_diag_precondition(int32_t n, const double *__restrict__ diag, const double *__restrict__ r,
                                    double *__restrict__ w) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x)
    w[c] = r ? (1.0 / diag[c]) * r[c] : 1.0 / diag[c];
}

void launch_diag_precondition(cudaStream_t s, const Launch &L, int32_t n, const double *diag,
                              const double *r, double *w) {
  k_diag_precondition<<<L.grid, BS, 0, s>>>(n, diag, r, w);
}
