// GAMG preconditioner kernels (§7 names AMG "a
// better alternative"; the algorithm is reading A43 in DESIGN.md) — included
// by kernels.cu (same translation unit: grid barrier / reduction helpers,
// the DIC full rows and the DIC kernel's Amul phase).
//
// One application w = M^-1 r is a symmetric V-cycle from a zero guess:
//   b_0 = r
//   l = 0..L-1:  x_l = omega rD_l b_l;  b_{l+1} = P^T (b_l - A_l x_l)
//   x_L = A_L^-1 b_L                      (dense inverse of the coarsest level)
//   l = L-1..0:  z = x_l + P x_{l+1};  x_l = z + omega rD_l (b_l - A_l z)
//   w = x_0
// with the Galerkin coarse matrices A_{l+1} = P^T A_l P of the current
// system formed at the start of every solve (as OpenFOAM agglomerates the
// matrix per solve).  Parallel form:
//   * a DOWN pass runs over the coarse cells I of level l+1: each sums, over
//     its members c (ascending), b_c - (A_l x_l)_c, where x_l at c and at
//     c's neighbours is recomputed as omega rD b (bitwise the same value
//     wherever it is formed) — no pass writes x_l, no barrier between the
//     smoothing, the residual and the restriction;
//   * an UP pass runs over the cells of level l: z at the cell and at its
//     neighbours is recomputed as omega rD b + x_{l+1}[agg], then the post-
//     smoothing sweep writes x_l;
//   * levels with at most 4096 cells (GamgDev.tail; env LF_GAMG_TAIL) and
//     the coarsest solve run in ONE block with __syncthreads between passes:
//     the small levels cost no grid barriers.  Per V-cycle: 2 t + 1 grid barriers, t = levels above
//     the tail (t = 3-4 at 200^3).
// Every product and sum is an explicit _rn operation in the oracle's order
// (rows in ascending neighbour label = the face loop of lduMatrix::Amul;
// members, internal faces and fine faces ascending), so the coarse
// matrices, the coarsest inverse and one application are BITWISE the
// oracle's (tests/test_gpu_gamg.py).

constexpr double GAMG_OMEGA = 0.9;  // reading A43
#ifndef LF_GAMG_TIMING
#define LF_GAMG_TIMING 0  // 1: block 0 prints the pass boundaries of iteration 5 (debug builds)
#endif
#if LF_GAMG_TIMING
__device__ unsigned long long g_gt[128];
__device__ int g_gtn, g_gton;
#define GT()                                                                       \
  do {                                                                             \
    if (blockIdx.x == 0 && threadIdx.x == 0 && g_gton && g_gtn < 128) g_gt[g_gtn++] = gtime_ns(); \
  } while (0)
#else
#define GT() \
  do {       \
  } while (0)
#endif
#ifndef LF_GAMG_QREC
#define LF_GAMG_QREC 1  // phase 1 forms q = A p by the recurrence A w + beta q_old (see LF_QREC)
#endif

// level-0 row: y += U x_j over the cell's neighbours in ascending label with
// explicit _rn operations.  RW > 0: the half-ELL slices (lower neighbours in
// the loE slots — ascending owner — then upper neighbours in the nbrE slots;
// the lower side's coefficient is re-read from its owner's slot); RW < 0:
// the full-row ELL (DIC rows, -RW slots, already ascending).
template <int RW, class XF>
__device__ __forceinline__ double gamg_row0(const MeshDev &m, const LduDev &a, int c, double y, XF xf) {
  if constexpr (RW < 0) {
    constexpr int KS = -RW;
    int lab[KS];
    double u[KS], x[KS];
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      lab[k] = __ldg(m.symN + k * m.ldS + c);
      u[k] = __ldg(a.symU + k * m.ldS + c);
    }
#pragma unroll
    for (int k = 0; k < KS; ++k) x[k] = lab[k] >= 0 ? xf(sym_cell(lab[k])) : 0.0;
#pragma unroll
    for (int k = 0; k < KS; ++k)
      if (lab[k] >= 0) y = __dadd_rn(y, __dmul_rn(u[k], x[k]));
    return y;
  } else {
    const int n = m.ldE;
    int lo[RW], nb[RW];
    double uo[RW], lu[RW], lx[RW], ox[RW];
#pragma unroll
    for (int k = 0; k < RW; ++k) {
      lo[k] = __ldg(m.loE + k * n + c);
      nb[k] = __ldg(m.nbrE + k * n + c);
      uo[k] = a.upperE[k * n + c];
    }
#pragma unroll
    for (int k = 0; k < RW; ++k) {
      const int oc = lo[k] & ELL_MASK;
      lu[k] = lo[k] >= 0 ? a.upperE[(lo[k] >> ELL_SHIFT) * n + oc] : 0.0;
      lx[k] = lo[k] >= 0 ? xf(oc) : 0.0;
      ox[k] = nb[k] >= 0 ? xf(nb[k]) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < RW; ++k)
      if (lo[k] >= 0) y = __dadd_rn(y, __dmul_rn(lu[k], lx[k]));
#pragma unroll
    for (int k = 0; k < RW; ++k)
      if (nb[k] >= 0) y = __dadd_rn(y, __dmul_rn(uo[k], ox[k]));
    return y;
  }
}

// coarse-level row (CSR, ascending neighbour label): the products of a
// chunk of 8 entries are formed with their loads in flight together, then
// added in order (the sum stays the sequential one)
template <class XF>
__device__ __forceinline__ double gamg_rowc(const GamgLevelDev &L, int c, double y, XF xf) {
  constexpr int B = 8;
  const int e1 = __ldg(L.rowStart + c + 1);
  for (int e0 = __ldg(L.rowStart + c); e0 < e1; e0 += B) {
    double pr[B];
#pragma unroll
    for (int k = 0; k < B; ++k)
      pr[k] = e0 + k < e1 ? __dmul_rn(L.rowU[e0 + k], xf(__ldg(L.rowCol + e0 + k))) : 0.0;
#pragma unroll
    for (int k = 0; k < B; ++k)
      if (e0 + k < e1) y = __dadd_rn(y, pr[k]);
  }
  return y;
}

// Loop over [0, n) by the whole grid (blk = false) or by block 0 alone.
template <class F>
__device__ __forceinline__ void gamg_range(int n, bool blk, F body) {
  const int s = blk ? (int)blockDim.x : (int)(gridDim.x * blockDim.x);
  for (int i = blk ? (int)threadIdx.x : (int)(blockIdx.x * blockDim.x + threadIdx.x); i < n; i += s) body(i);
}

// ---------------------------------------------------------------- set-up
// Galerkin coarse matrices of levels 1..L (one grid pass per level), then
// the Cholesky factor and the inverse of the coarsest matrix in block 0.
// Ends with a grid barrier.  lv: the level table (shared memory copy).
__device__ void gamg_galerkin(const GamgLevelDev *lv, int L, const GamgDev *g, const LduDev &a, unsigned *bar,
                              PcgCtl *ctl) {
  // level-0 reciprocal diagonal
  gamg_range(lv[0].n, false, [&](int c) { lv[0].rD[c] = __ddiv_rn(1.0, a.diag[c]); });
  for (int l = 0; l < L; ++l) {
    const GamgLevelDev &F = lv[l], &C = lv[l + 1];
    const double *Df = l == 0 ? a.diag : F.D;
    const double *Uf = l == 0 ? a.upper : F.U;
    gamg_range(C.n, false, [&](int I) {
      double s = 0.0;
      const int m1 = __ldg(F.memStart + I + 1), i1 = __ldg(F.inStart + I + 1);
      for (int e = __ldg(F.memStart + I); e < m1; ++e) s = __dadd_rn(s, Df[__ldg(F.mem + e)]);
      for (int e = __ldg(F.inStart + I); e < i1; ++e) {
        const double u = Uf[__ldg(F.inFace + e)];
        s = __dadd_rn(s, __dadd_rn(u, u));
      }
      C.D[I] = s;
      C.rD[I] = __ddiv_rn(1.0, s);
    });
    gamg_range(C.nf, false, [&](int Fc) {
      double s = 0.0;
      const int e1 = __ldg(F.cfStart + Fc + 1);
      for (int e = __ldg(F.cfStart + Fc); e < e1; ++e) s = __dadd_rn(s, Uf[__ldg(F.cfFace + e)]);
      C.U[Fc] = s;
    });
    grid_barrier(bar);
  }
  // each coarse row entry's coefficient inline (the V-cycle rows read it
  // contiguously instead of through the face index)
  for (int l = 1; l <= L; ++l) {
    const GamgLevelDev &C = lv[l];
    gamg_range(2 * C.nf, false, [&](int e) { C.rowU[e] = C.U[__ldg(C.rowFace + e)]; });
  }
  if (blockIdx.x == 0) {
    // dense coarsest matrix, Cholesky by columns (every element's sum in the
    // oracle's row-by-row order), inverse one column per thread
    const GamgLevelDev &Z = lv[L];
    const int n = Z.n;
    const double *Dz = L == 0 ? a.diag : Z.D;
    const double *Uz = L == 0 ? a.upper : Z.U;
    double *A = g->inv, *Lm = g->chol, *Y = g->ycol;
    for (int i = threadIdx.x; i < n * n; i += blockDim.x) {
      A[i] = 0.0;
      Lm[i] = 0.0;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < n; c += blockDim.x) A[c * n + c] = Dz[c];
    for (int f = threadIdx.x; f < Z.nf; f += blockDim.x) {
      const int l = Z.faceL[f], u = Z.faceU[f];
      A[l * n + u] = Uz[f];
      A[u * n + l] = Uz[f];
    }
    __syncthreads();
    __shared__ int bad;
    if (threadIdx.x == 0) bad = 0;
    for (int j = 0; j < n; ++j) {
      if (threadIdx.x == 0) {
        double s = A[j * n + j];
        for (int k = 0; k < j; ++k) s = __dsub_rn(s, __dmul_rn(Lm[j * n + k], Lm[j * n + k]));
        if (!(s > 0.0)) bad = 1;
        Lm[j * n + j] = __dsqrt_rn(s);
      }
      __syncthreads();
      const double ljj = Lm[j * n + j];
      for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) {
        double s = A[i * n + j];
        for (int k = 0; k < j; ++k) s = __dsub_rn(s, __dmul_rn(Lm[i * n + k], Lm[j * n + k]));
        Lm[i * n + j] = __ddiv_rn(s, ljj);
      }
      __syncthreads();
    }
    if (threadIdx.x == 0 && bad) ctl->fault = 1;
    for (int k = threadIdx.x; k < n; k += blockDim.x) {  // column k of the inverse
      double *y = Y + (size_t)k * n;
      for (int i = 0; i < n; ++i) {
        double s = i == k ? 1.0 : 0.0;
        for (int j = 0; j < i; ++j) s = __dsub_rn(s, __dmul_rn(Lm[i * n + j], y[j]));
        y[i] = __ddiv_rn(s, Lm[i * n + i]);
      }
      for (int i = n - 1; i >= 0; --i) {
        double s = y[i];
        for (int j = i + 1; j < n; ++j) s = __dsub_rn(s, __dmul_rn(Lm[j * n + i], A[j * n + k]));
        A[i * n + k] = __ddiv_rn(s, Lm[i * n + i]);  // A's column k is no longer read
      }
    }
  }
  grid_barrier(bar);
}

// ------------------------------------------------------------- V-cycle
// w = M^-1 r.  On entry lv[0].x holds x_0 = omega rD_0 r (phase 2 of the
// solve writes it with r; gamg_prep otherwise).  Every pass gathers ONE
// stored value per neighbour:
//   down pass l (per coarse cell I): b_{l+1}[I] = sum over members c of
//     b_c - (A_l x_l)_c, and x_{l+1}[I] = omega rD b_{l+1}[I] (stored);
//   coarsest / up pass l (per cell c): the post-smoothed x_l[c] is added
//     to x_{l-1} of c's members in place: lv[l-1].x becomes
//     z_{l-1} = x_{l-1} + P x_l (each member has one aggregate: no race);
//   up pass 0: w = z_0 + omega rD_0 (r - A z_0).
// reduce: ends in the reducing barrier publishing sum w.r to *out (NV = 1),
// else in a plain grid barrier.
template <int RW>
__device__ void gamg_vcycle(const GamgLevelDev *lv, int L, int tail, const double *inv, const MeshDev &m,
                            const LduDev &a, const double *__restrict__ r, double *__restrict__ w, unsigned *bar,
                            double *partials, double *out, bool reduce) {
  const double *rD0 = lv[0].rD;
  double v[1] = {0.0};
  if (L == 0) {  // one level: the coarsest solve is the whole preconditioner
    if (blockIdx.x == 0) {
      const int n = lv[0].n;
      for (int c = threadIdx.x; c < n; c += blockDim.x) {
        double s = 0.0;
        for (int k = 0; k < n; ++k) s = __dadd_rn(s, __dmul_rn(inv[c * n + k], r[k]));
        w[c] = s;
        v[0] = fma(s, r[c], v[0]);
      }
    }
  } else {
    // down pass of level l (restriction to l+1) by the grid or by block 0
    auto down = [&](int l, bool blk) {
      const GamgLevelDev &F = lv[l], &C = lv[l + 1];
      const double *__restrict__ xf = F.x;
      auto xg = [&](int j) { return xf[j]; };
      gamg_range(C.n, blk, [&](int I) {
        double acc = 0.0;
        const int m1 = __ldg(F.memStart + I + 1);
        if (l == 0) {
          // two members per step: their rows' loads are in flight together
          for (int e = __ldg(F.memStart + I); e < m1; e += 2) {
            const int c0 = __ldg(F.mem + e), c1 = e + 1 < m1 ? __ldg(F.mem + e + 1) : -1;
            const double y0 = gamg_row0<RW>(m, a, c0, __dmul_rn(a.diag[c0], xf[c0]), xg);
            const double b0 = r[c0];
            double y1 = 0.0, b1 = 0.0;
            if (c1 >= 0) {
              y1 = gamg_row0<RW>(m, a, c1, __dmul_rn(a.diag[c1], xf[c1]), xg);
              b1 = r[c1];
            }
            acc = __dadd_rn(acc, __dsub_rn(b0, y0));
            if (c1 >= 0) acc = __dadd_rn(acc, __dsub_rn(b1, y1));
          }
        } else {
          for (int e = __ldg(F.memStart + I); e < m1; ++e) {
            const int c = __ldg(F.mem + e);
            const double y = gamg_rowc(F, c, __dmul_rn(F.D[c], xf[c]), xg);
            acc = __dadd_rn(acc, __dsub_rn(F.b[c], y));
          }
        }
        C.b[I] = acc;
        C.x[I] = __dmul_rn(GAMG_OMEGA, __dmul_rn(C.rD[I], acc));
      });
    };
    // z_{l-1} += x_l[c] on the members of cell c of level l
    auto prolong = [&](int l, int c, double xc) {
      const GamgLevelDev &P = lv[l - 1];
      const int m1 = __ldg(P.memStart + c + 1);
      for (int e = __ldg(P.memStart + c); e < m1; ++e) {
        const int mm = __ldg(P.mem + e);
        P.x[mm] = __dadd_rn(P.x[mm], xc);
      }
    };
    // up pass of level l >= 1: x_l = z + omega rD (b - A z), prolonged
    auto up = [&](int l, bool blk) {
      const GamgLevelDev &F = lv[l];
      const double *__restrict__ zf = F.x;
      auto zg = [&](int j) { return zf[j]; };
      gamg_range(F.n, blk, [&](int c) {
        const double zc = zf[c];
        const double y = gamg_rowc(F, c, __dmul_rn(F.D[c], zc), zg);
        prolong(l, c, __dadd_rn(zc, __dmul_rn(GAMG_OMEGA, __dmul_rn(F.rD[c], __dsub_rn(F.b[c], y)))));
      });
    };
    const int t = tail < 1 ? 1 : (tail > L ? L : tail);  // first level run by block 0
    for (int l = 0; l < t; ++l) {
      down(l, false);
      grid_barrier(bar);
      GT();
    }
    if (blockIdx.x == 0) {
      for (int l = t; l < L; ++l) {
        down(l, true);
        __syncthreads();
      }
      const GamgLevelDev &Z = lv[L];
      const int n = Z.n;
      for (int c = threadIdx.x; c < n; c += blockDim.x) {
        double s = 0.0;
        for (int k = 0; k < n; ++k) s = __dadd_rn(s, __dmul_rn(inv[c * n + k], Z.b[k]));
        prolong(L, c, s);
      }
      __syncthreads();
      for (int l = L - 1; l >= t; --l) {
        up(l, true);
        __syncthreads();
      }
    }
    grid_barrier(bar);
    GT();
    for (int l = t - 1; l >= 1; --l) {
      up(l, false);
      grid_barrier(bar);
      GT();
    }
    // level 0: w = z_0 + omega rD0 (r - A z_0)
    const double *__restrict__ z0 = lv[0].x;
    auto zg = [&](int j) { return z0[j]; };
    gamg_range(lv[0].n, false, [&](int c) {
      const double zc = z0[c], rc = r[c];
      const double y = gamg_row0<RW>(m, a, c, __dmul_rn(a.diag[c], zc), zg);
      const double wc = __dadd_rn(zc, __dmul_rn(GAMG_OMEGA, __dmul_rn(rD0[c], __dsub_rn(rc, y))));
      w[c] = wc;
      v[0] = fma(wc, rc, v[0]);
    });
  }
  if (reduce) {
    P2PDev none{};
    grid_reduce_sync<1, false>(v, partials, bar, out, none LF_DBG_ARG(0));
  } else {
    grid_barrier(bar);
  }
}

// x_0 = omega rD_0 r for every cell (before a V-cycle whose r was not
// formed by the solve's phase 2); ends in a grid barrier
__device__ __forceinline__ void gamg_prep(const GamgLevelDev *lv, const double *__restrict__ r, unsigned *bar) {
  const double *rD0 = lv[0].rD;
  double *x0 = lv[0].x;
  gamg_range(lv[0].n, false, [&](int c) { x0[c] = __dmul_rn(GAMG_OMEGA, __dmul_rn(rD0[c], r[c])); });
  grid_barrier(bar);
}

// level table -> shared memory (read at every pass)
__device__ __forceinline__ void gamg_load_levels(const GamgDev *g, GamgLevelDev *lv, int &L, int &tail) {
  const int Lg = g->L;
  const int words = (int)((Lg + 1) * sizeof(GamgLevelDev) / sizeof(int));
  const int *src = reinterpret_cast<const int *>(g->lv);
  int *dst = reinterpret_cast<int *>(lv);
  for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
  L = Lg;
  tail = g->tail;
  __syncthreads();
}

// ----------------------------------------------- persistent GAMG-PCG solve
// k_pcg_dic's state machine with the preconditioner replaced by the V-cycle:
//   set-up:    Galerkin coarse matrices + coarsest inverse; w = M^-1 r; sum w.r
//   iteration: phase 1 (deferred psi, p = w + beta p_old, q = A p over the
//              full rows, sum p.q, sum psi) | r -= alpha q, sum|r| | stop test
//              | w = M^-1 r, sum w.r
// Single rank (no processor interfaces on the coarse levels, A43).
template <int RW>
__global__ void __launch_bounds__(BS, LF_MINB_P)
    k_pcg_gamg(MeshDev m, LduDev a, const GamgDev *g, Workspace ws, unsigned *bar) {
  PcgCtl *ctl = ws.ctl;
  if (ctl->stop) return;
  __shared__ GamgLevelDev lv[GAMG_MAXL + 1];
  struct St {
    double nf, initRes, finRes, wArA, alpha, beta;
    int k, cont, singular;
  };
  __shared__ St st;
  int L, tail;
  gamg_load_levels(g, lv, L, tail);
  double *psi = ctl->psi;
  double *r = ws.r, *w = ws.w, *q = ws.q;
  if (threadIdx.x == 0) {
    st.k = ctl->it;
    st.alpha = ctl->alpha;
    st.singular = 0;
    st.nf = __ldcg(&ws.gsum->setup[0]) + 1e-20;
    st.initRes = __ldcg(&ws.gsum->setup[1]) / st.nf;
    st.finRes = st.initRes;
    st.cont = ctl->minIter > 0 || !conv(st.finRes, st.initRes, ctl);
  }
  __syncthreads();
  if (st.cont) {
    gamg_galerkin(lv, L, g, a, bar, ctl);
    if (L > 0) gamg_prep(lv, r, bar);
    gamg_vcycle<RW>(lv, L, tail, g->inv, m, a, r, w, bar, ws.partials, &ws.gsum->p2[1], true);
  }
  P2PDev none{};
  for (;;) {
    if (threadIdx.x == 0) {
      const double wn = st.cont ? __ldcg(&ws.gsum->p2[1]) : 0.0;
      if (st.k == 0) {
        st.wArA = wn;
        st.beta = 0.0;
      } else if (st.cont) {
        st.beta = wn / st.wArA;
        st.wArA = wn;
      }
    }
    __syncthreads();
    const int k = st.k;
    const bool first = (k == 0), cont = st.cont != 0;
    const double beta = st.beta, alpha = st.alpha;
    const double *pold = (k & 1) ? ws.p[0] : ws.p[1];
    double *pnew = (k & 1) ? ws.p[1] : ws.p[0];
    double v1[2] = {0.0, 0.0};
#if LF_GAMG_QREC
    // deferred psi update; p = w + beta p_old; q = A p by the recurrence
    // q_k = A w_k + beta q_{k-1} (one gather per neighbour: w)
    auto wg = [&](int j) { return w[j]; };
    grid_range(0, m.n, [&](int c) {
      double ps = psi[c];
      if (!first) {
        ps = fma(alpha, pold[c], ps);
        psi[c] = ps;
      }
      v1[1] += ps;
      if (cont) {
        const double wc = w[c];
        const double pc = first ? wc : fma(beta, pold[c], wc);
        pnew[c] = pc;
        const double qo = first ? 0.0 : q[c];
        double qc = row_offdiag<RW>(m, a, c, a.diag[c] * wc, wg);
        if (!first) qc = fma(beta, qo, qc);
        q[c] = qc;
        v1[0] = fma(pc, qc, v1[0]);
      }
    });
#else
#error "LF_GAMG_QREC = 0 is not supported with the half-ELL rows"
#endif
#if LF_GAMG_TIMING
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      g_gton = (k == 5);
      if (k == 5) g_gtn = 0;
    }
#endif
    GT();
    grid_reduce_sync<2, false>(v1, ws.partials, bar, ws.gsum->p1, none LF_DBG_ARG(0));
    GT();
    if (!cont) break;
    if (threadIdx.x == 0) {
      const double pq = __ldcg(&ws.gsum->p1[0]);
      st.singular = fabs(pq) / st.nf < 1e-300;
      if (!st.singular) st.alpha = st.wArA / pq;
    }
    __syncthreads();
    if (st.singular) break;
    const double alphaK = st.alpha;
    double v2[1] = {0.0};
    const double *__restrict__ rD0 = lv[0].rD;
    double *__restrict__ x0 = lv[0].x;
    {
      // a pure stream: two consecutive cells per thread and trip (16-byte accesses)
      auto cell2 = [&](int c) {
        const double2 q2 = *reinterpret_cast<const double2 *>(q + c), r2 = *reinterpret_cast<const double2 *>(r + c);
        double2 rn;
        rn.x = fma(-alphaK, q2.x, r2.x);
        rn.y = fma(-alphaK, q2.y, r2.y);
        *reinterpret_cast<double2 *>(r + c) = rn;
        if (L > 0) {
          const double2 d2 = *reinterpret_cast<const double2 *>(rD0 + c);
          double2 xv;
          xv.x = __dmul_rn(GAMG_OMEGA, __dmul_rn(d2.x, rn.x));  // the V-cycle's x_0
          xv.y = __dmul_rn(GAMG_OMEGA, __dmul_rn(d2.y, rn.y));
          *reinterpret_cast<double2 *>(x0 + c) = xv;
        }
        v2[0] += fabs(rn.x);
        v2[0] += fabs(rn.y);
      };
      const int npair = m.n >> 1, S = gridDim.x * blockDim.x;
      for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < npair; i += S) cell2(2 * i);
      if ((m.n & 1) && blockIdx.x == gridDim.x - 1 && threadIdx.x == blockDim.x - 1) {
        const int c = m.n - 1;
        const double rn = fma(-alphaK, q[c], r[c]);
        r[c] = rn;
        if (L > 0) x0[c] = __dmul_rn(GAMG_OMEGA, __dmul_rn(rD0[c], rn));
        v2[0] += fabs(rn);
      }
    }
    GT();
    grid_reduce_sync<1, false>(v2, ws.partials, bar, &ws.gsum->p2[0], none LF_DBG_ARG(0));
    GT();
    if (threadIdx.x == 0) {
      ++st.k;
      st.finRes = __ldcg(&ws.gsum->p2[0]) / st.nf;
      st.cont = (st.k < ctl->maxIter && !conv(st.finRes, st.initRes, ctl)) || st.k < ctl->minIter;
    }
    __syncthreads();
    if (st.cont) gamg_vcycle<RW>(lv, L, tail, g->inv, m, a, r, w, bar, ws.partials, &ws.gsum->p2[1], true);
    GT();
  }
#if LF_GAMG_TIMING
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    printf("LF_GAMG_TIMING iteration 5, %d marks (us from the phase-1 end):", g_gtn);
    for (int i = 1; i < g_gtn; ++i) printf(" %.1f", (g_gt[i] - g_gt[0]) * 1e-3);
    printf("\n");
    g_gton = 0;
  }
#endif
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

// One application (ldu_precondition): Galerkin set-up + V-cycle.
template <int RW>
__global__ void __launch_bounds__(BS, LF_MINB_P)
    k_gamg_apply(MeshDev m, LduDev a, const GamgDev *g, const double *r, double *w, PcgCtl *ctl,
                 double *partials, unsigned *bar) {
  __shared__ GamgLevelDev lv[GAMG_MAXL + 1];
  int L, tail;
  gamg_load_levels(g, lv, L, tail);
  gamg_galerkin(lv, L, g, a, bar, ctl);
  if (L > 0) gamg_prep(lv, r, bar);
  gamg_vcycle<RW>(lv, L, tail, g->inv, m, a, r, w, bar, partials, nullptr, false);
}

// level-0 row layout of a mesh: the half-ELL slices when it has them, else
// the full rows (built by ensure_gamg)
static int gamg_rw(const MeshDev &m) {
  if (!LF_NO_ELL && m.K > 0 && m.K <= 3) return 3;
  if (!LF_NO_ELL && m.K == 4) return 4;
  return m.KS <= 6 ? -6 : -8;
}

static const void *gamg_solve_fn(int rw) {
  switch (rw) {
    case 3: return (const void *)k_pcg_gamg<3>;
    case 4: return (const void *)k_pcg_gamg<4>;
    case -6: return (const void *)k_pcg_gamg<-6>;
    default: return (const void *)k_pcg_gamg<-8>;
  }
}

static const void *gamg_apply_fn(int rw) {
  switch (rw) {
    case 3: return (const void *)k_gamg_apply<3>;
    case 4: return (const void *)k_gamg_apply<4>;
    case -6: return (const void *)k_gamg_apply<-6>;
    default: return (const void *)k_gamg_apply<-8>;
  }
}

int gamg_grid(int device, const MeshDev &m) {
  int sms = 0, best = 1 << 30;
  LF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  const int rw = gamg_rw(m);
  for (const void *fn : {gamg_solve_fn(rw), gamg_apply_fn(rw)}) {
    int nb = 0;
    LF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, BS, 0));
    best = std::min(best, nb);
  }
  return sms * (best < 1 ? 1 : best);
}

void launch_pcg_gamg(cudaStream_t s, int grid, const MeshDev &m, const LduDev &a, const GamgDev *g,
                     const Workspace &ws, unsigned *bar) {
  void *args[] = {(void *)&m, (void *)&a, (void *)&g, (void *)&ws, (void *)&bar};
  LF_CUDA(cudaLaunchCooperativeKernel(gamg_solve_fn(gamg_rw(m)), dim3(grid), dim3(BS), args, 0, s));
}

void launch_gamg_apply(cudaStream_t s, int grid, const MeshDev &m, const LduDev &a, const GamgDev *g,
                       const double *r, double *w, const Workspace &ws, unsigned *bar) {
  PcgCtl *ctl = ws.ctl;
  double *partials = ws.partials;
  void *args[] = {(void *)&m, (void *)&a, (void *)&g, (void *)&r, (void *)&w, (void *)&ctl, (void *)&partials,
                  (void *)&bar};
  LF_CUDA(cudaLaunchCooperativeKernel(gamg_apply_fn(gamg_rw(m)), dim3(grid), dim3(BS), args, 0, s));
}
