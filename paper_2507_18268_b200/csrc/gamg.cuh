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

// level-0 row: y += sum over the full row (ascending neighbour label) of U x_j
template <int KS, class XF>
__device__ __forceinline__ double gamg_row0(const DicDev &d, const LduDev &a, int c, double y, XF xf) {
#pragma unroll
  for (int k = 0; k < KS; ++k) {
    const int lab = __ldg(d.symN + k * d.ldS + c);
    if (lab >= 0) y = __dadd_rn(y, __dmul_rn(__ldg(a.symU + k * d.ldS + c), xf(sym_cell(lab))));
  }
  return y;
}

// coarse-level row (CSR, ascending neighbour label)
template <class XF>
__device__ __forceinline__ double gamg_rowc(const GamgLevelDev &L, int c, double y, XF xf) {
  const int e1 = __ldg(L.rowStart + c + 1);
  for (int e = __ldg(L.rowStart + c); e < e1; ++e)
    y = __dadd_rn(y, __dmul_rn(L.U[__ldg(L.rowFace + e)], xf(__ldg(L.rowCol + e))));
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
// w = M^-1 r.  reduce: ends in the reducing barrier publishing sum w.r to
// *out (NV = 1), else in a plain grid barrier.
template <int KS>
__device__ void gamg_vcycle(const GamgLevelDev *lv, int L, int tail, const double *inv, const DicDev &d,
                            const LduDev &a, const double *__restrict__ r, double *__restrict__ w, unsigned *bar,
                            double *partials, double *out, bool reduce) {
  const double *rD0 = lv[0].rD;
  auto x0 = [&](int j) { return __dmul_rn(GAMG_OMEGA, __dmul_rn(rD0[j], r[j])); };
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
      if (l == 0) {
        gamg_range(C.n, blk, [&](int I) {
          double acc = 0.0;
          const int m1 = __ldg(F.memStart + I + 1);
          for (int e = __ldg(F.memStart + I); e < m1; ++e) {
            const int c = __ldg(F.mem + e);
            const double y = gamg_row0<KS>(d, a, c, __dmul_rn(a.diag[c], x0(c)), x0);
            acc = __dadd_rn(acc, __dsub_rn(r[c], y));
          }
          C.b[I] = acc;
        });
      } else {
        auto xl = [&](int j) { return __dmul_rn(GAMG_OMEGA, __dmul_rn(F.rD[j], F.b[j])); };
        gamg_range(C.n, blk, [&](int I) {
          double acc = 0.0;
          const int m1 = __ldg(F.memStart + I + 1);
          for (int e = __ldg(F.memStart + I); e < m1; ++e) {
            const int c = __ldg(F.mem + e);
            const double y = gamg_rowc(F, c, __dmul_rn(F.D[c], xl(c)), xl);
            acc = __dadd_rn(acc, __dsub_rn(F.b[c], y));
          }
          C.b[I] = acc;
        });
      }
    };
    // up pass of level l >= 1: x_l = z + omega rD (b - A z), z = x_l + P x_{l+1}
    auto up = [&](int l, bool blk) {
      const GamgLevelDev &F = lv[l], &C = lv[l + 1];
      auto z = [&](int j) {
        return __dadd_rn(__dmul_rn(GAMG_OMEGA, __dmul_rn(F.rD[j], F.b[j])), C.x[__ldg(F.agg + j)]);
      };
      gamg_range(F.n, blk, [&](int c) {
        const double zc = z(c);
        const double y = gamg_rowc(F, c, __dmul_rn(F.D[c], zc), z);
        F.x[c] = __dadd_rn(zc, __dmul_rn(GAMG_OMEGA, __dmul_rn(F.rD[c], __dsub_rn(F.b[c], y))));
      });
    };
    const int t = tail < 1 ? 1 : (tail > L ? L : tail);  // first level run by block 0
    for (int l = 0; l < t; ++l) {
      down(l, false);
      grid_barrier(bar);
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
        Z.x[c] = s;
      }
      __syncthreads();
      for (int l = L - 1; l >= t; --l) {
        up(l, true);
        __syncthreads();
      }
    }
    grid_barrier(bar);
    for (int l = t - 1; l >= 1; --l) {
      up(l, false);
      grid_barrier(bar);
    }
    // level 0: w = z + omega rD0 (r - A z), z = x0 + x_1[agg]
    const GamgLevelDev &F = lv[0], &C = lv[1];
    auto z = [&](int j) { return __dadd_rn(x0(j), C.x[__ldg(F.agg + j)]); };
    gamg_range(F.n, false, [&](int c) {
      const double zc = z(c);
      const double y = gamg_row0<KS>(d, a, c, __dmul_rn(a.diag[c], zc), z);
      const double wc = __dadd_rn(zc, __dmul_rn(GAMG_OMEGA, __dmul_rn(rD0[c], __dsub_rn(r[c], y))));
      w[c] = wc;
      v[0] = fma(wc, r[c], v[0]);
    });
  }
  if (reduce) {
    P2PDev none{};
    grid_reduce_sync<1, false>(v, partials, bar, out, none LF_DBG_ARG(0));
  } else {
    grid_barrier(bar);
  }
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
template <int KS>
__global__ void __launch_bounds__(BS, LF_MINB_P)
    k_pcg_gamg(MeshDev m, LduDev a, DicDev d, const GamgDev *g, Workspace ws, unsigned *bar) {
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
    gamg_vcycle<KS>(lv, L, tail, g->inv, d, a, r, w, bar, ws.partials, &ws.gsum->p2[1], true);
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
    grid_range(0, m.n, [&](int c) {
      dic_amul_cell<KS, false>(m, a, d, ws, k, c, first, cont, alpha, beta, psi, w, pold, pnew, q, v1, false);
    });
    grid_reduce_sync<2, false>(v1, ws.partials, bar, ws.gsum->p1, none LF_DBG_ARG(0));
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
    grid_range(0, m.n, [&](int c) {
      const double rn = fma(-alphaK, q[c], r[c]);
      r[c] = rn;
      v2[0] += fabs(rn);
    });
    grid_reduce_sync<1, false>(v2, ws.partials, bar, &ws.gsum->p2[0], none LF_DBG_ARG(0));
    if (threadIdx.x == 0) {
      ++st.k;
      st.finRes = __ldcg(&ws.gsum->p2[0]) / st.nf;
      st.cont = (st.k < ctl->maxIter && !conv(st.finRes, st.initRes, ctl)) || st.k < ctl->minIter;
    }
    __syncthreads();
    if (st.cont) gamg_vcycle<KS>(lv, L, tail, g->inv, d, a, r, w, bar, ws.partials, &ws.gsum->p2[1], true);
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

// One application (ldu_precondition): Galerkin set-up + V-cycle.
template <int KS>
__global__ void __launch_bounds__(BS, LF_MINB_P)
    k_gamg_apply(LduDev a, DicDev d, const GamgDev *g, const double *r, double *w, PcgCtl *ctl, double *partials,
                 unsigned *bar) {
  __shared__ GamgLevelDev lv[GAMG_MAXL + 1];
  int L, tail;
  gamg_load_levels(g, lv, L, tail);
  gamg_galerkin(lv, L, g, a, bar, ctl);
  gamg_vcycle<KS>(lv, L, tail, g->inv, d, a, r, w, bar, partials, nullptr, false);
}

template <int KS>
static const void *gamg_solve_fn() {
  return (const void *)k_pcg_gamg<KS>;
}

int gamg_grid(int device, int KS) {
  int sms = 0, best = 1 << 30;
  LF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  for (const void *fn : {KS <= 6 ? (const void *)k_pcg_gamg<6> : (const void *)k_pcg_gamg<8>,
                         KS <= 6 ? (const void *)k_gamg_apply<6> : (const void *)k_gamg_apply<8>}) {
    int nb = 0;
    LF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, BS, 0));
    best = std::min(best, nb);
  }
  return sms * (best < 1 ? 1 : best);
}

void launch_pcg_gamg(cudaStream_t s, int grid, const MeshDev &m, const LduDev &a, const DicDev &d,
                     const GamgDev *g, const GamgDev &hg, const Workspace &ws, unsigned *bar) {
  (void)hg;
  void *args[] = {(void *)&m, (void *)&a, (void *)&d, (void *)&g, (void *)&ws, (void *)&bar};
  const void *fn = d.KS <= 6 ? (const void *)k_pcg_gamg<6> : (const void *)k_pcg_gamg<8>;
  LF_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(BS), args, 0, s));
}

void launch_gamg_apply(cudaStream_t s, int grid, const LduDev &a, const DicDev &d, const GamgDev *g,
                       const GamgDev &hg, const double *r, double *w, const Workspace &ws, unsigned *bar) {
  (void)hg;
  PcgCtl *ctl = ws.ctl;
  double *partials = ws.partials;
  void *args[] = {(void *)&a, (void *)&d, (void *)&g, (void *)&r, (void *)&w, (void *)&ctl, (void *)&partials,
                  (void *)&bar};
  const void *fn = d.KS <= 6 ? (const void *)k_gamg_apply<6> : (const void *)k_gamg_apply<8>;
  LF_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(BS), args, 0, s));
}
