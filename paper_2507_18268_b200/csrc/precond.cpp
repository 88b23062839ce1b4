// DIC preconditioner set-up (kernels in dic.cuh).
//
// Once per mesh, on the host from the device addressing: the level of every
// cell (0 without lower neighbours, else 1 + the largest level of its lower
// neighbours — the dependency depth of OpenFOAM's sequential forward loop),
// the cells grouped by level, and the full-row ELL labels (lower neighbours
// ascending, then upper neighbours ascending; bit 30 = neighbour on level 0).
// The coefficients of those rows (LduDev.symU) are written by every later
// assembly; a system assembled before the set-up is copied over once.
#include <algorithm>

#include "host.h"

namespace lf {

void require_dic(const lf_mesh *M) {
  // the DIC solve is one persistent launch: processor patches need the
  // peer-memory transport (halo and sums inside the kernel), not NCCL
  LF_REQUIRE(!M->ctx->comm && (M->nproc == 0 || M->p2pConnected),
             "the DIC preconditioner needs a single rank or the peer-memory transport (lf_p2p_*)");
  LF_REQUIRE(M->n < DIC_L0BIT, "the DIC preconditioner needs n_cells < 2^30");
}

void ensure_dic(lf_mesh *M) {
  require_dic(M);
  build_rows(M);
}

void ensure_upper(lf_mesh *M) {
  if (!M->upperStale) return;
  M->ctx->launch(LF_K_PRECOND, [&] { launch_upper_from_ell(M->ctx->stream, M->md, M->ld); });
  M->upperStale = false;
}

void build_rows(lf_mesh *M) {
  cudaStream_t s = M->ctx->stream;
  if (!M->dicBuilt) {
    LF_REQUIRE(M->n < DIC_L0BIT, "full-row ELL needs n_cells < 2^30");
    const int32_t n = M->n, F = M->F;
    std::vector<int32_t> os(n + 1), nb(F), ls(n + 1), lo(F);
    LF_CUDA(cudaMemcpyAsync(os.data(), M->md.ownerStart, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost, s));
    LF_CUDA(cudaMemcpyAsync(ls.data(), M->md.losortStart, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost, s));
    if (F > 0) {
      LF_CUDA(cudaMemcpyAsync(nb.data(), M->md.nbr, sizeof(int32_t) * F, cudaMemcpyDeviceToHost, s));
      LF_CUDA(cudaMemcpyAsync(lo.data(), M->md.losortOwner, sizeof(int32_t) * F, cudaMemcpyDeviceToHost, s));
    }
    LF_CUDA(cudaStreamSynchronize(s));
    // levels (lower neighbours have smaller labels: one pass in label order)
    std::vector<int32_t> level(n, 0);
    int32_t L = 1, deg = 0;
    for (int32_t c = 0; c < n; ++c) {
      int32_t lv = 0;
      for (int32_t j = ls[c]; j < ls[c + 1]; ++j) lv = std::max(lv, level[lo[j]] + 1);
      level[c] = lv;
      L = std::max(L, lv + 1);
      deg = std::max(deg, (ls[c + 1] - ls[c]) + (os[c + 1] - os[c]));
    }
    LF_REQUIRE(deg <= 8, "the DIC preconditioner supports cells with at most 8 neighbours");
    const int32_t KS = deg <= 6 ? 6 : 8;
    const int32_t ld = (n + 3) & ~3;
    // cells by level (stable): lvlStart[L+1], lvlCells[n]
    std::vector<int32_t> lstart(L + 1, 0), cells(n);
    for (int32_t c = 0; c < n; ++c) lstart[level[c] + 1]++;
    for (int32_t l = 0; l < L; ++l) lstart[l + 1] += lstart[l];
    {
      std::vector<int32_t> fillp(lstart.begin(), lstart.end() - 1);
      for (int32_t c = 0; c < n; ++c) cells[fillp[level[c]]++] = c;
    }
    bool contig = true;
    for (int32_t t = 0; t < n && contig; ++t) contig = cells[t] == t;
    // full-row labels
    std::vector<int32_t> symN((size_t)KS * ld, -1);
    auto lab = [&](int32_t j) { return j | (level[j] == 0 ? DIC_L0BIT : 0); };
    for (int32_t c = 0; c < n; ++c) {
      int32_t k = 0;
      for (int32_t j = ls[c]; j < ls[c + 1]; ++j) symN[(size_t)(k++) * ld + c] = lab(lo[j]);
      for (int32_t i = os[c]; i < os[c + 1]; ++i) symN[(size_t)(k++) * ld + c] = lab(nb[i]);
    }
    DevArena &A = M->arena;
    int32_t *dStart = A.alloc<int32_t>(L + 1);
    int32_t *dCells = contig ? nullptr : A.alloc<int32_t>(n);
    int32_t *dSymN = A.alloc<int32_t>((size_t)KS * ld);
    double *symU = A.alloc<double>((size_t)KS * ld);
    LF_CUDA(cudaMemcpyAsync(dStart, lstart.data(), sizeof(int32_t) * (L + 1), cudaMemcpyHostToDevice, s));
    if (dCells) LF_CUDA(cudaMemcpyAsync(dCells, cells.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
    LF_CUDA(cudaMemcpyAsync(dSymN, symN.data(), sizeof(int32_t) * KS * (size_t)ld, cudaMemcpyHostToDevice, s));
    LF_CUDA(cudaMemsetAsync(symU, 0, sizeof(double) * KS * (size_t)ld, s));
    DicDev &d = M->dic;
    d.L = L;
    d.contig = contig ? 1 : 0;
    d.lvlStart = dStart;
    d.lvlCells = dCells;
    d.KS = KS;
    d.ldS = ld;
    d.symN = dSymN;
    d.rD = A.alloc<double>(n);
    d.rDu = A.alloc<double>(n);
    M->hLvlStart = lstart;
    M->dicGrid = persistent_tail()  // SM-uniform grid: the passes spread their tail trips
                     ? std::max(1, std::min(dic_grid(M->ctx->device, KS), (n + kernel_block_size() - 1) / kernel_block_size()))
                     : balanced_grid(n, dic_grid(M->ctx->device, KS));
    if (M->dicGrid > M->ws.maxGrid) {  // partials sized for the largest grid
      M->ws.partials = A.alloc<double>(4 * (size_t)M->dicGrid);
      M->ws.maxGrid = M->dicGrid;
    }
    LF_CUDA(cudaStreamSynchronize(s));  // host vectors are released on return
    M->ld.symU = symU;
    M->ld.ldS = ld;
    for (lf::MeshDev *md : {&M->md, &M->mdVar}) {
      md->KS = KS;
      md->ldS = ld;
      md->symN = dSymN;
    }
    M->dicBuilt = true;
    if (M->ldu.assembled) {
      ensure_upper(M);
      M->ctx->launch(LF_K_PRECOND, [&] { launch_sym_fill(s, M->Lamul, M->md, M->ld); });
    }
  }
}

// w = M^-1 r (ldu_precondition): diagonal, or the DIC factor and sweeps as
// one launch per level.
void precondition(lf_mesh *M, int precond, const double *r, double *w, double *rD) {
  lf_context *ctx = M->ctx;
  cudaStream_t s = ctx->stream;
  const int32_t n = M->n;
  if (precond == LF_PRECOND_DIAGONAL) {
    ctx->launch(LF_K_PRECOND, [&] { launch_diag_precondition(s, M->Lamul, n, M->ld.diag, r, w); });
    if (rD) ctx->launch(LF_K_PRECOND, [&] { launch_diag_precondition(s, M->Lamul, n, M->ld.diag, nullptr, rD); });
    return;
  }
  ensure_dic(M);
  const DicDev &d = M->dic;
  const int L = d.L;
  for (int l = 0; l < L; l += (l == 0 ? 2 : 1))  // pass 0 covers levels 0 and 1
    ctx->launch(LF_K_PRECOND, [&] { launch_dic_factor_level(s, M->Lamul, M->md, M->ld, d, l); });
  for (int l = 1; l < L; ++l)
    ctx->launch(LF_K_PRECOND, [&] { launch_dic_sweep_level(s, M->Lamul, M->md, M->ld, d, l, true, r, w); });
  for (int l = L >= 2 ? L - 2 : 0; l >= 0; --l)
    ctx->launch(LF_K_PRECOND, [&] { launch_dic_sweep_level(s, M->Lamul, M->md, M->ld, d, l, false, r, w); });
  if (rD) LF_CUDA(cudaMemcpyAsync(rD, d.rD, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
}

}  // namespace lf
