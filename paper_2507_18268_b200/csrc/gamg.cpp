// GAMG preconditioner set-up (reading A43 in
// DESIGN.md; kernels in gamg.cuh).
//
// Once per mesh, on the host from the device addressing (as OpenFOAM builds
// its agglomeration once, on the CPU): pairwise agglomeration levels, the
// coarse graphs and every index list the device passes need.  The matrix
// values of the coarse levels are formed on the device per solve (Galerkin).
//
// Pairing pass (reading A43): cells visited in ascending label (descending on
// odd passes); an unassigned cell pairs with its unassigned neighbour of
// largest face weight (the first in ascending neighbour label on ties), else
// joins the aggregate of its strongest neighbour, else stays alone;
// aggregates numbered in creation order; the coarse graph has one face per
// pair of adjacent aggregates, sorted (I < J), weight = the fine weights
// summed in ascending fine-face order.  A level = two passes; levels are
// added while the level has more than 64 cells and the next has at most 90%
// of its cells.
#include <algorithm>
#include <cstdlib>
#include <utility>

#include "host.h"

namespace lf {

namespace {

constexpr int32_t kNMin = 64;          // stop coarsening at <= 64 cells
constexpr int32_t kMaxCoarsest = 2048; // dense coarsest solve
constexpr int32_t kTailDefault = 4096; // levels with <= this many cells run in one block

struct Graph {  // faces sorted by (l, u), l < u
  int32_t n = 0;
  std::vector<int32_t> l, u;
  std::vector<double> w;
  int32_t nf() const { return (int32_t)l.size(); }
};

// cell -> incident faces: the faces where the cell is the upper side (their
// lower labels ascend), then those where it is the lower side (upper labels
// ascend) — i.e. ascending neighbour label
struct Adj {
  std::vector<int32_t> start, face;
};

Adj adjacency(const Graph &g) {
  Adj A;
  A.start.assign((size_t)g.n + 1, 0);
  const int32_t nf = g.nf();
  for (int32_t f = 0; f < nf; ++f) {
    A.start[g.l[f] + 1]++;
    A.start[g.u[f] + 1]++;
  }
  for (int32_t c = 0; c < g.n; ++c) A.start[c + 1] += A.start[c];
  A.face.resize((size_t)2 * nf);
  std::vector<int32_t> pos(A.start.begin(), A.start.end() - 1);
  for (int32_t f = 0; f < nf; ++f) A.face[pos[g.u[f]]++] = f;
  for (int32_t f = 0; f < nf; ++f) A.face[pos[g.l[f]]++] = f;
  return A;
}

inline int32_t other(const Graph &g, int32_t f, int32_t c) { return g.l[f] == c ? g.u[f] : g.l[f]; }

// items grouped by key (stable: ascending item within a key)
void group(const std::vector<int32_t> &key, int32_t nkeys, std::vector<int32_t> &start,
           std::vector<int32_t> &items, bool skipNeg = false) {
  start.assign((size_t)nkeys + 1, 0);
  for (int32_t k : key)
    if (k >= 0) start[k + 1]++;
    else if (!skipNeg) throw Error{LF_ERR_INTERNAL, "GAMG: unassigned item"};
  for (int32_t k = 0; k < nkeys; ++k) start[k + 1] += start[k];
  items.resize(start[nkeys]);
  std::vector<int32_t> pos(start.begin(), start.end() - 1);
  for (int32_t i = 0; i < (int32_t)key.size(); ++i)
    if (key[i] >= 0) items[pos[key[i]]++] = i;
}

// one pairing pass: agg[g.n], the coarse graph, cface[g.nf] (-1: inside an aggregate)
void pair_pass(const Graph &g, bool descending, std::vector<int32_t> &agg, Graph &cg, std::vector<int32_t> &cface) {
  const Adj A = adjacency(g);
  agg.assign(g.n, -1);
  int32_t nc = 0;
  for (int32_t i = 0; i < g.n; ++i) {
    const int32_t c = descending ? g.n - 1 - i : i;
    if (agg[c] >= 0) continue;
    int32_t best = -1;
    double bw = -1.0;
    for (int32_t e = A.start[c]; e < A.start[c + 1]; ++e) {
      const int32_t f = A.face[e], j = other(g, f, c);
      if (agg[j] < 0 && g.w[f] > bw) {
        bw = g.w[f];
        best = j;
      }
    }
    if (best >= 0) {
      agg[c] = agg[best] = nc++;
      continue;
    }
    bw = -1.0;
    for (int32_t e = A.start[c]; e < A.start[c + 1]; ++e) {
      const int32_t f = A.face[e];
      if (g.w[f] > bw) {
        bw = g.w[f];
        best = other(g, f, c);
      }
    }
    agg[c] = best >= 0 ? agg[best] : nc++;
  }
  std::vector<int32_t> mstart, mem;
  group(agg, nc, mstart, mem);
  cface.assign(g.nf(), -1);
  cg = Graph{};
  cg.n = nc;
  std::vector<std::pair<int32_t, int32_t>> lst;  // (J, fine face) of aggregate I, J > I
  for (int32_t I = 0; I < nc; ++I) {
    lst.clear();
    for (int32_t k = mstart[I]; k < mstart[I + 1]; ++k) {
      const int32_t c = mem[k];
      for (int32_t e = A.start[c]; e < A.start[c + 1]; ++e) {
        const int32_t f = A.face[e], J = agg[other(g, f, c)];
        if (J > I) lst.emplace_back(J, f);
      }
    }
    std::sort(lst.begin(), lst.end());
    for (size_t k = 0; k < lst.size(); ++k) {
      if (k == 0 || lst[k].first != lst[k - 1].first) {
        cg.l.push_back(I);
        cg.u.push_back(lst[k].first);
        cg.w.push_back(0.0);
      }
      const int32_t F = cg.nf() - 1;
      cface[lst[k].second] = F;
      cg.w[F] += g.w[lst[k].second];  // ascending fine face within (I, J)
    }
  }
}

template <class T>
T *upload(DevArena &A, const std::vector<T> &h, cudaStream_t s) {
  T *d = A.alloc<T>(h.size());
  if (!h.empty()) LF_CUDA(cudaMemcpyAsync(d, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, s));
  return d;
}

int tail_cells() {
  const char *e = std::getenv("LF_GAMG_TAIL");
  return e ? std::max(0, std::atoi(e)) : kTailDefault;
}

}  // namespace

void require_gamg(const lf_mesh *M) {
  LF_REQUIRE(!M->ctx->comm && M->nproc == 0,
             "the GAMG preconditioner is single-rank (no processor patches; reading A43)");
  LF_REQUIRE(M->n < DIC_L0BIT, "the GAMG preconditioner needs n_cells < 2^30");
}

void ensure_gamg(lf_mesh *M) {
  require_gamg(M);
  build_rows(M);  // level-0 rows: the full-row ELL (neighbours ascending) + symU
  M->ld.writeUpper = 1;  // the Galerkin set-up reads the face-order upper
  ensure_upper(M);
  if (M->gamgBuilt) return;
  cudaStream_t s = M->ctx->stream;
  const int32_t n = M->n, F = M->F;
  // level 0 from the device addressing (internal, upper-triangular face order)
  Graph g0;
  g0.n = n;
  g0.l.resize(F);
  g0.u.resize(F);
  g0.w.resize(F);
  {
    std::vector<int32_t> os(n + 1);
    std::vector<double> mag(F), del(F);
    LF_CUDA(cudaMemcpyAsync(os.data(), M->md.ownerStart, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost, s));
    if (F > 0) {
      LF_CUDA(cudaMemcpyAsync(g0.u.data(), M->md.nbr, sizeof(int32_t) * F, cudaMemcpyDeviceToHost, s));
      LF_CUDA(cudaMemcpyAsync(mag.data(), M->md.magSf, sizeof(double) * F, cudaMemcpyDeviceToHost, s));
      LF_CUDA(cudaMemcpyAsync(del.data(), M->md.delta, sizeof(double) * F, cudaMemcpyDeviceToHost, s));
    }
    LF_CUDA(cudaStreamSynchronize(s));
    for (int32_t c = 0; c < n; ++c)
      for (int32_t i = os[c]; i < os[c + 1]; ++i) g0.l[i] = c;
    for (int32_t f = 0; f < F; ++f) g0.w[f] = mag[f] * del[f];  // agglomeration weight |Sf| delta
  }
  // levels
  std::vector<Graph> G;
  std::vector<std::vector<int32_t>> AGG, CF;  // level l -> l+1
  G.push_back(std::move(g0));
  int pass = 0;
  while ((int)G.size() - 1 < GAMG_MAXL && G.back().n > kNMin) {
    const Graph &a = G.back();
    std::vector<int32_t> agg1, cf1, agg2, cf2;
    Graph g1, g2;
    pair_pass(a, pass & 1, agg1, g1, cf1);
    pair_pass(g1, (pass + 1) & 1, agg2, g2, cf2);
    pass += 2;
    if ((double)g2.n > 0.9 * (double)a.n) break;  // coarsening stalled: a is the coarsest
    std::vector<int32_t> agg(a.n), cf(a.nf());
    for (int32_t c = 0; c < a.n; ++c) agg[c] = agg2[agg1[c]];
    for (int32_t f = 0; f < a.nf(); ++f) cf[f] = cf1[f] < 0 ? -1 : cf2[cf1[f]];
    AGG.push_back(std::move(agg));
    CF.push_back(std::move(cf));
    G.push_back(std::move(g2));
  }
  const int32_t L = (int32_t)G.size() - 1;
  LF_REQUIRE(G.back().n <= kMaxCoarsest, "GAMG: coarsening stalled above 2048 cells (coarsest solve is dense)");
  // device structures
  DevArena &A = M->arena;
  GamgDev h{};
  h.L = L;
  const int tc = tail_cells();
  h.tail = L;
  for (int32_t l = 1; l <= L; ++l)
    if (G[l].n <= tc) {
      h.tail = l;
      break;
    }
  M->gamgLevels.clear();
  for (int32_t l = 0; l <= L; ++l) {
    const Graph &g = G[l];
    GamgLevelDev &v = h.lv[l];
    v.n = g.n;
    v.nf = g.nf();
    M->gamgLevels.push_back({g.n, g.nf()});
    v.rD = A.alloc<double>(g.n);
    if (L > 0) v.x = A.alloc<double>(g.n);  // pre-smoothed x, then z (in place)
    if (l >= 1) {
      const Adj adj = adjacency(g);
      std::vector<int32_t> col(adj.face.size());
      for (int32_t c = 0; c < g.n; ++c)
        for (int32_t e = adj.start[c]; e < adj.start[c + 1]; ++e) col[e] = other(g, adj.face[e], c);
      v.rowStart = upload(A, adj.start, s);
      v.rowCol = upload(A, col, s);
      v.rowFace = upload(A, adj.face, s);
      v.rowU = A.alloc<double>(adj.face.size());
      v.D = A.alloc<double>(g.n);
      v.U = A.alloc<double>(g.nf());
      v.b = A.alloc<double>(g.n);
    }
    if (l == L) {
      v.faceL = upload(A, g.l, s);
      v.faceU = upload(A, g.u, s);
    }
    if (l < L) {
      const int32_t nc = G[l + 1].n;
      std::vector<int32_t> st, it;
      v.agg = upload(A, AGG[l], s);
      group(AGG[l], nc, st, it);
      v.memStart = upload(A, st, s);
      v.mem = upload(A, it, s);
      std::vector<int32_t> inKey(g.nf());
      for (int32_t f = 0; f < g.nf(); ++f) inKey[f] = CF[l][f] < 0 ? AGG[l][g.l[f]] : -1;
      group(inKey, nc, st, it, true);
      v.inStart = upload(A, st, s);
      v.inFace = upload(A, it, s);
      group(CF[l], G[l + 1].nf(), st, it, true);
      v.cfStart = upload(A, st, s);
      v.cfFace = upload(A, it, s);
    }
  }
  const size_t nL = (size_t)G.back().n;
  h.inv = A.alloc<double>(nL * nL);
  h.chol = A.alloc<double>(nL * nL);
  h.ycol = A.alloc<double>(nL * nL);
  GamgDev *d = A.alloc<GamgDev>(1);
  LF_CUDA(cudaMemcpyAsync(d, &h, sizeof(GamgDev), cudaMemcpyHostToDevice, s));
  LF_CUDA(cudaStreamSynchronize(s));  // host vectors are released on return
  M->hGamg = h;
  M->dGamg = d;
  M->gamgGrid = std::max(1, std::min(gamg_grid(M->ctx->device, M->md),
                                     (n + kernel_block_size() - 1) / kernel_block_size()));
  if (M->gamgGrid > M->ws.maxGrid) {  // partials sized for the largest grid
    M->ws.partials = A.alloc<double>(4 * (size_t)M->gamgGrid);
    M->ws.maxGrid = M->gamgGrid;
  }
  M->gamgBuilt = true;
}

// w = M^-1 r (ldu_precondition): Galerkin set-up + one V-cycle, one launch
void gamg_precondition(lf_mesh *M, const double *r, double *w, double *rD) {
  ensure_gamg(M);
  lf_context *ctx = M->ctx;
  cudaStream_t s = ctx->stream;
  ctx->launch(LF_K_PRECOND, [&] {
    launch_gamg_apply(s, M->gamgGrid, M->md, M->ld, M->dGamg, r, w, M->ws, M->gridBar);
  });
  M->gamgFormed = true;
  if (rD) LF_CUDA(cudaMemcpyAsync(rD, M->hGamg.lv[0].rD, sizeof(double) * M->n, cudaMemcpyDeviceToDevice, s));
}

// host copies of level `level`'s coarse matrix (after a GAMG solve or
// application) and of the hierarchy
void gamg_export(lf_mesh *M, int32_t level, double *D, double *U, int32_t *fl, int32_t *fu) {
  LF_REQUIRE(M->gamgFormed, "no GAMG solve or application yet");
  const GamgDev &h = M->hGamg;
  LF_REQUIRE(level >= 1 && level <= h.L, "GAMG level out of range");
  cudaStream_t s = M->ctx->stream;
  const GamgLevelDev &v = h.lv[level];
  if (D) LF_CUDA(cudaMemcpyAsync(D, v.D, sizeof(double) * v.n, cudaMemcpyDeviceToHost, s));
  if (U && v.nf) LF_CUDA(cudaMemcpyAsync(U, v.U, sizeof(double) * v.nf, cudaMemcpyDeviceToHost, s));
  if ((fl || fu) && v.nf) {
    // faces from the rows: entry e of row c with neighbour j > c is face (c, j)
    std::vector<int32_t> st(v.n + 1), col(2 * (size_t)v.nf), fc(2 * (size_t)v.nf);
    LF_CUDA(cudaMemcpyAsync(st.data(), v.rowStart, sizeof(int32_t) * (v.n + 1), cudaMemcpyDeviceToHost, s));
    LF_CUDA(cudaMemcpyAsync(col.data(), v.rowCol, sizeof(int32_t) * 2 * v.nf, cudaMemcpyDeviceToHost, s));
    LF_CUDA(cudaMemcpyAsync(fc.data(), v.rowFace, sizeof(int32_t) * 2 * v.nf, cudaMemcpyDeviceToHost, s));
    LF_CUDA(cudaStreamSynchronize(s));
    for (int32_t c = 0; c < v.n; ++c)
      for (int32_t e = st[c]; e < st[c + 1]; ++e)
        if (col[e] > c) {
          if (fl) fl[fc[e]] = c;
          if (fu) fu[fc[e]] = col[e];
        }
  }
  LF_CUDA(cudaStreamSynchronize(s));
}

void gamg_hierarchy(lf_mesh *M, int32_t *n_levels, int32_t *cells, int32_t *faces, int32_t *agg) {
  ensure_gamg(M);
  const GamgDev &h = M->hGamg;
  if (n_levels) *n_levels = h.L + 1;
  size_t off = 0;
  cudaStream_t s = M->ctx->stream;
  for (int32_t l = 0; l <= h.L; ++l) {
    if (cells) cells[l] = h.lv[l].n;
    if (faces) faces[l] = h.lv[l].nf;
    if (agg && l < h.L) {
      LF_CUDA(cudaMemcpyAsync(agg + off, h.lv[l].agg, sizeof(int32_t) * h.lv[l].n, cudaMemcpyDeviceToHost, s));
      off += h.lv[l].n;
    }
  }
  LF_CUDA(cudaStreamSynchronize(s));
}

}  // namespace lf
