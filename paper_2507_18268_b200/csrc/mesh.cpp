// mesh_create: validation, optional RCM renumbering, upload and the
// device-side build of the atomic-free addressing of P:387-429 / P:471-481.
#include <algorithm>
#include <cmath>
#include <numeric>

#include "host.h"

#ifndef LF_NO_SYM_ROWS
#define LF_NO_SYM_ROWS 0  // 1: meshes with K > 4 keep the CSR gather (ablation)
#endif

namespace lf {

// Reverse Cuthill-McKee on the cell graph (host, once per mesh).  Returns
// order[i] = caller label of internal cell i.  Start of each component: a
// pseudo-peripheral cell (two BFS sweeps from the minimum-degree cell).
static std::vector<int32_t> rcm_order(int32_t n, int32_t F, const int32_t *own, const int32_t *nbr) {
  std::vector<int32_t> deg(n, 0), start(n + 1, 0), adj(2 * (size_t)F);
  for (int32_t f = 0; f < F; ++f) {
    deg[own[f]]++;
    deg[nbr[f]]++;
  }
  for (int32_t c = 0; c < n; ++c) start[c + 1] = start[c] + deg[c];
  std::vector<int32_t> fill(start.begin(), start.end() - 1);
  for (int32_t f = 0; f < F; ++f) {
    adj[fill[own[f]]++] = nbr[f];
    adj[fill[nbr[f]]++] = own[f];
  }
  for (int32_t c = 0; c < n; ++c)
    std::sort(adj.begin() + start[c], adj.begin() + start[c + 1], [&](int32_t a, int32_t b) {
      return deg[a] != deg[b] ? deg[a] < deg[b] : a < b;
    });
  std::vector<int32_t> order;
  order.reserve(n);
  std::vector<int32_t> level(n, -1);
  std::vector<char> visited(n, 0);
  auto bfs_last = [&](int32_t s, std::vector<int32_t> &touched) {
    // BFS from s; returns min-degree cell of the last level
    touched.clear();
    touched.push_back(s);
    level[s] = 0;
    size_t head = 0;
    int32_t maxl = 0;
    while (head < touched.size()) {
      int32_t u = touched[head++];
      for (int32_t k = start[u]; k < start[u + 1]; ++k) {
        int32_t v = adj[k];
        if (level[v] < 0) {
          level[v] = level[u] + 1;
          maxl = std::max(maxl, level[v]);
          touched.push_back(v);
        }
      }
    }
    int32_t best = s;
    for (int32_t u : touched)
      if (level[u] == maxl && (deg[u] < deg[best] || level[best] != maxl)) best = u;
    for (int32_t u : touched) level[u] = -1;
    return best;
  };
  std::vector<int32_t> touched;
  std::vector<int32_t> byDeg(n);
  std::iota(byDeg.begin(), byDeg.end(), 0);
  std::stable_sort(byDeg.begin(), byDeg.end(), [&](int32_t a, int32_t b) { return deg[a] < deg[b]; });
  for (int32_t s0 : byDeg) {
    if (visited[s0]) continue;
    int32_t s = bfs_last(s0, touched);
    s = bfs_last(s, touched);
    size_t head = order.size();
    order.push_back(s);
    visited[s] = 1;
    while (head < order.size()) {
      int32_t u = order[head++];
      for (int32_t k = start[u]; k < start[u + 1]; ++k) {
        int32_t v = adj[k];
        if (!visited[v]) {
          visited[v] = 1;
          order.push_back(v);
        }
      }
    }
  }
  std::reverse(order.begin(), order.end());
  return order;
}

// Greedy first-fit colouring in label order (renumber = 2): colour(c) = the
// smallest colour not used by a lower-labelled neighbour.  Returns order[i]
// = caller label of internal cell i, cells sorted by (colour, label): every
// colour class is a contiguous, dependency-free block — the DIC levels.
static std::vector<int32_t> colour_order(int32_t n, int32_t F, const int32_t *own, const int32_t *nbr) {
  std::vector<int32_t> start(n + 1, 0), adj(2 * (size_t)F);
  for (int32_t f = 0; f < F; ++f) {
    start[own[f] + 1]++;
    start[nbr[f] + 1]++;
  }
  for (int32_t c = 0; c < n; ++c) start[c + 1] += start[c];
  std::vector<int32_t> fill(start.begin(), start.end() - 1);
  int32_t maxDeg = 0;
  for (int32_t c = 0; c < n; ++c) maxDeg = std::max(maxDeg, start[c + 1] - start[c]);
  for (int32_t f = 0; f < F; ++f) {
    adj[fill[own[f]]++] = nbr[f];
    adj[fill[nbr[f]]++] = own[f];
  }
  std::vector<int32_t> col(n, 0), stamp(maxDeg + 2, -1);
  int32_t nCol = 1;
  for (int32_t c = 0; c < n; ++c) {
    for (int32_t k = start[c]; k < start[c + 1]; ++k)
      if (adj[k] < c) stamp[col[adj[k]]] = c;
    int32_t k = 0;
    while (stamp[k] == c) ++k;
    col[c] = k;
    nCol = std::max(nCol, k + 1);
  }
  std::vector<int32_t> cnt(nCol + 1, 0), order(n);
  for (int32_t c = 0; c < n; ++c) cnt[col[c] + 1]++;
  for (int32_t k = 0; k < nCol; ++k) cnt[k + 1] += cnt[k];
  for (int32_t c = 0; c < n; ++c) order[cnt[col[c]]++] = c;
  return order;
}

int balanced_grid(int64_t n, int g0) {
  const int BSZ = kernel_block_size();
  const int need = (int)((n + BSZ - 1) / BSZ);
  if (need <= g0) return std::max(1, need);
  const int T = (need + g0 - 1) / g0;
  return (need + T - 1) / T;
}

static void validate(const lf_mesh_desc *d, int rank) {
  LF_REQUIRE(d != nullptr, "desc is NULL");
  LF_REQUIRE(d->n_cells >= 1, "n_cells must be >= 1");
  LF_REQUIRE(d->n_faces >= 0, "n_faces must be >= 0");
  LF_REQUIRE(d->n_patches >= 0, "n_patches must be >= 0");
  LF_REQUIRE(d->n_faces == 0 || (d->owner && d->neighbour && d->mag_sf && d->delta_coeffs),
             "owner/neighbour/mag_sf/delta_coeffs required");
  LF_REQUIRE(d->V != nullptr, "V required");
  LF_REQUIRE(d->renumber >= 0 && d->renumber <= 2, "renumber must be 0, 1 (RCM) or 2 (colour)");
  LF_REQUIRE(d->n_patches == 0 || d->patches, "patches required");
  const int32_t n = d->n_cells;
  for (int32_t f = 0; f < d->n_faces; ++f) {
    const int32_t o = d->owner[f], nb = d->neighbour[f];
    if (o < 0 || o >= n || nb < 0 || nb >= n)
      throw Error{LF_ERR_INVALID_ARG, "face " + std::to_string(f) + ": label out of range"};
    if (o == nb) throw Error{LF_ERR_INVALID_ARG, "face " + std::to_string(f) + ": owner == neighbour"};
    if (!(d->mag_sf[f] > 0.0) || !std::isfinite(d->mag_sf[f]))
      throw Error{LF_ERR_INVALID_ARG, "face " + std::to_string(f) + ": mag_sf must be > 0"};
    if (!(d->delta_coeffs[f] > 0.0) || !std::isfinite(d->delta_coeffs[f]))
      throw Error{LF_ERR_INVALID_ARG, "face " + std::to_string(f) + ": delta_coeffs must be > 0"};
  }
  for (int32_t c = 0; c < n; ++c)
    if (!(d->V[c] > 0.0) || !std::isfinite(d->V[c]))
      throw Error{LF_ERR_INVALID_ARG, "cell " + std::to_string(c) + ": V must be > 0"};
  int selfOpen = 0;
  for (int32_t p = 0; p < d->n_patches; ++p) {
    const lf_patch_desc &P = d->patches[p];
    const std::string pn = "patch " + std::to_string(p);
    LF_REQUIRE(P.type == LF_PATCH_FIXED_VALUE || P.type == LF_PATCH_ZERO_GRADIENT ||
                   P.type == LF_PATCH_PROCESSOR,
               pn + ": unknown type");
    LF_REQUIRE(P.n_faces >= 0, pn + ": n_faces < 0");
    LF_REQUIRE(P.n_faces == 0 || (P.face_cells && P.mag_sf && P.delta_coeffs),
               pn + ": face_cells/mag_sf/delta_coeffs required");
    for (int32_t i = 0; i < P.n_faces; ++i) {
      LF_REQUIRE(P.face_cells[i] >= 0 && P.face_cells[i] < n, pn + ": face_cells out of range");
      LF_REQUIRE(P.mag_sf[i] > 0.0 && std::isfinite(P.mag_sf[i]), pn + ": mag_sf must be > 0");
      LF_REQUIRE(P.delta_coeffs[i] > 0.0 && std::isfinite(P.delta_coeffs[i]),
                 pn + ": delta_coeffs must be > 0");
    }
    if (P.type == LF_PATCH_PROCESSOR && P.neighb_rank == rank) selfOpen ^= 1;
  }
  LF_REQUIRE(selfOpen == 0, "self-coupled processor patches must come in pairs");
  // full geometry (non-orthogonal path): all or nothing
  if (d->sf || d->cf || d->c) {
    LF_REQUIRE(d->c && (d->n_faces == 0 || (d->sf && d->cf)), "sf, cf and c must be given together");
    for (int32_t p = 0; p < d->n_patches; ++p) {
      const lf_patch_desc &P = d->patches[p];
      LF_REQUIRE(P.n_faces == 0 || P.sf, "patch " + std::to_string(p) + ": sf required with full geometry");
      LF_REQUIRE((P.cf == nullptr) == (P.cn == nullptr), "patch " + std::to_string(p) + ": cf and cn go together");
      if (P.cf) {
        LF_REQUIRE(P.type == LF_PATCH_PROCESSOR, "patch " + std::to_string(p) + ": cf/cn are for processor patches");
        for (int64_t i = 0; i < 3 * (int64_t)P.n_faces; ++i)
          LF_REQUIRE(std::isfinite(P.cf[i]) && std::isfinite(P.cn[i]), "cf/cn must be finite");
      }
    }
    for (int64_t i = 0; i < 3 * (int64_t)d->n_faces; ++i)
      LF_REQUIRE(std::isfinite(d->sf[i]) && std::isfinite(d->cf[i]), "sf/cf must be finite");
    for (int64_t i = 0; i < 3 * (int64_t)n; ++i) LF_REQUIRE(std::isfinite(d->c[i]), "c must be finite");
  }
}

}  // namespace lf

using namespace lf;

lf_mesh::~lf_mesh() {
  for (auto &g : chunkGraph)
    if (g) cudaGraphExecDestroy(g);
  for (void *p : ipcOpened) cudaIpcCloseMemHandle(p);
  if (hctl) cudaFreeHost(hctl);
  arena.release();
}

static void build_mesh(lf_context *ctx, const lf_mesh_desc *d, lf_mesh *M) {
  validate(d, ctx->rank);
  cudaStream_t s = ctx->stream;
  DevArena &A = M->arena;
  const int32_t n = d->n_cells, F = d->n_faces;
  M->ctx = ctx;
  M->n = n;
  M->F = F;
  M->nPatches = d->n_patches;

  // ---------------------------------------------- optional renumbering
  std::vector<int32_t> iperm;  // caller -> internal
  if (d->renumber) {
    std::vector<int32_t> order = d->renumber == 2 ? colour_order(n, F, d->owner, d->neighbour)
                                                  : rcm_order(n, F, d->owner, d->neighbour);
    iperm.assign(n, 0);
    for (int32_t i = 0; i < n; ++i) iperm[order[i]] = i;
    M->renumbered = true;
    M->cellPerm = A.alloc<int32_t>(n);
    M->cellIperm = A.alloc<int32_t>(n);
    LF_CUDA(cudaMemcpyAsync(M->cellPerm, order.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
    LF_CUDA(cudaMemcpyAsync(M->cellIperm, iperm.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
    LF_CUDA(cudaStreamSynchronize(s));
  }
  auto relabel = [&](const int32_t *src, size_t m) {
    std::vector<int32_t> out(src, src + m);
    if (!iperm.empty())
      for (auto &x : out) x = iperm[x];
    return out;
  };

  // ------------------------------------------------- internal faces
  // upper-triangular re-sort: key = (min label, max label), stable
  int32_t *ownerU = A.alloc<int32_t>(F), *nbrU = A.alloc<int32_t>(F);
  uint64_t *keys = nullptr;
  LF_CUDA(cudaMallocAsync(&keys, sizeof(uint64_t) * std::max(F, 1), s));
  {
    std::vector<int32_t> o = relabel(d->owner, F), nb = relabel(d->neighbour, F);
    for (int32_t f = 0; f < F; ++f) M->bandwidth = std::max<int64_t>(M->bandwidth, std::abs((int64_t)o[f] - nb[f]));
    LF_CUDA(cudaMemcpyAsync(ownerU, o.data(), sizeof(int32_t) * F, cudaMemcpyHostToDevice, s));
    LF_CUDA(cudaMemcpyAsync(nbrU, nb.data(), sizeof(int32_t) * F, cudaMemcpyHostToDevice, s));
    launch_make_keys(s, ownerU, nbrU, F, keys);
    LF_CUDA(cudaStreamSynchronize(s));
  }
  M->facePerm = A.alloc<int32_t>(F);
  launch_iota(s, M->facePerm, F);
  int bits = 1;
  while ((1ll << bits) < (long long)n) ++bits;
  sort_pairs_u64(s, keys, M->facePerm, F, 32 + bits);
  int32_t *owner = ownerU, *nbr = nbrU;  // reuse buffers for the sorted labels
  launch_split_keys(s, keys, F, owner, nbr);
  LF_CUDA(cudaFreeAsync(keys, s));
  M->ownerInt = owner;

  double *magSf = A.alloc<double>(F), *delta = A.alloc<double>(F);
  {
    double *tmp = nullptr;
    LF_CUDA(cudaMallocAsync(&tmp, sizeof(double) * std::max(F, 1), s));
    LF_CUDA(cudaMemcpyAsync(tmp, d->mag_sf, sizeof(double) * F, cudaMemcpyHostToDevice, s));
    launch_gather_f64(s, F, M->facePerm, tmp, magSf);
    LF_CUDA(cudaMemcpyAsync(tmp, d->delta_coeffs, sizeof(double) * F, cudaMemcpyHostToDevice, s));
    launch_gather_f64(s, F, M->facePerm, tmp, delta);
    LF_CUDA(cudaFreeAsync(tmp, s));
  }
  int32_t *ownerStart = A.alloc<int32_t>(n + 1);
  launch_starts_from_sorted(s, owner, F, n, ownerStart);
  // losort = stable argsort of neighbour (the paper's neighbourList)
  int32_t *losort = A.alloc<int32_t>(F), *losortStart = A.alloc<int32_t>(n + 1),
          *losortOwner = A.alloc<int32_t>(F);
  {
    int32_t *k2 = nullptr;
    LF_CUDA(cudaMallocAsync(&k2, sizeof(int32_t) * std::max(F, 1), s));
    LF_CUDA(cudaMemcpyAsync(k2, nbr, sizeof(int32_t) * F, cudaMemcpyDeviceToDevice, s));
    launch_iota(s, losort, F);
    sort_pairs_i32(s, k2, losort, F, bits);
    launch_starts_from_sorted(s, k2, F, n, losortStart);
    launch_gather_i32(s, F, losort, owner, losortOwner);
    LF_CUDA(cudaFreeAsync(k2, s));
  }
  double *V = A.alloc<double>(n);
  {
    if (iperm.empty()) {
      LF_CUDA(cudaMemcpyAsync(V, d->V, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    } else {
      std::vector<double> v(n);
      for (int32_t c = 0; c < n; ++c) v[iperm[c]] = d->V[c];
      LF_CUDA(cudaMemcpyAsync(V, v.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s));
      LF_CUDA(cudaStreamSynchronize(s));
    }
  }

  // ------------------------------------------------------ boundary
  int32_t B = 0;
  for (int32_t p = 0; p < d->n_patches; ++p) B += d->patches[p].n_faces;
  M->B = B;
  std::vector<int32_t> hCell(B), hSlot(B, -1);
  std::vector<int8_t> hType(B);
  std::vector<double> hMag(B), hDel(B), hVal(B, 0.0);
  M->patchStart.assign(d->n_patches + 1, 0);
  int32_t nproc = 0;
  std::vector<int32_t> sendCells;
  std::vector<int32_t> selfOpenSeg;
  for (int32_t p = 0, off = 0; p < d->n_patches; ++p) {
    const lf_patch_desc &P = d->patches[p];
    M->patchType.push_back(P.type);
    M->patchRank.push_back(P.type == LF_PATCH_PROCESSOR ? P.neighb_rank : -1);
    if (P.type == LF_PATCH_PROCESSOR) {
      LF_REQUIRE(P.neighb_rank >= 0 && P.neighb_rank < ctx->nranks,
                 "patch " + std::to_string(p) + ": neighb_rank out of range for the communicator");
      HaloSeg sg{nproc, P.n_faces, P.neighb_rank, -1};
      if (P.neighb_rank == ctx->rank) {
        if (selfOpenSeg.empty()) {
          selfOpenSeg.push_back((int32_t)M->segs.size());
        } else {
          const int32_t a = selfOpenSeg.back();
          selfOpenSeg.pop_back();
          LF_REQUIRE(M->segs[a].count == P.n_faces, "self-coupled processor patches differ in size");
          sg.partner = a;
          M->segs[a].partner = (int32_t)M->segs.size();
        }
      }
      M->segs.push_back(sg);
    }
    for (int32_t i = 0; i < P.n_faces; ++i) {
      const int32_t fi = off + i;
      hCell[fi] = iperm.empty() ? P.face_cells[i] : iperm[P.face_cells[i]];
      hType[fi] = (int8_t)P.type;
      hMag[fi] = P.mag_sf[i];
      hDel[fi] = P.delta_coeffs[i];
      if (P.type == LF_PATCH_FIXED_VALUE && P.value) hVal[fi] = P.value[i];
      if (P.type == LF_PATCH_PROCESSOR) {
        hSlot[fi] = nproc++;
        sendCells.push_back(hCell[fi]);
      }
    }
    off += P.n_faces;
    M->patchStart[p + 1] = off;
  }
  M->nproc = nproc;
  M->bCell = A.alloc<int32_t>(B);
  int8_t *bType = A.alloc<int8_t>(B);
  double *bMag = A.alloc<double>(B), *bDel = A.alloc<double>(B);
  M->bValue = A.alloc<double>(B);
  int32_t *bSlot = A.alloc<int32_t>(B);
  LF_CUDA(cudaMemcpyAsync(M->bCell, hCell.data(), sizeof(int32_t) * B, cudaMemcpyHostToDevice, s));
  LF_CUDA(cudaMemcpyAsync(bType, hType.data(), B, cudaMemcpyHostToDevice, s));
  LF_CUDA(cudaMemcpyAsync(bMag, hMag.data(), sizeof(double) * B, cudaMemcpyHostToDevice, s));
  LF_CUDA(cudaMemcpyAsync(bDel, hDel.data(), sizeof(double) * B, cudaMemcpyHostToDevice, s));
  LF_CUDA(cudaMemcpyAsync(M->bValue, hVal.data(), sizeof(double) * B, cudaMemcpyHostToDevice, s));
  LF_CUDA(cudaMemcpyAsync(bSlot, hSlot.data(), sizeof(int32_t) * B, cudaMemcpyHostToDevice, s));

  // per-cell groups of coefficient faces (fixedValue + processor), kept in
  // (patch, face) order by the stable sort: facePatchIndex/facePatchStart
  // of P:471-481 over all patches at once.
  auto group_cells = [&](const std::vector<int32_t> &sel, int32_t *&startOut, int32_t *&itemsOut) {
    const int32_t m = (int32_t)sel.size();
    startOut = A.alloc<int32_t>(n + 1);
    itemsOut = A.alloc<int32_t>(m);
    std::vector<int32_t> k(m);
    for (int32_t i = 0; i < m; ++i) k[i] = hCell[sel[i]];
    int32_t *dk = nullptr;
    LF_CUDA(cudaMallocAsync(&dk, sizeof(int32_t) * std::max(m, 1), s));
    LF_CUDA(cudaMemcpyAsync(dk, k.data(), sizeof(int32_t) * m, cudaMemcpyHostToDevice, s));
    LF_CUDA(cudaMemcpyAsync(itemsOut, sel.data(), sizeof(int32_t) * m, cudaMemcpyHostToDevice, s));
    sort_pairs_i32(s, dk, itemsOut, m, bits);
    launch_starts_from_sorted(s, dk, m, n, startOut);
    LF_CUDA(cudaFreeAsync(dk, s));
    LF_CUDA(cudaStreamSynchronize(s));
  };
  std::vector<int32_t> selBc, selProc;
  for (int32_t i = 0; i < B; ++i) {
    if (hType[i] != LF_PATCH_ZERO_GRADIENT) selBc.push_back(i);
    if (hType[i] == LF_PATCH_PROCESSOR) selProc.push_back(i);
  }
  int32_t *bcStart, *bcFace;
  group_cells(selBc, bcStart, bcFace);
  int32_t *pcStart = nullptr, *pcFace = nullptr;
  if (nproc > 0) group_cells(selProc, pcStart, pcFace);

  // ------------------------------------------------------- matrix
  LduDev &L = M->ld;
  L.diag = A.alloc<double>(n);
  L.upper = A.alloc<double>(F);
  L.writeUpper = 1;
  L.source = A.alloc<double>(n);
  L.bInt = A.alloc<double>(B);
  L.bBnd = A.alloc<double>(B);
  LF_CUDA(cudaMemsetAsync(L.bInt, 0, sizeof(double) * std::max(B, 1), s));
  LF_CUDA(cudaMemsetAsync(L.bBnd, 0, sizeof(double) * std::max(B, 1), s));

  MeshDev &md = M->md;
  md.n = n;
  md.F = F;
  md.ownerStart = ownerStart;
  md.nbr = nbr;
  md.losortStart = losortStart;
  md.losort = losort;
  md.losortOwner = losortOwner;
  md.magSf = magSf;
  md.delta = delta;
  md.V = V;
  md.bcStart = bcStart;
  md.bcFace = bcFace;
  md.bType = bType;
  md.bMagSf = bMag;
  md.bDelta = bDel;
  md.bValue = M->bValue;
  md.bSlot = bSlot;
  md.pcStart = pcStart;
  md.pcFace = pcFace;
  md.hasProc = nproc > 0;
  md.procMask = nullptr;
  if (nproc > 0) {
    std::vector<uint32_t> mask(((size_t)n + 31) / 32, 0u);
    for (int32_t fi = 0; fi < B; ++fi)
      if (hType[fi] == LF_PATCH_PROCESSOR) mask[hCell[fi] >> 5] |= 1u << (hCell[fi] & 31);
    unsigned *dm = A.alloc<unsigned>(mask.size());
    LF_CUDA(cudaMemcpyAsync(dm, mask.data(), sizeof(uint32_t) * mask.size(), cudaMemcpyHostToDevice, s));
    LF_CUDA(cudaStreamSynchronize(s));
    md.procMask = dm;
  }

  // -------------------------- full geometry (non-orthogonal correction path)
  // Internal face order and orientation: Sf is negated where the relabelled
  // owner > neighbour (the upper-triangular re-sort swapped the sides).
  // weights / nonOrthCorrectionVectors are then computed on the device from
  // the internal geometry (k_weights_corr).
  if (d->c) {
    M->hasGeom = true;
    std::vector<int32_t> fp(F);
    LF_CUDA(cudaMemcpyAsync(fp.data(), M->facePerm, sizeof(int32_t) * F, cudaMemcpyDeviceToHost, s));
    LF_CUDA(cudaStreamSynchronize(s));
    std::vector<double> sfA(3 * (size_t)F), cfA(3 * (size_t)F), cA(3 * (size_t)n), bsf(3 * (size_t)B);
    for (int32_t f = 0; f < F; ++f) {
      const int32_t src = fp[f];
      int32_t o = d->owner[src], nb = d->neighbour[src];
      if (!iperm.empty()) {
        o = iperm[o];
        nb = iperm[nb];
      }
      const double sg = o > nb ? -1.0 : 1.0;
      for (int k = 0; k < 3; ++k) {
        sfA[3 * (size_t)f + k] = sg * d->sf[3 * (size_t)src + k];
        cfA[3 * (size_t)f + k] = d->cf[3 * (size_t)src + k];
      }
    }
    for (int32_t c = 0; c < n; ++c) {
      const int32_t ci = iperm.empty() ? c : iperm[c];
      for (int k = 0; k < 3; ++k) cA[3 * (size_t)ci + k] = d->c[3 * (size_t)c + k];
    }
    for (int32_t p = 0, off = 0; p < d->n_patches; ++p) {
      const lf_patch_desc &P = d->patches[p];
      for (int32_t i = 0; i < P.n_faces; ++i)
        for (int k = 0; k < 3; ++k) bsf[(size_t)k * B + off + i] = P.sf[3 * (size_t)i + k];
      off += P.n_faces;
    }
    double *tmp = nullptr;
    const size_t tF = 3 * (size_t)std::max(F, 1), tN = 3 * (size_t)n;
    LF_CUDA(cudaMallocAsync(&tmp, sizeof(double) * (2 * tF + tN), s));
    LF_CUDA(cudaMemcpyAsync(tmp, sfA.data(), sizeof(double) * 3 * F, cudaMemcpyHostToDevice, s));
    LF_CUDA(cudaMemcpyAsync(tmp + tF, cfA.data(), sizeof(double) * 3 * F, cudaMemcpyHostToDevice, s));
    LF_CUDA(cudaMemcpyAsync(tmp + 2 * tF, cA.data(), sizeof(double) * tN, cudaMemcpyHostToDevice, s));
    GeomDev &g = M->geo;
    g.n = n;
    g.F = F;
    g.B = B;
    double *w = A.alloc<double>(F), *corr = A.alloc<double>(3 * (size_t)F), *SfS = A.alloc<double>(3 * (size_t)F);
    launch_weights_corr(s, F, owner, nbr, tmp, tmp + tF, tmp + 2 * tF, magSf, delta, w, corr, SfS);
    LF_CUDA(cudaFreeAsync(tmp, s));
    double *bSf = A.alloc<double>(3 * (size_t)B);
    LF_CUDA(cudaMemcpyAsync(bSf, bsf.data(), sizeof(double) * 3 * B, cudaMemcpyHostToDevice, s));
    std::vector<int32_t> selAll(B);
    for (int32_t i = 0; i < B; ++i) selAll[i] = i;
    int32_t *abStart, *abFace;
    group_cells(selAll, abStart, abFace);
    g.w = w;
    g.corr = corr;
    g.Sf = SfS;
    g.bSf = bSf;
    g.bW = g.bCorr = nullptr;
    // processor faces with cf/cn: the owner-side interpolation weight and the
    // correction vector of the coupled face (the internal-face formulas of
    // k_weights_corr with C_N = the coupled cell's centre), flat boundary order
    bool anyProc = false, allGeo = true;
    for (int32_t p = 0; p < d->n_patches; ++p)
      if (d->patches[p].type == LF_PATCH_PROCESSOR && d->patches[p].n_faces > 0) {
        anyProc = true;
        allGeo = allGeo && d->patches[p].cf != nullptr;
      }
    if (anyProc && allGeo) {
      std::vector<double> bw(B, 1.0), bc(3 * (size_t)B, 0.0);
      for (int32_t p = 0, off = 0; p < d->n_patches; ++p) {
        const lf_patch_desc &P = d->patches[p];
        if (P.type == LF_PATCH_PROCESSOR)
          for (int32_t i = 0; i < P.n_faces; ++i) {
            const double *Cp = d->c + 3 * (size_t)P.face_cells[i], *Cn = P.cn + 3 * (size_t)i;
            const double *Cf = P.cf + 3 * (size_t)i, *S = P.sf + 3 * (size_t)i;
            double so = 0.0, sn = 0.0;
            for (int k = 0; k < 3; ++k) {
              so = so + S[k] * (Cf[k] - Cp[k]);
              sn = sn + S[k] * (Cn[k] - Cf[k]);
            }
            so = std::fabs(so);
            sn = std::fabs(sn);
            const double sum = so + sn;
            bw[off + i] = std::fabs(sum) > 1e-150 ? sn / sum : 0.5;
            for (int k = 0; k < 3; ++k)
              bc[(size_t)k * B + off + i] = S[k] / P.mag_sf[i] - (Cn[k] - Cp[k]) * P.delta_coeffs[i];
          }
        off += P.n_faces;
      }
      double *dW = A.alloc<double>(B), *dC = A.alloc<double>(3 * (size_t)B);
      LF_CUDA(cudaMemcpyAsync(dW, bw.data(), sizeof(double) * B, cudaMemcpyHostToDevice, s));
      LF_CUDA(cudaMemcpyAsync(dC, bc.data(), sizeof(double) * 3 * B, cudaMemcpyHostToDevice, s));
      g.bW = dW;
      g.bCorr = dC;
      M->procGeom = true;
    }
    g.abStart = abStart;
    g.abFace = abFace;
    M->gradS = A.alloc<double>(3 * (size_t)n);
    M->lapSrc = A.alloc<double>(n);
    M->T0 = A.alloc<double>(n);
    LF_CUDA(cudaStreamSynchronize(s));
  }

  // ------------------------------------------ ELL slices for the solve
  // K = max faces per side (3 on hex meshes); built when 1 <= K <= 4 and the
  // packed owner-slot label fits (n < 2^29), else the CSR gather is used.
  md.K = 0;
  md.nbrE = md.loE = nullptr;
  md.codeE = nullptr;
  md.uniE = nullptr;
  md.offE = nullptr;
  md.ngE = 0;
  L.upperE = nullptr;
  md.KS = md.ldS = 0;  // full-row ELL: built at the end for K > 4 meshes
  md.symN = nullptr;
  L.symU = nullptr;
  if (F > 0 && n < (1 << 29)) {
    std::vector<int32_t> hs(n + 1), hl(n + 1);
    LF_CUDA(cudaMemcpyAsync(hs.data(), ownerStart, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost, s));
    LF_CUDA(cudaMemcpyAsync(hl.data(), losortStart, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost, s));
    LF_CUDA(cudaStreamSynchronize(s));
    int K = 0;
    for (int32_t c = 0; c < n; ++c) K = std::max({K, hs[c + 1] - hs[c], hl[c + 1] - hl[c]});
    if (K >= 1 && K <= 4) {
      const int KE = K <= 3 ? 3 : 4;  // kernels are specialised for 3 and 4 slots
      const int32_t ld = (n + 3) & ~3;
      int32_t *nbrE = A.alloc<int32_t>((size_t)KE * ld), *loE = A.alloc<int32_t>((size_t)KE * ld);
      L.upperE = A.alloc<double>((size_t)KE * ld);
      LF_CUDA(cudaMemsetAsync(L.upperE, 0, sizeof(double) * KE * (size_t)ld, s));
      md.K = KE;
      md.ldE = ld;
#if defined(LF_NO_ELL) && LF_NO_ELL
      L.writeUpper = 1;
#else
      L.writeUpper = 0;  // the solve reads upperE; upper on demand (ensure_upper)
#endif
      launch_build_ell(s, md, owner, KE, nbrE, loE);
      md.nbrE = nbrE;
      md.loE = loE;
      md.uniE = nullptr;
#if defined(LF_UNI) && LF_UNI
      {
        // uniform 32-cell label groups (kernels.cu, k_build_uni)
        md.ngE = (n + 31) / 32;
        int2 *uniE = A.alloc<int2>((size_t)KE * md.ngE);
        launch_build_uni(s, md, uniE);
        md.uniE = uniE;
      }
#endif
      if (ctx->compressedLabels) {
        // 16-bit label codes for the HBM-bound gathers (kernels.cu, k_build_ell16)
        md.ngE = (n + 31) / 32;
        uint32_t *codeE = A.alloc<uint32_t>((size_t)KE * ld);
        int2 *offE = A.alloc<int2>((size_t)KE * md.ngE);
        int32_t *dEsc = A.alloc<int32_t>(1);
        launch_build_ell16(s, md, codeE, offE, dEsc);
        LF_CUDA(cudaMemcpyAsync(&M->ell16Escapes, dEsc, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        LF_CUDA(cudaStreamSynchronize(s));
        md.codeE = codeE;
        md.offE = offE;
      }
    }
  }

  // ------------------------------------------------------ workspace
  const int BSZ = kernel_block_size();
  // Resident grid with EQUAL grid-stride trips for every block: with G0
  // co-resident blocks, T = ceil(blocks needed / G0) trips, G = ceil(need/T)
  // (e.g. 1M cells: 652 blocks x 6 trips instead of 740 blocks doing 5 or 6),
  // so no block idles at the phase end (ncu r1j: 31% of warp samples waited
  // at the grid barrier with the unbalanced grid).
#ifndef LF_SMUNIFORM
#define LF_SMUNIFORM 0
#endif
  auto balanced = [&](int g0) {
    const int need = (int)((n + BSZ - 1) / BSZ);
    if (need <= g0) return std::max(1, need);
    if (LF_SMUNIFORM) return g0;  // every SM holds the same number of blocks
    const int T = (need + g0 - 1) / g0;
    return (need + T - 1) / T;
  };
  auto grid = [&](int kid) { return Launch{balanced(occupancy_grid(kid, ctx->device)), BSZ}; };
  M->Lasm = grid(0);
  M->Lp1 = grid(1);
  M->Lp2 = grid(2);
  M->Lamul = grid(3);
  M->Lsetup = grid(4);
  M->Lsum = grid(5);
  // persistent kernel: contiguous chunks on an SM-uniform grid (every SM
  // holds the same number of blocks), or balanced grid-stride trips
  M->persistentGrid = persistent_chunked()
                          ? std::max(1, std::min(persistent_grid(ctx->device, md.K), (int)((n + 31) / 32)))
                      : persistent_tail()
                          ? std::max(1, std::min(persistent_grid(ctx->device, md.K), (int)((n + BSZ - 1) / BSZ)))
                          : balanced(persistent_grid(ctx->device, md.K));
  int maxGrid = std::max({M->Lasm.grid, M->Lp1.grid, M->Lp2.grid, M->Lamul.grid, M->Lsetup.grid, M->Lsum.grid,
                          M->persistentGrid});
  M->gridBar = A.alloc<unsigned>(2);  // {arrivals, generation}
  LF_CUDA(cudaMemsetAsync(M->gridBar, 0, 2 * sizeof(unsigned), s));
  Workspace &ws = M->ws;
  ws.maxGrid = maxGrid;
  // Moving psi += alpha p into the wait of the beta barrier hides it in the
  // barrier latency but re-reads p: a win while an iteration's working set
  // (~96n + 16F bytes) is within ~1.5x the L2 — latency-bound sizes (r2h:
  // 100^3 -4.8% time) — and a loss once HBM-bound (200^3 +3.4%).
  {
    int l2 = 0;
    LF_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, ctx->device));
    const double bytesIter = 96.0 * n + 16.0 * F;
    M->l2Resident = bytesIter <= 1.5 * (double)l2;
    M->stashOK = persistent_tail() && (int64_t)n / ((int64_t)M->persistentGrid * BSZ) + 1 <= stash_trips();
    ws.idleFlush = (M->l2Resident && M->stashOK) ? 1 : 0;
    // HBM-bound solve, next-trip L2 prefetch (LF_LPF): the L2 must hold the
    // neighbour-reuse window (cells c - bw .. c + bw), the current trip and
    // the prefetched one at the iteration's bytes per cell.  Measured
    // crossover: 200^3 (55 MB by this count) +0-6% (r6b/r6c/r6zb), 300^3
    // (69.5 MB) -10% (r6zb), 400^3 (90 MB) -5% (r6b).
    const double trip = (double)M->persistentGrid * BSZ;
    const double pfBytes = (2.0 * (double)M->bandwidth + 2.0 * trip) * bytesIter / std::max<double>(n, 1);
    M->pfFits = !M->l2Resident && pfBytes <= 0.5 * (double)l2;
    ws.l2pf = M->pfFits ? 1 : 0;
  }
  ws.r = A.alloc<double>(n);
  ws.w = A.alloc<double>(n);
  ws.q = A.alloc<double>(n);
#if defined(LF_W88) && LF_W88 == 2
  ws.rDiag = A.alloc<double>(n);
#endif
  ws.p[0] = A.alloc<double>(n);
  ws.p[1] = A.alloc<double>(n);
  ws.partials = A.alloc<double>(4 * (size_t)maxGrid);
  ws.dynCap = (int)(n / BSZ) + 2 * maxGrid + 2;
  ws.partialsD = A.alloc<double>(2 * (size_t)ws.dynCap);
  ws.tickets = A.alloc<unsigned>(16);
  LF_CUDA(cudaMemsetAsync(ws.tickets, 0, 16 * sizeof(unsigned), s));
  ws.ctl = A.alloc<PcgCtl>(1);
  LF_CUDA(cudaMemsetAsync(ws.ctl, 0, sizeof(PcgCtl), s));
  ws.gsum = A.alloc<RedSlots>(1);
  LF_CUDA(cudaMemsetAsync(ws.gsum, 0, sizeof(RedSlots), s));
  ws.lsum = ctx->comm ? A.alloc<RedSlots>(1) : ws.gsum;
  if (ctx->comm) LF_CUDA(cudaMemsetAsync(ws.lsum, 0, sizeof(RedSlots), s));
  ws.sendBuf = A.alloc<double>(nproc);
  ws.pH[0] = A.alloc<double>(nproc);
  ws.pH[1] = A.alloc<double>(nproc);
  // one cudaMalloc block (IPC-exportable for the peer-memory transport):
  // [mailbox flags 2*MAXP u32 | mailbox vals 2*MAXP*4 f64 | recvT[2] | recvW]
  {
    auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
    M->offFlags = 0;
    M->offVals = up(2 * LF_MAXP * sizeof(unsigned));
    M->offRecvT = up(M->offVals + 2 * LF_MAXP * 4 * sizeof(double));
    M->offRecvW = up(M->offRecvT + 2 * sizeof(double) * std::max(nproc, 1));  // recvT[2][nproc]
    M->offRecvX = up(M->offRecvW + sizeof(double) * std::max(nproc, 1));      // recvW[nproc]
    M->p2pBytes = up(M->offRecvX + 3 * sizeof(double) * std::max(nproc, 1));  // recvX[3][nproc]
    M->p2pBlock = A.alloc<char>(M->p2pBytes);
    LF_CUDA(cudaMemsetAsync(M->p2pBlock, 0, M->p2pBytes, s));
    ws.recvT = reinterpret_cast<double *>(M->p2pBlock + M->offRecvT);
    ws.recvW = reinterpret_cast<double *>(M->p2pBlock + M->offRecvW);
    ws.recvX = reinterpret_cast<double *>(M->p2pBlock + M->offRecvX);
  }
  std::memset(&ws.p2p, 0, sizeof(ws.p2p));
  ws.sendCell = A.alloc<int32_t>(nproc);
  LF_CUDA(cudaMemcpyAsync(ws.sendCell, sendCells.data(), sizeof(int32_t) * nproc, cudaMemcpyHostToDevice, s));
  if (nproc > 0) {
    // cells without / with processor faces (the NCCL iteration overlaps the
    // w halo with the first group's Amul)
    std::vector<char> bnd(n, 0);
    for (int32_t c : sendCells) bnd[c] = 1;
    std::vector<int32_t> ci, cb;
    for (int32_t c = 0; c < n; ++c) (bnd[c] ? cb : ci).push_back(c);
    M->nInt = (int32_t)ci.size();
    M->nBnd = (int32_t)cb.size();
    M->cellsInt = A.alloc<int32_t>(ci.size());
    M->cellsBnd = A.alloc<int32_t>(cb.size());
    if (!ci.empty())
      LF_CUDA(cudaMemcpyAsync(M->cellsInt, ci.data(), sizeof(int32_t) * ci.size(), cudaMemcpyHostToDevice, s));
    LF_CUDA(cudaMemcpyAsync(M->cellsBnd, cb.data(), sizeof(int32_t) * cb.size(), cudaMemcpyHostToDevice, s));
    LF_CUDA(cudaStreamSynchronize(s));  // the host vectors go out of scope
  }
  M->T = A.alloc<double>(n);
  LF_CUDA(cudaMemsetAsync(M->T, 0, sizeof(double) * n, s));
  M->scratch = A.alloc<double>(n);
  LF_CUDA(cudaMallocHost(&M->hctl, sizeof(PcgCtl)));
  std::memset(M->hctl, 0, sizeof(PcgCtl));

  // global cell count for gAverage (allreduce once)
  double nloc = (double)n;
  if (ctx->comm) {
    double *dn = nullptr;
    LF_CUDA(cudaMallocAsync(&dn, 2 * sizeof(double), s));
    LF_CUDA(cudaMemcpyAsync(dn, &nloc, sizeof(double), cudaMemcpyHostToDevice, s));
    nccl_allreduce_sum(ctx->comm, dn, dn + 1, 1, s);
    LF_CUDA(cudaMemcpyAsync(&M->nTotal, dn + 1, sizeof(double), cudaMemcpyDeviceToHost, s));
    LF_CUDA(cudaFreeAsync(dn, s));
  } else {
    M->nTotal = nloc;
  }
  // ---------------------------------------------- full-row ELL (K > 4)
  // Meshes with more than 4 faces on a side (e.g. randomly numbered ones)
  // take the full-row rows of the DIC for the Amul gathers when every cell
  // has at most 8 neighbours: labels and coefficients coalesced, no
  // start offsets, no face -> coefficient indirection; else the CSR gather.
  if (md.K == 0 && F > 0 && n < (1 << 29) && !LF_NO_SYM_ROWS) {
    std::vector<int32_t> hs(n + 1), hl(n + 1);
    LF_CUDA(cudaMemcpyAsync(hs.data(), ownerStart, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost, s));
    LF_CUDA(cudaMemcpyAsync(hl.data(), losortStart, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost, s));
    LF_CUDA(cudaStreamSynchronize(s));
    int32_t deg = 0;
    for (int32_t c = 0; c < n; ++c) deg = std::max(deg, (hs[c + 1] - hs[c]) + (hl[c + 1] - hl[c]));
    if (deg <= 8) build_rows(M);
  }

  LF_CUDA(cudaStreamSynchronize(s));
  LF_CUDA(cudaGetLastError());
  M->ldu.mesh = M;
}

namespace lf {
void mesh_create_impl(lf_context *ctx, const lf_mesh_desc *d, lf_mesh **out) {
  LF_REQUIRE(ctx != nullptr && out != nullptr, "NULL context or out");
  LF_CUDA(cudaSetDevice(ctx->device));
  std::unique_ptr<lf_mesh> M(new lf_mesh());
  build_mesh(ctx, d, M.get());
  *out = M.release();
}
}  // namespace lf
