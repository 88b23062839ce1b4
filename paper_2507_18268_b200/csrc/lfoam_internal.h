// Internal declarations of liblfoam.so (not part of the ABI).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "lfoam.h"

namespace lf {

struct Error {
  lf_status st;
  std::string msg;
};

#define LF_CUDA(x)                                                                     \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess)                                                             \
      throw ::lf::Error{e_ == cudaErrorMemoryAllocation ? LF_ERR_OOM : LF_ERR_CUDA,    \
                        std::string(#x) + ": " + cudaGetErrorString(e_)};              \
  } while (0)

#define LF_REQUIRE(cond, msg)                                                          \
  do {                                                                                 \
    if (!(cond)) throw ::lf::Error{LF_ERR_INVALID_ARG, (msg)};                         \
  } while (0)

// ------------------------------------------------------------ device memory
// Every device array of a mesh is allocated once at mesh_create.
struct DevArena {
  std::vector<void *> ptrs;
  int64_t bytes = 0;
  template <class T>
  T *alloc(size_t n) {
    void *p = nullptr;
    size_t b = sizeof(T) * (n > 0 ? n : 1);
    LF_CUDA(cudaMalloc(&p, b));
    ptrs.push_back(p);
    bytes += (int64_t)b;
    return static_cast<T *>(p);
  }
  void release() {
    for (void *p : ptrs) cudaFree(p);
    ptrs.clear();
    bytes = 0;
  }
  ~DevArena() { release(); }
};

// ---------------------------------------------------------- solver control
// Device-resident PCG state.  Kernels read it at entry; only the LAST block
// of a launch (ticket order) writes it, after every block has read it, so a
// launch never observes its own updates.  See DESIGN.md "Device-side loop".
struct PcgCtl {
  double tol, relTol;
  int32_t maxIter, minIter;
  double nTotal;        // global cell count (gAverage denominator)
  double *psi;          // solution vector of the current solve
  double normFactor, initRes, finRes;
  double wArA, alpha;
  int32_t it, stop, converged, singular;
  int32_t precond;      // lf_preconditioner of the current solve (host side)
  int32_t fault;        // set by a kernel: the GAMG coarsest matrix is not SPD
};

// Global sums consumed by the next launch (after the allreduce in multi-GPU).
struct RedSlots {
  double setup[3];  // sum(|A psi - tmp| + |b - tmp|), sum|r|, sum w.r
  double p1[2];     // sum p.q, sum psi
  double p2[2];     // sum|r|, sum w.r
  double p1x[2];    // phase 1 split (NCCL halo overlap): the interior cells' p.q, psi
};

// Read-only view of a mesh on the device (kernel argument, by value).
struct MeshDev {
  int32_t n, F;
  const int32_t *ownerStart, *nbr, *losortStart, *losort, *losortOwner;
  const double *magSf, *delta, *V;
  // boundary faces with coefficients (fixedValue + processor) grouped per cell
  const int32_t *bcStart, *bcFace;
  const int8_t *bType;  // per flat boundary face (lf_patch_type)
  const double *bMagSf, *bDelta, *bValue;
  const int32_t *bSlot;  // per flat boundary face: halo slot (processor) or -1
  // processor faces grouped per cell (Amul interface term); null if none
  const int32_t *pcStart, *pcFace;
  int32_t hasProc;
  // bit c of procMask[c / 32]: cell c has processor faces (one broadcast
  // word per warp instead of a pcStart pair per cell in the hot loops)
  const unsigned *procMask;
  // ELL slices of the same addressing (K = max faces per side, 0 = none);
  // slot k of cell c at k*n + c.  See kernels.cu header.
  int32_t K, ldE;  // ldE: slab stride (n rounded up to 4: 16-byte aligned slabs)
  const int32_t *nbrE, *loE;
  // the same labels compressed to 16 bits each (one u32 per slot and cell,
  // kernels.cu "compressed ELL labels"): codeE[k*ldE + c], per-(slot, 32-cell
  // group) offsets offE[k*ngE + c/32]; escapes fall back to nbrE/loE.  null:
  // not built (the persistent solve then gathers through nbrE/loE)
  const uint32_t *codeE;
  const int2 *offE;
  int32_t ngE;
  // uniform 32-cell groups (LF_UNI): per (slot, group) {nbr - c, (kk << 29)
  // | (c - owner)} when every cell of the group has it (> 0), 0 when none
  // has the slot, -1: the labels differ -> read nbrE / loE.  null: not built
  const int2 *uniE;
  // full-row ELL (the DIC rows, DicDev): used by the Amul gathers of meshes
  // with more than 4 faces on a side (K == 0) and at most 8 neighbours
  int32_t KS, ldS;
  const int32_t *symN;
  // spatially varying DT (§8(f) row 2): face / boundary diffusivities, or
  // null (the scalar DT argument of the kernels)
  const double *gammaF, *gammaB;
};

struct LduDev {
  double *upperE;  // [K*n] ELL copy of upper (owner side), 0 in padding
  double *diag, *upper, *source;
  double *bInt, *bBnd;  // per flat boundary face: internalCoeffs, boundaryCoeffs
  double *symU;    // [KS*ldS] full-row ELL coefficients (DIC meshes), or null
  int32_t ldS;     // its slab stride
  // 0: the assembly writes the coefficients only to upperE (ELL meshes whose
  // consumers all read the ELL copy); `upper` is rebuilt from upperE on
  // demand (launch_upper_from_ell: export, full-row fill).  1: both.
  int32_t writeUpper;
};

// DIC preconditioner (dic.cuh), built on first use.
// Full-row ELL: slot k of cell c at k*ldS + c holds its k-th neighbour in
// ascending label order (lower neighbours, then upper) — for upper-triangular
// face order that is the order of the faces in OpenFOAM's sequential loops.
// Label bit 30 marks a neighbour on level 0; empty slots are -1.
constexpr int DIC_L0BIT = 1 << 30;
struct DicDev {
  int32_t L;               // number of levels (>= 1)
  int32_t contig;          // 1: level l = cells [lvlStart[l], lvlStart[l+1])
  const int32_t *lvlStart; // [L+1] device
  const int32_t *lvlCells; // [n] cells ordered by level (null when contig)
  int32_t KS, ldS;         // row width (6 or 8) and slab stride
  const int32_t *symN;     // [KS*ldS]
  double *rD, *rDu;        // reciprocal DIC diagonal; unreciprocated (levels >= 1)
};

// GAMG preconditioner (reading A43 in DESIGN.md;
// gamg.cpp builds the hierarchy once per mesh, gamg.cuh runs it).  Level 0
// is the mesh: its rows are the full-row ELL (DicDev.symN / LduDev.symU),
// D = LduDev.diag, U = LduDev.upper; only rD is stored here.  Levels >= 1
// hold CSR rows (neighbours ascending, entry -> face of the level).
constexpr int GAMG_MAXL = 30;
struct GamgLevelDev {
  int32_t n, nf;
  const int32_t *rowStart, *rowCol, *rowFace;  // levels >= 1: [n+1], [2nf], [2nf]
  double *rowU;                                // levels >= 1: [2nf] U of each row entry (per solve)
  const int32_t *faceL, *faceU;                // coarsest level only: [nf]
  double *D, *rD, *U;                          // [n], [n], [nf] (level 0: D, U alias the system)
  double *b, *x;                               // V-cycle right-hand side / correction (levels >= 1)
  // restriction to level l+1 (l < L): cell -> coarse cell; coarse cell ->
  // members (ascending) and internal faces (ascending); coarse face -> fine
  // faces (ascending)
  const int32_t *agg;
  const int32_t *memStart, *mem;
  const int32_t *inStart, *inFace;
  const int32_t *cfStart, *cfFace;
};
struct GamgDev {
  int32_t L;     // index of the coarsest level (levels 0..L)
  int32_t tail;  // levels >= tail (>= 1) run in one block (no grid barriers)
  double *inv;   // [nL*nL] inverse of the coarsest matrix (row major)
  double *chol;  // [nL*nL] its Cholesky factor (scratch)
  double *ycol;  // [nL*nL] forward-substitution scratch, column k at k*nL
  GamgLevelDev lv[GAMG_MAXL + 1];
};

// ---------------------------------------------------------------- kernels
struct Launch {
  int grid, block;
};

// Peer-memory (CUDA IPC / NVLink P2P) transport, see DESIGN.md §9.
// Mailbox of rank q: flags[2 parity][LF_MAXP] (u32) and vals[2][LF_MAXP][4]
// (f64) in one IPC-exported allocation; every rank holds mapped pointers to
// all mailboxes.  P == 0: transport off.
constexpr int LF_MAXP = 16;
constexpr int LF_MAXSEG = 16;  // processor patches (halo segments) per rank
struct P2PDev {
  int32_t P, rank;
  unsigned *seq;              // own allreduce sequence counter (device)
  unsigned *flags[LF_MAXP];   // mailbox flags of every rank (mapped)
  double *vals[LF_MAXP];      // mailbox values of every rank (mapped)
  // halo destinations, base + offset per segment: local send slots
  // [segBeg[g], segBeg[g+1]) go to dstW[g][slot - segBeg[g]] in the
  // neighbour's recvW (own buffer for self pairs), likewise recvT, which is
  // double-buffered by the parity tPar of the push (a standalone ldu_amul on
  // one rank may still read parity p while a faster rank pushes p ^ 1)
  int32_t nseg, tPar;
  int32_t segBeg[LF_MAXSEG + 1];
  double *dstW[LF_MAXSEG];
  double *dstT[2][LF_MAXSEG];
  // vector halo (the gradient, the DT field): component k of send slot s of
  // segment g goes to dstX[g][k * xStr[g] + (s - segBeg[g])] (xStr = the
  // destination rank's processor-face count)
  double *dstX[LF_MAXSEG];
  int32_t xStr[LF_MAXSEG];
};

struct Workspace {
  double *r, *w, *q, *p[2];
  double *rDiag;        // 1/diag of the current solve (LF_W88 == 2 variant only)
  double *partials;     // [4 * maxGrid]
  double *partialsD;    // [2 * dynCap] per-unit sums of the run-time scheduled phase-1 trips
  int dynCap;           // capacity of partialsD per sum
  int dynTrips;         // HBM-bound persistent solve: phase-1 trips scheduled at run time (solver.cpp)
  unsigned *tickets;    // [16]
  PcgCtl *ctl;
  RedSlots *gsum;       // global sums
  RedSlots *lsum;       // local sums (== gsum when single rank or P2P)
  // processor-patch halos (slot = flat processor-face index, n_proc slots)
  double *sendBuf;      // staging for NCCL / local copies
  double *recvT, *recvW;  // neighbour T (assembly; [2][n_proc] by push parity) and w (PCG) at each slot
  double *pH[2];        // p at the halo slots, recomputed locally (double-buffered like p)
  double *recvX;        // [3][n_proc] vector halo (gradient, DT field)
  int32_t *sendCell;    // [n_proc] local cell of each send slot
  int maxGrid;
  int idleFlush;        // persistent solve: psi flush in the beta-barrier wait (see mesh.cpp)
  int l2pf;             // HBM-bound persistent solve: next-trip L2 prefetch (see mesh.cpp)
  P2PDev p2p;
};

// kernels.cu launchers (all stream-ordered, no host sync)
void launch_sum(cudaStream_t s, const Launch &L, const MeshDev &m, const double *x, const Workspace &ws,
                double *out);
void launch_assemble(cudaStream_t s, const Launch &L, const MeshDev &m, const LduDev &a,
                     double DT, double rDeltaT, const double *T, const double *halo,
                     bool setup, const Workspace &ws, const double *T0 = nullptr,
                     const double *lapSrc = nullptr);

// ---------------------------------------- non-orthogonal correction path
// (nonorth.cu).  Internal face order / numbering, SoA
// vectors: component k of item i at k*count + i.
struct GeomDev {
  int32_t n, F, B;
  const double *w;        // [F] owner interpolation weights (Listing "weights")
  const double *corr;     // [3][F] nonOrthCorrectionVectors
  const double *Sf;       // [3][F] area vectors (owner -> neighbour)
  const double *bSf;      // [3][B] boundary area vectors (outward), patch order
  const int32_t *abStart, *abFace;  // per-cell groups of ALL boundary faces
  // processor faces (meshes whose processor patches carry cf/cn; else null):
  // owner-side interpolation weight [B] and correction vectors [3][B]
  // (flat boundary order; 1 / 0 on non-coupled faces)
  const double *bW, *bCorr;
};
void launch_weights_corr(cudaStream_t s, int32_t F, const int32_t *owner, const int32_t *nbr,
                         const double *SfA, const double *CfA, const double *CA, const double *magSf,
                         const double *delta, double *w, double *corr, double *SfS);
void launch_grad(cudaStream_t s, const Launch &L, const MeshDev &m, const GeomDev &g, const double *x,
                 const double *halo, double *gradS, double *gradA);
void launch_grad_bc(cudaStream_t s, const MeshDev &m, const GeomDev &g, const int32_t *bCell,
                    const double *x, const double *gradS, double *bgradA);
void launch_face_gamma(cudaStream_t s, const MeshDev &m, const GeomDev &g, const int32_t *owner,
                       const int32_t *bCell, const double *DTc, const double *haloDT, double *gammaF,
                       double *gammaB);
void launch_lap_corr(cudaStream_t s, const Launch &L, const MeshDev &m, const GeomDev &g, double DT,
                     const double *gradS, const double *haloG, int32_t nproc, double *lapSrc);
// vector halo through the peer-memory transport: x[k*stride + cell] of the
// processor-face cells into the neighbours' recvX, ordered by an allreduce
void launch_push_x(cudaStream_t s, const Launch &L, const MeshDev &m, const double *x, int64_t stride, int ncomp,
                   const Workspace &ws, double *out);
void launch_pcg_setup(cudaStream_t s, const Launch &L, const MeshDev &m, const LduDev &a,
                      const double *halo, const Workspace &ws);
void launch_phase1(cudaStream_t s, const Launch &L, const MeshDev &m, const LduDev &a,
                   const Workspace &ws);
// phase 1 over a cell list: part 1 = the cells without processor faces (sums
// into p1x, no state commit), part 2 = the cells with them (sums + p1x into
// p1, commits the state) — the halo-overlapped NCCL iteration
void launch_phase1_part(cudaStream_t s, const Launch &L, const MeshDev &m, const LduDev &a, const Workspace &ws,
                        int part, const int32_t *cells, int32_t count);
void launch_phase2(cudaStream_t s, const Launch &L, const MeshDev &m, const LduDev &a,
                   const Workspace &ws);
void launch_amul(cudaStream_t s, const Launch &L, const MeshDev &m, const LduDev &a,
                 const double *halo, const double *x, double *y);
int persistent_grid(int device, int K);
bool persistent_tail();  // LF_TAIL: SM-uniform grid, evenly spread tail trip
int stash_trips();       // max grid-stride trips of the L2-resident variant (0: none)
int dynamic_trips_pct();  // default % of phase-1 trips scheduled at run time (HBM-bound variant)
bool persistent_chunked();
void launch_pcg_persistent(cudaStream_t s, int grid, const MeshDev &m, const LduDev &a,
                           const Workspace &ws, unsigned *bar);
// DIC (dic.cuh)
int dic_grid(int device, int KS);  // co-resident grid of the DIC solve kernel
void launch_pcg_dic(cudaStream_t s, int grid, const MeshDev &m, const LduDev &a, const DicDev &d,
                    const Workspace &ws, unsigned *bar);
void launch_sym_fill(cudaStream_t s, const Launch &L, const MeshDev &m, const LduDev &a);
// standalone level passes (ldu_precondition): factor pass l (0 = levels 0 and
// 1), forward level l >= 1, backward level l; w = M^-1 r without r update
void launch_dic_factor_level(cudaStream_t s, const Launch &L, const MeshDev &m, const LduDev &a,
                             const DicDev &d, int l);
void launch_dic_sweep_level(cudaStream_t s, const Launch &L, const MeshDev &m, const LduDev &a,
                            const DicDev &d, int l, bool forward, const double *r, double *w);
void launch_diag_precondition(cudaStream_t s, const Launch &L, int32_t n, const double *diag,
                              const double *r, double *w);
// GAMG (gamg.cuh): co-resident grid; the persistent GAMG-PCG solve; one
// application w = M^-1 r (Galerkin set-up + V-cycle) as a cooperative launch.
// g: device copy of the hierarchy.
int gamg_grid(int device, const MeshDev &m);
void launch_pcg_gamg(cudaStream_t s, int grid, const MeshDev &m, const LduDev &a, const GamgDev *g,
                     const Workspace &ws, unsigned *bar);
void launch_gamg_apply(cudaStream_t s, int grid, const MeshDev &m, const LduDev &a, const GamgDev *g,
                       const double *r, double *w, const Workspace &ws, unsigned *bar);
void launch_pack_x(cudaStream_t s, int32_t nsend, const int32_t *cells, const double *x,
                   double *buf);
void launch_set_ctl(cudaStream_t s, PcgCtl *ctl, const PcgCtl &value);  // *ctl = value, stream-ordered
void launch_permute(cudaStream_t s, int32_t n, const int32_t *idx, const double *in, double *out,
                    bool scatter);
void launch_gather_f64(cudaStream_t s, int64_t n, const int32_t *idx, const double *in,
                       double *out);

// mesh-build kernels (kernels.cu)
void launch_iota(cudaStream_t s, int32_t *a, int64_t n);
void launch_starts_from_sorted(cudaStream_t s, const int32_t *sorted, int64_t m, int32_t n,
                               int32_t *starts);
void launch_split_keys(cudaStream_t s, const uint64_t *keys, int64_t m, int32_t *lo, int32_t *hi);
void launch_make_keys(cudaStream_t s, const int32_t *a, const int32_t *b, int64_t m,
                      uint64_t *keys);
void launch_gather_i32(cudaStream_t s, int64_t n, const int32_t *idx, const int32_t *in,
                       int32_t *out);
void launch_build_ell(cudaStream_t s, const MeshDev &m, const int32_t *owner, int32_t K, int32_t *nbrE,
                      int32_t *loE);
// compressed labels from nbrE/loE (md.K, md.ldE, md.nbrE, md.loE set);
// *nEsc (device int, zeroed here) receives the number of escaped entries
void launch_build_ell16(cudaStream_t s, const MeshDev &m, uint32_t *codeE, int2 *offE, int32_t *nEsc);
void launch_build_uni(cudaStream_t s, const MeshDev &m, int2 *uniE);  // md.K, ldE, ngE, nbrE, loE set
void launch_upper_from_ell(cudaStream_t s, const MeshDev &m, const LduDev &a);  // upper[f] <- upperE
// CUB wrappers (kernels.cu): stable radix sort of (key, value) pairs.
void sort_pairs_u64(cudaStream_t s, uint64_t *keys, int32_t *vals, int64_t m, int end_bit);
void sort_pairs_i32(cudaStream_t s, int32_t *keys, int32_t *vals, int64_t m, int end_bit);

int kernel_block_size();
int occupancy_grid(int kernel_id, int device);  // resident-grid size for a kernel

}  // namespace lf
