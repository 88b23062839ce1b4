// Host-side objects behind the opaque ABI handles.
#pragma once
#include <array>
#include <functional>
#include <string>
#include <vector>

#include "lfoam_internal.h"

namespace lf {

// ------------------------------------------------------------------ comm
// NCCL, loaded with dlopen at lf_comm_init (no link-time dependency).
struct Nccl;
Nccl *nccl_load();  // throws Error{LF_ERR_NCCL} if unavailable
void nccl_unique_id(void *out128);
void *nccl_comm_init(const void *uid128, int nranks, int rank, int device);
void nccl_comm_destroy(void *comm);
void *nccl_comm_split(void *comm, int rank);
void nccl_allreduce_sum(void *comm, const double *send, double *recv, size_t count, cudaStream_t s);
void nccl_group_start();
void nccl_group_end();
void nccl_send(void *comm, const double *buf, size_t count, int peer, cudaStream_t s);
void nccl_recv(void *comm, double *buf, size_t count, int peer, cudaStream_t s);
void nccl_check_async(void *comm);

}  // namespace lf

struct lf_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool ownStream = false;
  int nranks = 1, rank = 0;
  void *comm = nullptr;  // ncclComm_t (transport NCCL): reductions, on `stream`
  // NCCL halos overlapped with the interior Amul: a split communicator on its
  // own stream; evPacked (compute -> comm) / evHalo (comm -> compute)
  void *commHalo = nullptr;
  cudaStream_t commStream = nullptr;
  cudaEvent_t evPacked = nullptr, evHalo = nullptr;
  bool overlapHalo = true;  // LF_OPT_OVERLAP_HALO
  bool p2p = false;      // transport: peer memory (lf_p2p_init)
  int smCount = 0;
  // instrumentation
  bool instrument = false;
  bool capturing = false;  // stream capture in progress: no events, no counting
  bool useGraphs = true;   // replay iteration chunks as CUDA graphs
  bool persistent = true;  // single-rank, no processor patches: one cooperative launch per solve
  int solveVariant = 0;    // LF_OPT_SOLVE_VARIANT: 0 by mesh size, 1 L2-resident, 2 HBM-bound
  int dynPct = -1;         // LF_OPT_DYNAMIC_TRIPS: % of phase-1 trips scheduled at run time (-1 default)
  int l2Prefetch = 0;      // LF_OPT_L2_PREFETCH: 0 by mesh (lf_mesh::pfFits), 1 on, 2 off
  bool compressedLabels = false;  // LF_OPT_COMPRESSED_LABELS (mesh_create; r4d: slower, off)
  struct Pending {
    int kind;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> evFree;
  std::array<int64_t, LF_K_COUNT> kLaunches{};
  std::array<double, LF_K_COUNT> kMs{};
  int64_t launches = 0;

  // Launch wrapper: counts the launch and, if instrumented, brackets it
  // with CUDA events on the context stream.
  void launch(int kind, const std::function<void()> &fn);
  void harvest();  // after a stream sync: accumulate event timings
  cudaEvent_t event();
  ~lf_context();
};

struct HaloSeg {
  int32_t offset, count, peer;  // slots [offset, offset+count) of send/recv buffers
  int32_t partner;              // self pairs: index of the partner segment, else -1
};

struct lf_ldu {
  lf_mesh *mesh = nullptr;
  bool assembled = false;
};

struct lf_mesh {
  lf_context *ctx = nullptr;
  int32_t n = 0, F = 0, B = 0, nproc = 0;
  int32_t nPatches = 0;
  lf::DevArena arena;
  lf::MeshDev md{};
  lf::LduDev ld{};
  lf::Workspace ws{};
  lf::Launch Lasm{}, Lp1{}, Lp2{}, Lamul{}, Lsetup{}, Lsum{};
  std::vector<int32_t> patchType, patchStart, patchRank;
  std::vector<HaloSeg> segs;
  bool renumbered = false;
  int32_t *facePerm = nullptr;   // internal face -> caller face
  int32_t *cellPerm = nullptr;   // internal cell -> caller cell (renumbered only)
  int32_t *cellIperm = nullptr;  // caller cell -> internal cell (renumbered only)
  int32_t *ownerInt = nullptr;   // internal owner per internal face (export)
  int32_t *bCell = nullptr;      // per flat boundary face (internal numbering)
  double *bValue = nullptr;
  double *T = nullptr;
  double *scratch = nullptr;     // n doubles (permutation staging)
  lf::PcgCtl *hctl = nullptr;    // pinned host mirror
  double nTotal = 0.0;
  bool sumPsiValid = false;
  int32_t lastIters = -1;
  bool broken = false;
  lf_ldu ldu;
  bool upperStale = false;    // the last assembly wrote upperE only (LduDev.writeUpper == 0)
  // CUDA graphs of 2^i PCG iterations (captured once per mesh, replayed)
  static constexpr int kMaxGraphLog = 8;
  cudaGraphExec_t chunkGraph[kMaxGraphLog] = {};
  int kernelsPerIteration = 0;
  int persistentGrid = 0;     // co-resident grid of k_pcg_persistent
  bool l2Resident = false;    // an iteration's working set fits ~1.5x the L2 (mesh.cpp)
  bool stashOK = false;       // few enough trips per thread for the L2-resident variant
  bool pfFits = false;        // HBM-bound solve: next-trip L2 prefetch fits the L2 (mesh.cpp)
  int64_t bandwidth = 0;      // max |neighbour - owner| over internal faces (internal numbering)
  // NCCL transport, halo overlapped with the interior Amul: phase 1 split
  // into the cells without processor faces (interior) and those with
  int32_t *cellsInt = nullptr, *cellsBnd = nullptr;
  int32_t nInt = 0, nBnd = 0;
  bool haloPending = false;   // a w halo was started on the comm stream and not yet waited for
  int32_t ell16Escapes = -1;  // escaped compressed-label entries (-1: not built)
  unsigned *gridBar = nullptr;  // device {count, generation}
  // peer-memory transport: one IPC-exportable block [flags | vals | recvT | recvW]
  char *p2pBlock = nullptr;
  size_t p2pBytes = 0, offFlags = 0, offVals = 0, offRecvT = 0, offRecvW = 0, offRecvX = 0;
  std::vector<void *> ipcOpened;  // peer blocks mapped with cudaIpcOpenMemHandle
  bool p2pConnected = false;
  int tPar = 0;  // parity of the last peer-memory T halo push (recvT double buffer)
  // recvT half holding the current T halo (parity 0 for host-side exchanges)
  double *haloT() { return ws.recvT + (p2pConnected ? (size_t)tPar * (size_t)nproc : 0); }
  // non-orthogonal correction path (full geometry given at mesh_create)
  bool hasGeom = false;
  bool procGeom = false;     // processor patches carry cf/cn (corrected / DT paths across ranks)
  lf::GeomDev geo{};
  double *gradS = nullptr;   // [3][n] fvc::grad(T), SoA
  double *lapSrc = nullptr;  // [n] explicit laplacian correction source
  double *T0 = nullptr;      // [n] old-time T of the current step (correctors)
  // spatially varying DT (LF_FIELD_DT): cell field and face diffusivities
  double *DTc = nullptr, *gammaF = nullptr, *gammaB = nullptr;
  bool dtSet = false;
  lf::MeshDev mdVar{};       // md with gammaF/gammaB set (variable_DT solves)
  // DIC preconditioner: levels + full-row ELL, built on
  // first use (precond.cpp)
  bool dicBuilt = false;
  lf::DicDev dic{};
  int dicGrid = 0;            // co-resident grid of k_pcg_dic
  std::vector<int32_t> hLvlStart;  // host copy of the level starts
  // GAMG preconditioner (reading A43): agglomeration
  // hierarchy built on first use (gamg.cpp); hGamg holds the device pointers
  bool gamgBuilt = false;
  bool gamgFormed = false;       // a GAMG solve / application formed the coarse matrices
  lf::GamgDev hGamg{};
  lf::GamgDev *dGamg = nullptr;  // device copy (kernel argument)
  int gamgGrid = 0;              // co-resident grid of k_pcg_gamg
  std::vector<std::array<int32_t, 2>> gamgLevels;  // {cells, faces} per level
  ~lf_mesh();
};

namespace lf {
// solver.cpp
void solve_loop(lf_mesh *M, const lf_solver_controls *c, double *psi, bool fromAssembly,
                const lf_laplacian_params *p, lf_solver_perf *out, const double *T0 = nullptr,
                const double *lapSrc = nullptr);
// nonorth path (solver.cpp): gradS <- grad(x), lapSrc <- correction of gradS
void correction_source(lf_mesh *M, const MeshDev &md, double DT, const double *x);
void require_corrected(const lf_mesh *M);
// the MeshDev a solve with params p assembles with (variable DT or not)
const MeshDev &mesh_for(const lf_mesh *M, const lf_laplacian_params *p);
void halo_exchange(lf_mesh *M, const double *send, double *recv);
void field_halo(lf_mesh *M, const double *x);
void vector_halo(lf_mesh *M, const double *x, int64_t stride, int ncomp);  // -> ws.recvX
// p2p.cpp
void p2p_init(lf_context *ctx, int nranks, int rank);
void p2p_export(lf_mesh *M, void *handle);
void p2p_connect(lf_mesh *M, int nranks, int rank, const void *handles);
void allreduce(lf_mesh *M, const double *local, double *global, size_t count);
void upload_controls(lf_mesh *M, const lf_solver_controls *c, double *psi);
// precond.cpp
void ensure_dic(lf_mesh *M);  // build the DIC levels / rows (once), fill symU if assembled
void build_rows(lf_mesh *M);  // the same without the DIC transport check (mesh_create, K > 4)
void ensure_upper(lf_mesh *M);  // rebuild ld.upper from upperE if the last assembly skipped it
void require_dic(const lf_mesh *M);  // INVALID_ARG where the DIC kernels cannot run
void precondition(lf_mesh *M, int precond, const double *r, double *w, double *rD);
// gamg.cpp
void require_gamg(const lf_mesh *M);  // INVALID_ARG where the GAMG kernels cannot run
void ensure_gamg(lf_mesh *M);         // build the hierarchy (once) and the level-0 rows
void gamg_precondition(lf_mesh *M, const double *r, double *w, double *rD);
void gamg_export(lf_mesh *M, int32_t level, double *D, double *U, int32_t *fl, int32_t *fu);
void gamg_hierarchy(lf_mesh *M, int32_t *n_levels, int32_t *cells, int32_t *faces, int32_t *agg);
// mesh.cpp: resident grid with equal grid-stride trips per block
int balanced_grid(int64_t n, int g0);
}  // namespace lf
