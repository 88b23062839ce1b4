/*
 * lfoam.h — C ABI of the B200 laplacianFoam hot-path library (liblfoam.so).
 *
 * One implicit time step of dT/dt = div(DT grad T) on a finite-volume mesh in
 * OpenFOAM LDU face addressing (PAPER.md = P):
 *   TEqn( fvm::ddt(T) - fvm::laplacian(DT, T) == fvOptions(T) ); TEqn.solve();
 *   Listing 1, P:233-261 (§5.1); PCG + diagonal preconditioner.
 * The library assembles the matrix (fvm::ddt + fvm::laplacian face loop as an
 * atomic-free cell gather over the paper's CSR lists, §5.2), injects
 * boundary coefficients (P:457-497 pattern), runs lduMatrix::Amul and the
 * OpenFOAM PCG with fused reductions, on one or several B200 GPUs (processor
 * patches + NCCL, one process per GPU, §6.2).
 *
 * Conventions for every call:
 *   - Return value lf_status; LF_OK = 0.  No exceptions or aborts cross the
 *     ABI; lf_last_error() gives a thread-local detail string.
 *   - Labels are int32, values IEEE fp64 (reading A12).
 *   - "host" pointers are plain CPU memory; "device" pointers are CUDA device
 *     memory on the context's device (e.g. torch tensors' data_ptr()).
 *   - All device work is enqueued on the context's stream (the one passed to
 *     lf_context_create, or a private non-blocking stream if NULL).
 *   - Calls are not thread-safe on the same context.
 *   - After LF_ERR_CUDA / LF_ERR_NCCL a mesh is unusable: later calls on it
 *     return LF_ERR_STATE.
 */
#ifndef LFOAM_H
#define LFOAM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LF_VERSION 2

#if defined(__GNUC__)
#define LF_API __attribute__((visibility("default")))
#else
#define LF_API
#endif

typedef enum {
  LF_OK = 0,
  LF_ERR_INVALID_ARG = 1, /* bad label/size/value; argument named in lf_last_error() */
  LF_ERR_STATE = 2,       /* object unusable or call out of order */
  LF_ERR_OOM = 3,         /* device or host allocation failed */
  LF_ERR_CUDA = 4,        /* CUDA runtime error */
  LF_ERR_NCCL = 5,        /* NCCL missing or failed */
  LF_ERR_INTERNAL = 6
} lf_status;

LF_API const char *lf_status_string(lf_status s);
LF_API const char *lf_last_error(void);
LF_API int lf_version(void);

/* ------------------------------------------------------------- context */
typedef struct lf_context lf_context;

/* device: CUDA ordinal.  cuda_stream: a cudaStream_t (borrowed, must outlive
 * the context) or NULL for a private non-blocking stream. */
LF_API lf_status lf_context_create(int device, void *cuda_stream, lf_context **out);
LF_API lf_status lf_context_destroy(lf_context *ctx);

/* Multi-GPU ("1 MPI process for each GPU").
 * lf_comm_unique_id writes a 128-byte NCCL unique id (call on rank 0 and
 * broadcast it, e.g. through torch.distributed).  lf_comm_init joins the
 * communicator; all later reductions and processor-patch halos of meshes
 * created on this context are global over it.  NCCL is loaded at run time
 * (libnccl.so.2); if absent: LF_ERR_NCCL.  nranks == 1 is valid. */
LF_API lf_status lf_comm_unique_id(void *out_128_bytes);
LF_API lf_status lf_comm_init(lf_context *ctx, const void *unique_id_128, int nranks, int rank);
LF_API lf_status lf_comm_info(const lf_context *ctx, int *nranks, int *rank);

/* ---------------------------------------------------------------- mesh */
typedef enum {
  LF_PATCH_FIXED_VALUE = 0,   /* Dirichlet T_b (fvPatchField fixedValue)       */
  LF_PATCH_ZERO_GRADIENT = 1, /* homogeneous Neumann, contributes nothing      */
  LF_PATCH_PROCESSOR = 2      /* coupled to cells of rank neighb_rank          */
} lf_patch_type;

typedef struct {
  lf_patch_type type;
  int32_t n_faces;
  const int32_t *face_cells;   /* host [n_faces] local cell labels (faceCells)             */
  const double *mag_sf;        /* host [n_faces] |Sf| > 0                                  */
  const double *delta_coeffs;  /* host [n_faces] 1/|n.(Cf-C_P)| (wall), 1/|C_N-C_P| (proc)  */
  const double *value;         /* host [n_faces] fixedValue T_b, or NULL (= 0)             */
  int32_t neighb_rank;         /* processor only.  Faces must be in the same order on both
                                  sides (e.g. ascending global face id).  neighb_rank ==
                                  own rank: coupled to the NEXT processor patch that also
                                  names the own rank (self pairs, a loopback used by tests). */
  const double *sf;            /* host [n_faces][3] outward area vectors, or NULL; required by
                                  lf_fvc_grad / the corrected laplacian (with lf_mesh_desc.sf) */
  const double *cf;            /* processor patches of a full-geometry mesh: host [n_faces][3]
                                  face centres, and                                         */
  const double *cn;            /* host [n_faces][3] centres of the coupled cells across the
                                  interface (OpenFOAM's patchNeighbourField of C).  Both or
                                  neither; with them the interface gets interpolation weights
                                  w = |Sf.(C_N-Cf)| / (|Sf.(Cf-C_P)| + |Sf.(C_N-Cf)|) and
                                  correction vectors n - delta (C_N - C_P), and the corrected
                                  laplacian and DT fields run across processor patches
                                  (their halos: T, the gradient, DT).  NULL elsewhere.      */
} lf_patch_desc;

typedef struct {
  int32_t n_cells;             /* >= 1                                                      */
  int32_t n_faces;             /* internal faces, >= 0                                      */
  int32_t n_patches;
  const int32_t *owner;        /* host [n_faces] 0 <= owner,neighbour < n_cells,           */
  const int32_t *neighbour;    /* owner != neighbour; any face order, any orientation      */
  const double *mag_sf;        /* host [n_faces] |Sf|                                       */
  const double *delta_coeffs;  /* host [n_faces] 1/|C_N - C_P| (orthogonal meshes, A4)      */
  const double *V;             /* host [n_cells] > 0                                        */
  const lf_patch_desc *patches;/* host [n_patches]                                          */
  int32_t renumber;            /* 0 keep numbering; 1 reverse Cuthill-McKee inside the
                                  library; 2 multicolour: greedy first-fit colouring in cell
                                  order (colour = smallest not used by a lower-labelled
                                  neighbour), cells renumbered colour by colour, ascending
                                  label within a colour — the numbering under which the DIC
                                  sweeps run in #colours parallel levels (2 on hex blocks).
                                  Fields still speak the caller's numbering.              */
  /* Full geometry (all NULL, or all set together with every non-empty patch's
   * sf; c != NULL marks a geometry mesh, sf/cf may be NULL only if n_faces == 0): the
   * non-orthogonal correction path (fvc::grad and the
   * Gauss linear corrected laplacian).  Then delta_coeffs must be OpenFOAM's
   * nonOrthDeltaCoeffs 1/max(n.d, 0.05|d|). */
  const double *sf;            /* host [n_faces][3] area vectors, owner -> neighbour      */
  const double *cf;            /* host [n_faces][3] face centres                          */
  const double *c;             /* host [n_cells][3] cell centres                          */
} lf_mesh_desc;

typedef struct lf_mesh lf_mesh;

/* Copies every host array (caller keeps ownership), validates labels and
 * values (LF_ERR_INVALID_ARG), uploads to the device and builds the
 * atomic-free cell->face lists of P:387-429 (§5.2) on the GPU:
 *   internal faces re-sorted upper-triangular (owner, then neighbour),
 *   ownerStart[n+1]; losort = stable argsort of neighbour ("neighbourList"),
 *   losortStart[n+1]; per-cell boundary-face groups (facePatchIndex/Start,
 *   P:471-481).  Allocates every work array once (no per-step allocation,
 *   the lesson of P:728).  T starts at 0. */
LF_API lf_status mesh_create(lf_context *ctx, const lf_mesh_desc *desc, lf_mesh **out);
LF_API lf_status mesh_destroy(lf_mesh *mesh);

/* Peer-memory transport (SURVEY §8(e) option A), the
 * alternative to NCCL: halos and the PCG sums move through device memory the
 * ranks map from each other with CUDA IPC (NVLink 5 between GPUs; the same
 * memory when ranks share a GPU).  Kernels store halo values straight into
 * the neighbour's buffers and exchange the reduction sums in the last block
 * of each reduction, so the whole solve stays on the device (persistent
 * kernel).  Sequence:
 *   lf_p2p_init(ctx, nranks, rank)            before mesh_create
 *   mesh_create(...)                          processor patches as for NCCL
 *   lf_p2p_export(mesh, h)                    LF_P2P_HANDLE_BYTES per rank
 *   (all-gather the handles, e.g. torch.distributed)
 *   lf_p2p_connect(mesh, nranks, rank, all)   all[q*LF_P2P_HANDLE_BYTES] = rank q's
 * All ranks must make the same sequence of solver calls (collective). */
#define LF_P2P_HANDLE_BYTES 1024
LF_API lf_status lf_p2p_init(lf_context *ctx, int nranks, int rank);
LF_API lf_status lf_p2p_export(lf_mesh *mesh, void *handle_out);
LF_API lf_status lf_p2p_connect(lf_mesh *mesh, int nranks, int rank, const void *handles);

/* Sizes: n_cells, internal faces, total boundary faces, device bytes held. */
LF_API lf_status lf_mesh_info(const lf_mesh *mesh, int32_t *n_cells, int32_t *n_faces,
                       int32_t *n_boundary_faces, int64_t *device_bytes);

/* Gather layout chosen by mesh_create (for tests and reports; any pointer may
 * be NULL): ell_width = slots per side of the ELL slices (3 or 4; 0 = CSR or
 * full rows), row_width = slots of the full-row ELL (6 or 8; 0 = none),
 * label_escapes = compressed-label entries that escape to int32 labels
 * (-1 = compressed labels not built, LF_OPT_COMPRESSED_LABELS). */
LF_API lf_status lf_mesh_layout(const lf_mesh *mesh, int32_t *ell_width, int32_t *row_width,
                                int32_t *label_escapes);

/* Host copies of the addressing built by mesh_create, for tests (internal
 * numbering and face order).  Any pointer may be NULL.
 *   owner_start[n+1], losort[F], losort_start[n+1], face_order[F] (internal
 *   face i = caller's face face_order[i]), cell_order[n] (internal cell i =
 *   caller's cell cell_order[i]). */
LF_API lf_status lf_mesh_export_addressing(const lf_mesh *mesh, int32_t *owner_start,
                                    int32_t *losort, int32_t *losort_start,
                                    int32_t *face_order, int32_t *cell_order);

/* Device arrays between the caller's and the internal cell numbering
 * (identity copy when renumber == 0).  to_internal: 1 caller->internal. */
LF_API lf_status lf_permute(const lf_mesh *mesh, int to_internal, const double *in_dev, double *out_dev);

/* --------------------------------------------------------------- fields */
typedef enum {
  LF_FIELD_T = 0,            /* cell values, n = n_cells, patch = -1            */
  LF_FIELD_DT = 2,           /* spatially varying diffusivity DT (cell values > 0, n =
                                n_cells, patch = -1).  Setting it
                                computes the face diffusivities once, on the device:
                                gamma_f = w (DT_P - DT_N) + DT_N with the geometric
                                weights, boundary DT[faceCell] (reading A38),
                                processor faces w (DT_P - DT_N) + DT_N with the coupled
                                cell's DT (a halo exchange; collective across ranks).
                                Needs the full geometry (and the processor patches'
                                cf / cn); used by solves with
                                lf_laplacian_params.variable_DT. */
  LF_FIELD_PATCH_VALUE = 1   /* boundary values of patch `patch`, n = n_faces.
                                fixedValue: T_b (set/get).  zeroGradient: get
                                returns T[faceCells] (correctBoundaryConditions);
                                set is ignored.  processor: get returns 0.      */
} lf_field;

/* on_device: 1 if v is a device pointer, 0 host.  Stream-ordered; a host
 * field_get returns after the copy is complete. */
LF_API lf_status field_set(lf_mesh *mesh, lf_field f, int32_t patch, const double *v, int64_t n, int on_device);
LF_API lf_status field_get(const lf_mesh *mesh, lf_field f, int32_t patch, double *v, int64_t n, int on_device);

/* ---------------------------------------------------------- assembly */
typedef struct {
  double DT;   /* uniform diffusivity > 0 (reading A11)   */
  double dt;   /* time step > 0 (P:608 uses 0.2 s)        */
  int32_t corrected;   /* 0: orthogonal two-point laplacian (A4).  1: Gauss linear
                          corrected — adds the explicit non-orthogonal correction
                          +V div(DT|Sf| corrVec . interpolate(grad T)) to the source
                          (needs full geometry; processor patches need their cf/cn
                          and exchange the T and gradient halos — collective)    */
  int32_t n_non_orth_correctors;  /* laplacianFoam_step: extra corrector passes per
                          step (simple.correctNonOrthogonal()); each pass
                          re-evaluates the correction from the current T and solves
                          again from it, ddt keeping T0 of the step (0 = one pass) */
  int32_t variable_DT; /* 1: the laplacian's diffusivity is the LF_FIELD_DT cell field
                          (gammaMagSf = gamma_f |Sf| in place of DT |Sf|; DT ignored);
                          LF_ERR_STATE if that field was never set */
} lf_laplacian_params;

typedef struct lf_ldu lf_ldu;   /* owned by its mesh, reused every step */

/* fvm::ddt(T) - fvm::laplacian(DT,T) with T0 = current T (Listing 1
 * line 12; readings A3-A5): per internal face u = delta*(DT*magSf),
 * upper = -u; diag = V/dt + sum u (+ boundary internalCoeffs);
 * source = (T0/dt)*V (+ fixedValue boundaryCoeffs), with p->corrected the
 * explicit non-orthogonal correction of T as well.  One kernel, a per-cell
 * gather (no float atomics); deterministic.  Errors: DT/dt <= 0, corrected
 * without geometry or with processor patches lacking cf/cn -> INVALID_ARG. */
LF_API lf_status laplacian_assemble(lf_mesh *mesh, const lf_laplacian_params *p, lf_ldu **sys);

/* fvc::grad(x) with gaussGrad + linear interpolation — the kernels the paper
 * ported (§5.2: weights P:321-334, interpolation/dotInterpolate P:293-315,
 * gradf owner/neighbour and boundary gathers P:435-497, field division
 * P:503-528) — as atomic-free per-cell gathers, plus correctBoundaryConditions
 * (P:539-556).  x_dev: device [n_cells] (internal numbering); boundary values
 * from the mesh's patches (fixedValue T_b, zeroGradient x[faceCell]).
 * grad_dev: device [n_cells][3]; bgrad_dev: device [boundary faces][3] (patch
 * order) or NULL; processor faces interpolate with the coupled cell's x
 * (halo exchange, collective) and are not corrected (coupled patches).
 * Needs full geometry (processor patches: their cf/cn). */
LF_API lf_status lf_fvc_grad(lf_mesh *mesh, const double *x_dev, double *grad_dev, double *bgrad_dev);

/* Host copies in the CALLER's numbering and face order; any pointer may be
 * NULL.  internal/boundary_coeffs: [total boundary faces] in patch order
 * (internalCoeffs = a; boundaryCoeffs = a*T_b fixedValue, a processor). */
LF_API lf_status lf_ldu_export(const lf_ldu *sys, double *diag, double *upper, double *source,
                        double *internal_coeffs, double *boundary_coeffs);

/* y = A x (lduMatrix::Amul incl. processor interfaces).  x_dev, y_dev:
 * device [n_cells] in INTERNAL numbering (== caller's when renumber == 0),
 * must not alias.  Asynchronous, stream-ordered. */
LF_API lf_status ldu_amul(const lf_ldu *sys, const double *x_dev, double *y_dev);

/* ---------------------------------------------------------------- PCG */
/* Preconditioners (OpenFOAM fvSolution names).
 *   LF_PRECOND_DIAGONAL  rD = 1/diag, w = rD r — the paper's choice.
 *   LF_PRECOND_DIC       OpenFOAM DICPreconditioner:
 *                        rD = diag; for faces in upper-triangular order
 *                        rD[u] -= upper^2/rD[l]; rD = 1/rD;  w = rD r;
 *                        forward  for f ascending:  w[u] -= rD[u] upper_f w[l];
 *                        backward for f descending: w[l] -= rD[l] upper_f w[u].
 *                        Exact OpenFOAM semantics on any numbering: the sweeps
 *                        run level by level (a cell's level = 1 + the largest
 *                        level of its lower neighbours), so the parallel depth
 *                        is the number of levels — 2 on a hex block numbered
 *                        with renumber = 2, 3N-2 on the natural N^3 numbering.
 *                        Processor-local like OpenFOAM's (interfaces do not enter
 *                        the factor or the sweeps: block-Jacobi IC(0) across
 *                        ranks); processor patches need the peer-memory
 *                        transport (lf_p2p_*), not NCCL (else INVALID_ARG); runs
 *                        in the persistent solver whatever LF_OPT_PERSISTENT
 *                        says; cells may have at most 8 neighbours.
 *   LF_PRECOND_DILU      OpenFOAM DILUPreconditioner; on this symmetric matrix
 *                        (lower == upper) its recurrences are DIC's term for
 *                        term, so it runs the DIC kernels.
 *   LF_PRECOND_GAMG      algebraic multigrid (P:773 names
 *                        AMG "a better alternative"; reading A43):
 *                        pairwise face agglomeration of the mesh graph (built
 *                        once per mesh on first use, weights |Sf| delta),
 *                        Galerkin coarse matrices P^T A P formed per solve,
 *                        one symmetric V-cycle per application (weighted
 *                        Jacobi omega = 0.9 before and after the coarse
 *                        correction, exact dense solve of the coarsest level
 *                        of <= 64 cells).  Single rank: a mesh with processor
 *                        patches is INVALID_ARG; coarsening that stalls above
 *                        2048 cells is INVALID_ARG; cells may have at most 8
 *                        neighbours (the level-0 rows). */
typedef enum { LF_PRECOND_DIAGONAL = 0, LF_PRECOND_DIC = 1, LF_PRECOND_DILU = 2,
               LF_PRECOND_GAMG = 3 } lf_preconditioner;

typedef struct {
  double tolerance;   /* absolute on the normalised L1 residual (1e-10)   */
  double rel_tol;     /* 0 = off                                          */
  int32_t max_iter;   /* 1000 (OpenFOAM default)                          */
  int32_t min_iter;   /* 0                                                */
  int32_t preconditioner;  /* lf_preconditioner; 0 (zero-initialised) = diagonal */
  int32_t reserved;   /* 0                                                */
} lf_solver_controls;

typedef struct {
  double initial_residual, final_residual;
  int32_t n_iterations, converged, singular, reserved;
} lf_solver_perf;

/* w = M^-1 r for the preconditioner of the assembled system (the call PCG
 * makes once per iteration): r_dev, w_dev device [n_cells] in internal
 * numbering, must not alias; rD_dev: device [n_cells] receives the
 * reciprocal (DIC) diagonal, or NULL.  Stream-ordered.  Errors as pcg_solve. */
LF_API lf_status ldu_precondition(const lf_ldu *sys, int32_t preconditioner, const double *r_dev,
                                  double *w_dev, double *rD_dev);

/* GAMG hierarchy of a mesh (LF_PRECOND_GAMG; builds it if needed), for
 * tests and inspection: *n_levels = L + 1; cells[l], faces[l] for l <= L
 * (arrays of >= 31 entries); agg: the level l -> l+1 maps concatenated
 * (sum of cells[l] for l < L entries), internal numbering.  Any pointer may
 * be NULL.  INVALID_ARG where GAMG cannot run (see LF_PRECOND_GAMG). */
LF_API lf_status lf_gamg_hierarchy(lf_mesh *mesh, int32_t *n_levels, int32_t *cells, int32_t *faces,
                                   int32_t *agg);

/* Host copies of the Galerkin matrix of GAMG level 1 <= level <= L as the
 * last GAMG solve or ldu_precondition formed it: D[cells], U[faces] with the
 * faces' lower / upper cells (face_l < face_u, faces sorted).  Any pointer
 * may be NULL.  STATE before the first GAMG use. */
LF_API lf_status lf_gamg_export(const lf_ldu *sys, int32_t level, double *D, double *U, int32_t *face_l,
                                int32_t *face_u);

/* OpenFOAM PCG, preconditioner from c:
 * psi_dev (device [n_cells], internal numbering) is the initial guess and
 * receives the solution.  Two fused kernels per iteration (diagonal) or one
 * persistent launch per solve; alpha, beta and the stopping rule are
 * evaluated on the device.  With DIC the preconditioner is rebuilt from the
 * current coefficients at every solve (as OpenFOAM constructs it per solve).
 * Returns once *out is on the host.  Non-convergence and singularity are
 * LF_OK with flags set; an unknown preconditioner, or DIC with NCCL
 * processor patches / more than 8 neighbours per cell, is INVALID_ARG. */
LF_API lf_status pcg_solve(lf_ldu *sys, double *psi_dev, const lf_solver_controls *c, lf_solver_perf *out);

/* n_steps laplacianFoam time steps on the mesh's T field: each step
 * assembles (fused with the PCG setup) and solves in place (Listing 1), with
 * 1 + n_non_orth_correctors passes when p->corrected.
 * per_step: host [n_steps * (1 + (corrected ? n_non_orth_correctors : 0))]
 * (one entry per solve) or NULL. */
LF_API lf_status laplacianFoam_step(lf_mesh *mesh, const lf_laplacian_params *p,
                             const lf_solver_controls *c, int32_t n_steps,
                             lf_solver_perf *per_step);

/* ------------------------------------------------------- instrumentation */
/* Kernel kinds for lf_kernel_stats. */
typedef enum {
  LF_K_ASSEMBLE = 0, LF_K_SETUP = 1, LF_K_PHASE1 = 2, LF_K_PHASE2 = 3,
  LF_K_AMUL = 4, LF_K_SUMPSI = 5, LF_K_PACK = 6,
  LF_K_PCG = 7,      /* persistent whole-solve kernel (single rank, no processor patches) */
  LF_K_NONORTH = 8,  /* gradient / non-orthogonal correction kernels (lf_fvc_grad, corrected) */
  LF_K_PCG_DIC = 9,  /* persistent whole-solve kernel with the DIC preconditioner */
  LF_K_PRECOND = 10, /* standalone preconditioner kernels (ldu_precondition, DIC set-up) */
  LF_K_PCG_GAMG = 11,/* persistent whole-solve kernel with the GAMG preconditioner */
  LF_K_COUNT = 12
} lf_kernel_kind;

/* Execution options of a context:
 *   LF_OPT_PERSISTENT  (default 1) single-rank meshes without processor
 *                      patches run the whole PCG loop as ONE cooperative
 *                      launch (grid barriers between the phases); 0 = one
 *                      launch per phase
 *   LF_OPT_GRAPHS      (default 1) phase launches are replayed from CUDA
 *                      graphs of 2^i iterations; 0 = direct launches
 *   LF_OPT_SOLVE_VARIANT (default 0 = by mesh size) persistent solve variant
 *                      (single rank or peer-memory transport; diagonal and
 *                      DIC): 1 the L2-resident one (psi update in
 *                      the beta-barrier wait, {q, diag} kept in shared memory
 *                      between the phases; needs <= 8 grid-stride trips per
 *                      thread, else variant 2 runs), 2 the HBM-bound one (psi
 *                      update deferred into the Amul phase); mesh_create picks
 *                      1 when an iteration's working set fits ~1.5x the L2
 *   LF_OPT_COMPRESSED_LABELS (default 0; read by mesh_create) ELL meshes also
 *                      store their gather labels as 16-bit codes relative to a
 *                      per-32-cell offset (4 B instead of 8 B per face slot,
 *                      escapes to the int32 labels where a code does not fit);
 *                      the persistent diagonal solve gathers through them.
 *                      0 = int32 labels only.  Decoded labels are identical,
 *                      so results are bitwise the same either way.  Measured
 *                      slower (200^3: 53.8 vs 40.5 ms/step: the decode adds
 *                      dependent integer work to every gather), hence off.
 *   LF_OPT_OVERLAP_HALO (default 1) NCCL transport: the processor-patch halo
 *                      of w runs on a second communicator (ncclCommSplit) and
 *                      stream while the Amul phase of the cells WITHOUT
 *                      processor faces runs; the cells with them follow once
 *                      the halo has arrived (north_star: halos "overlapped with
 *                      the interior Amul").  0 = the serial sequence.
 *   LF_OPT_L2_PREFETCH (default 0 = chosen per mesh by mesh_create; 1 on, 2
 *                      off; read at each solve) HBM-bound persistent diagonal
 *                      solve: every warp prefetches into L2 the lines of its
 *                      own-cell streams (labels, owner-side coefficients, w,
 *                      diag, p_old, psi) one grid-stride trip ahead
 *                      (prefetch.global.L2, lane-distributed), so a trip's
 *                      first loads hit L2 instead of HBM.  On when the
 *                      neighbour-reuse window plus two trips fits ~0.57 of the
 *                      L2 (200^3: +6%; 400^3 would evict its reuse window: off).
 *                      Pure prefetch: results are bitwise the same.
 *   LF_OPT_DYNAMIC_TRIPS (default -1 = 30 in builds with -DLF_DYN=1, where the
 *                      run-time trips are compiled in; the default build
 *                      compiles them out and keeps the static schedule, the
 *                      option is then accepted and has no effect; 0..100
 *                      forces the percentage; read at each solve) HBM-bound
 *                      persistent diagonal solve, one
 *                      rank: the last N% of phase 1's grid-stride trips are
 *                      handed out at run time (a global counter, units of 2
 *                      trips x one 512-cell block run in sweep order), so SMs
 *                      that run slower take fewer.  Each unit's sums are
 *                      reduced per warp, then over the unit's warps in warp
 *                      order, and stored per unit; the barrier adds them in
 *                      unit order — the totals do not depend on which block
 *                      ran which unit (deterministic; the grouping differs
 *                      from N = 0 at rounding level).
 * Results are identical up to reduction grid size (all are deterministic). */
typedef enum { LF_OPT_PERSISTENT = 0, LF_OPT_GRAPHS = 1, LF_OPT_SOLVE_VARIANT = 2,
               LF_OPT_COMPRESSED_LABELS = 3, LF_OPT_OVERLAP_HALO = 4,
               LF_OPT_L2_PREFETCH = 5, LF_OPT_DYNAMIC_TRIPS = 6 } lf_option;
LF_API lf_status lf_set_option(lf_context *ctx, lf_option opt, int value);

/* enable != 0: bracket every launch of the hot kernels with CUDA events on
 * the context stream and accumulate their durations (timings are read back
 * at the per-solve sync).  Counters reset on enable. */
LF_API lf_status lf_set_instrumentation(lf_context *ctx, int enable);
/* launches and summed device milliseconds of one kernel kind since enable;
 * also the number of kernels the library launched in total. */
LF_API lf_status lf_kernel_stats(const lf_context *ctx, lf_kernel_kind k, int64_t *launches,
                          double *total_ms);
LF_API lf_status lf_launch_count(const lf_context *ctx, int64_t *kernels_launched);

#ifdef __cplusplus
}
#endif
#endif /* LFOAM_H */
