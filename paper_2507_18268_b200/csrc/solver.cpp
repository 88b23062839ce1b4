// L3 solver driver: step loop, PCG loop control, halo exchange, reductions.
//
// The PCG loop is device-driven (SURVEY.md §7 "loop control without host
// round trips"): alpha, beta and the OpenFOAM stopping rule are evaluated by
// the kernels from device-resident sums (PcgCtl); iterations past the stop
// are no-op launches.  The host enqueues iterations in chunks — the first
// chunk sized from the previous solve's iteration count — and reads the
// stop flag once per chunk, so a steady step costs one host sync.
#include <algorithm>

#include "host.h"

namespace lf {

void allreduce(lf_mesh *M, const double *local, double *global, size_t count) {
  lf_context *ctx = M->ctx;
  if (!ctx->comm) return;  // single rank: kernels wrote the global slot directly
  nccl_allreduce_sum(ctx->comm, local, global, count, ctx->stream);
}

// recv[seg] <- neighbour's send[seg'] for every processor patch (on the
// context's communicator and stream, or the given ones).
static void halo_exchange_on(lf_mesh *M, const double *send, double *recv, void *comm, cudaStream_t s);
void halo_exchange(lf_mesh *M, const double *send, double *recv) {
  halo_exchange_on(M, send, recv, M->ctx->comm, M->ctx->stream);
}

static void halo_exchange_on(lf_mesh *M, const double *send, double *recv, void *comm, cudaStream_t s) {
  if (M->nproc == 0) return;
  lf_context *ctx = M->ctx;
  if (!comm) {
    for (const HaloSeg &g : M->segs) {
      if (g.partner < 0) throw Error{LF_ERR_STATE, "processor patch to another rank needs lf_comm_init"};
      const HaloSeg &p = M->segs[g.partner];
      LF_CUDA(cudaMemcpyAsync(recv + g.offset, send + p.offset, sizeof(double) * g.count,
                              cudaMemcpyDeviceToDevice, s));
    }
    return;
  }
  // NCCL: per peer, the i-th send matches the i-th recv.  Real peers have one
  // patch each side in the same face order.  Self pairs (a,b): sends a,b;
  // recvs b,a so that recv[b] <- send[a] and recv[a] <- send[b].
  nccl_group_start();
  for (const HaloSeg &g : M->segs) nccl_send(comm, send + g.offset, g.count, g.peer, s);
  for (const HaloSeg &g : M->segs) {
    const HaloSeg &dst = g.partner >= 0 ? M->segs[g.partner] : g;
    nccl_recv(comm, recv + dst.offset, dst.count, g.peer, s);
  }
  nccl_group_end();
}

// ------------------------------------- NCCL halo overlapped with the Amul
// The w halo runs on the split communicator and the comm stream; phase 1 of
// the cells without processor faces runs meanwhile, the rest after evHalo.
static bool overlap_halo(const lf_mesh *M) {
  return M->ctx->comm && M->ctx->commHalo && M->ctx->overlapHalo && M->nproc > 0 && M->cellsInt;
}

// the compute stream waits for the halo started last (if any)
static void wait_w_halo(lf_mesh *M) {
  if (!M->haloPending) return;
  LF_CUDA(cudaStreamWaitEvent(M->ctx->stream, M->ctx->evHalo, 0));
  M->haloPending = false;
}

// pack w at the send cells (compute stream), exchange on the comm stream
static void start_w_halo(lf_mesh *M) {
  lf_context *ctx = M->ctx;
  const Workspace &ws = M->ws;
  wait_w_halo(M);  // the previous exchange still reads sendBuf
  ctx->launch(LF_K_PACK, [&] { launch_pack_x(ctx->stream, M->nproc, ws.sendCell, ws.w, ws.sendBuf); });
  LF_CUDA(cudaEventRecord(ctx->evPacked, ctx->stream));
  LF_CUDA(cudaStreamWaitEvent(ctx->commStream, ctx->evPacked, 0));
  halo_exchange_on(M, ws.sendBuf, ws.recvW, ctx->commHalo, ctx->commStream);
  LF_CUDA(cudaEventRecord(ctx->evHalo, ctx->commStream));
  M->haloPending = true;
}

void upload_controls(lf_mesh *M, const lf_solver_controls *c, double *psi) {
  LF_REQUIRE(c != nullptr, "controls is NULL");
  LF_REQUIRE(c->tolerance >= 0.0 && c->rel_tol >= 0.0, "tolerances must be >= 0");
  LF_REQUIRE(c->max_iter >= 0 && c->min_iter >= 0, "max_iter/min_iter must be >= 0");
  LF_REQUIRE(c->preconditioner >= LF_PRECOND_DIAGONAL && c->preconditioner <= LF_PRECOND_GAMG,
             "unknown preconditioner");
  if (c->preconditioner == LF_PRECOND_GAMG)
    require_gamg(M);
  else if (c->preconditioner != LF_PRECOND_DIAGONAL)
    require_dic(M);
  PcgCtl *h = M->hctl;
  std::memset(h, 0, sizeof(PcgCtl));
  h->tol = c->tolerance;
  h->relTol = c->rel_tol;
  h->maxIter = c->max_iter;
  h->minIter = c->min_iter;
  h->nTotal = M->nTotal;
  h->psi = psi;
  h->precond = c->preconditioner;
  h->stop = 1;  // nothing runs until a setup kernel resets it
  // passed by value to a one-thread kernel: stream-ordered, no host sync
  // (a host->device copy from the pinned mirror would have to be waited for
  // before the mirror is reused — a host round trip inside every step)
  M->ctx->launch(LF_K_SETUP, [&] { launch_set_ctl(M->ctx->stream, M->ws.ctl, *h); });
}

// Host-side halo of a cell field (NCCL / local copies): x at the send cells
// -> sendBuf -> neighbour's recv.  With the peer-memory transport the
// kernels store straight into the neighbour's buffers instead.
static bool host_halo(lf_mesh *M) { return M->nproc > 0 && !M->p2pConnected; }

static void exchange_field(lf_mesh *M, const double *x, double *recv) {
  lf_context *ctx = M->ctx;
  const Workspace &ws = M->ws;
  ctx->launch(LF_K_PACK, [&] { launch_pack_x(ctx->stream, M->nproc, ws.sendCell, x, ws.sendBuf); });
  halo_exchange(M, ws.sendBuf, recv);
}

// Halo of a cell field into recvT for the standalone calls (assembly, Amul):
// peer memory -> the sum kernel's put + allreduce (its sum is discarded);
// otherwise pack + exchange.
void field_halo(lf_mesh *M, const double *x) {
  if (M->nproc == 0) return;
  lf_context *ctx = M->ctx;
  if (M->p2pConnected) {
    M->ws.p2p.tPar = M->tPar ^= 1;  // the other recvT half: a slower rank may still read this one
    ctx->launch(LF_K_SUMPSI, [&] { launch_sum(ctx->stream, M->Lsum, M->md, x, M->ws, M->scratch); });
  }
  else
    exchange_field(M, x, M->ws.recvT);
}

// One PCG iteration: phase 1 (uses the halo of w from the previous phase 2
// and recomputes halo p locally), phase 2, then the halo of the new w.
static void iteration(lf_mesh *M) {
  lf_context *ctx = M->ctx;
  cudaStream_t s = ctx->stream;
  const Workspace &ws = M->ws;
  if (overlap_halo(M)) {
    // interior Amul while the w halo is in flight, then the cells with
    // processor faces; the p2 allreduce overlaps the next halo
    ctx->launch(LF_K_PHASE1, [&] { launch_phase1_part(s, M->Lp1, M->md, M->ld, ws, 1, M->cellsInt, M->nInt); });
    wait_w_halo(M);
    ctx->launch(LF_K_PHASE1, [&] { launch_phase1_part(s, M->Lp1, M->md, M->ld, ws, 2, M->cellsBnd, M->nBnd); });
    allreduce(M, ws.lsum->p1, ws.gsum->p1, 2);
    ctx->launch(LF_K_PHASE2, [&] { launch_phase2(s, M->Lp2, M->md, M->ld, ws); });
    start_w_halo(M);
    allreduce(M, ws.lsum->p2, ws.gsum->p2, 2);
    return;
  }
  ctx->launch(LF_K_PHASE1, [&] { launch_phase1(s, M->Lp1, M->md, M->ld, ws); });
  allreduce(M, ws.lsum->p1, ws.gsum->p1, 2);
  ctx->launch(LF_K_PHASE2, [&] { launch_phase2(s, M->Lp2, M->md, M->ld, ws); });
  if (host_halo(M)) exchange_field(M, ws.w, ws.recvW);
  allreduce(M, ws.lsum->p2, ws.gsum->p2, 2);
}

// Enqueue `count` PCG iterations: as CUDA-graph replays of 2^i-iteration
// chunks (binary decomposition of count), or as direct launches when the
// context is instrumented (events bracket every kernel).
static void enqueue_iterations(lf_mesh *M, int count) {
  lf_context *ctx = M->ctx;
  cudaStream_t s = ctx->stream;
  if (ctx->instrument || !ctx->useGraphs) {
    for (int i = 0; i < count; ++i) iteration(M);
    return;
  }
  // graphs are self-contained: a halo started before them is waited for
  // outside the capture, and every chunk joins its last halo
  wait_w_halo(M);
  if (M->kernelsPerIteration == 0) M->kernelsPerIteration = overlap_halo(M) ? 4 : host_halo(M) ? 3 : 2;
  for (int b = lf_mesh::kMaxGraphLog - 1; b >= 0 && count > 0;) {
    const int k = 1 << b;
    if (count < k) {
      --b;
      continue;
    }
    if (!M->chunkGraph[b]) {
      cudaGraph_t g = nullptr;
      ctx->capturing = true;
      LF_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      try {
        for (int i = 0; i < k; ++i) iteration(M);
        wait_w_halo(M);  // join the comm stream back into the capture
      } catch (...) {
        cudaStreamEndCapture(s, &g);
        if (g) cudaGraphDestroy(g);
        ctx->capturing = false;
        throw;
      }
      LF_CUDA(cudaStreamEndCapture(s, &g));
      ctx->capturing = false;
      cudaError_t e = cudaGraphInstantiate(&M->chunkGraph[b], g, 0);
      cudaGraphDestroy(g);
      LF_CUDA(e);
    }
    LF_CUDA(cudaGraphLaunch(M->chunkGraph[b], s));
    ctx->launches += (int64_t)k * M->kernelsPerIteration;
    ctx->kLaunches[LF_K_PHASE1] += overlap_halo(M) ? 2 * k : k;
    ctx->kLaunches[LF_K_PHASE2] += k;
    if (host_halo(M)) ctx->kLaunches[LF_K_PACK] += k;
    count -= k;
  }
}

// Runs the iterations after a setup launch (assembly+setup or pcg setup)
// until the device sets ctl->stop; fills *out.
static void run_iterations(lf_mesh *M, lf_solver_perf *out) {
  lf_context *ctx = M->ctx;
  cudaStream_t s = ctx->stream;
  const int maxIter = M->hctl->maxIter, minIter = M->hctl->minIter;
  const int64_t bound = (int64_t)std::max(maxIter, minIter) + 2;
  int64_t launched = 0;
  int chunk = M->lastIters >= 0 ? M->lastIters + 1 : 8;
  // persistent variant: L2-resident (idle psi flush) or HBM-bound (TMA)
  // (the L2-resident variant needs few enough trips per thread for its stash)
  M->ws.idleFlush = M->stashOK && (ctx->solveVariant == 0 ? M->l2Resident : ctx->solveVariant == 1) ? 1 : 0;
  M->ws.l2pf = (ctx->l2Prefetch == 0 ? M->pfFits : ctx->l2Prefetch == 1) ? 1 : 0;
  {
    // HBM-bound solve, one rank: the last trips of phase 1 are handed out at
    // run time (kernels.cu "run-time trips")
    const int64_t nFull = M->n / ((int64_t)M->persistentGrid * kernel_block_size());
    const int pct = ctx->dynPct >= 0 ? ctx->dynPct : dynamic_trips_pct();
    M->ws.dynTrips = M->ws.idleFlush ? 0 : (int)(nFull * pct / 100);
  }
  if (M->hctl->precond == LF_PRECOND_GAMG) {
    // GAMG: one persistent launch (Galerkin set-up, V-cycles; single rank)
    ctx->launch(LF_K_PCG_GAMG, [&] {
      launch_pcg_gamg(s, M->gamgGrid, M->md, M->ld, M->dGamg, M->ws, M->gridBar);
    });
    LF_CUDA(cudaMemcpyAsync(M->hctl, M->ws.ctl, sizeof(PcgCtl), cudaMemcpyDeviceToHost, s));
    LF_CUDA(cudaStreamSynchronize(s));
    ctx->harvest();
    M->gamgFormed = true;
    if (M->hctl->fault) throw Error{LF_ERR_INVALID_ARG, "GAMG: the coarsest matrix is not positive definite"};
    chunk = 0;
  } else if (M->hctl->precond != LF_PRECOND_DIAGONAL) {
    // DIC (DILU = DIC on this symmetric matrix): one persistent launch with
    // the level-scheduled sweeps (single rank, checked in upload_controls)
    ctx->launch(LF_K_PCG_DIC, [&] { launch_pcg_dic(s, M->dicGrid, M->md, M->ld, M->dic, M->ws, M->gridBar); });
    LF_CUDA(cudaMemcpyAsync(M->hctl, M->ws.ctl, sizeof(PcgCtl), cudaMemcpyDeviceToHost, s));
    LF_CUDA(cudaStreamSynchronize(s));
    ctx->harvest();
    chunk = 0;
  } else if (ctx->persistent && !ctx->comm && !host_halo(M)) {
    // no host-side halo (single rank, or peer-memory transport): the whole
    // loop in one cooperative launch
    ctx->launch(LF_K_PCG, [&] { launch_pcg_persistent(s, M->persistentGrid, M->md, M->ld, M->ws, M->gridBar); });
    LF_CUDA(cudaMemcpyAsync(M->hctl, M->ws.ctl, sizeof(PcgCtl), cudaMemcpyDeviceToHost, s));
    LF_CUDA(cudaStreamSynchronize(s));
    ctx->harvest();
    chunk = 0;  // skip the chunked loop
  }
  for (; chunk > 0;) {
    chunk = (int)std::max<int64_t>(1, std::min<int64_t>(chunk, bound + 1 - launched));
    enqueue_iterations(M, chunk);
    launched += chunk;
    LF_CUDA(cudaMemcpyAsync(M->hctl, M->ws.ctl, sizeof(PcgCtl), cudaMemcpyDeviceToHost, s));
    LF_CUDA(cudaStreamSynchronize(s));
    ctx->harvest();
    if (ctx->comm) nccl_check_async(ctx->comm);
    if (M->hctl->stop) break;
    if (launched > bound) throw Error{LF_ERR_INTERNAL, "PCG loop did not stop within max_iter"};
    chunk = 8;
  }
  wait_w_halo(M);  // no halo left in flight past the solve
  const PcgCtl *h = M->hctl;
  M->lastIters = h->it;
  if (out) {
    out->initial_residual = h->initRes;
    out->final_residual = h->finRes;
    out->n_iterations = h->it;
    out->converged = h->converged;
    out->singular = h->singular;
    out->reserved = 0;
  }
}

static void sum_psi(lf_mesh *M, const double *psi) {
  lf_context *ctx = M->ctx;
  if (M->p2pConnected) M->ws.p2p.tPar = M->tPar ^= 1;  // this launch also pushes the T halo
  ctx->launch(LF_K_SUMPSI, [&] { launch_sum(ctx->stream, M->Lsum, M->md, psi, M->ws, &M->ws.lsum->p1[1]); });
  allreduce(M, M->ws.lsum->p1, M->ws.gsum->p1, 2);
}

void require_corrected(const lf_mesh *M) {
  LF_REQUIRE(M->hasGeom, "the non-orthogonal path needs the full geometry (lf_mesh_desc.sf/cf/c)");
  LF_REQUIRE(M->nproc == 0 || M->procGeom,
             "the non-orthogonal path across processor patches needs the patches' cf and cn");
}

// Vector halo: x[k*stride + cell] at every send slot -> ws.recvX[k*nproc +
// slot] of the coupled rank (peer memory: pushed by a kernel; NCCL /
// loopback: packed and exchanged component by component).
void vector_halo(lf_mesh *M, const double *x, int64_t stride, int ncomp) {
  if (M->nproc == 0) return;
  lf_context *ctx = M->ctx;
  const Workspace &ws = M->ws;
  if (M->p2pConnected) {
    ctx->launch(LF_K_SUMPSI,
                [&] { launch_push_x(ctx->stream, M->Lsum, M->md, x, stride, ncomp, ws, M->scratch); });
    return;
  }
  for (int k = 0; k < ncomp; ++k) {
    ctx->launch(LF_K_PACK, [&] { launch_pack_x(ctx->stream, M->nproc, ws.sendCell, x + k * stride, ws.sendBuf); });
    halo_exchange(M, ws.sendBuf, ws.recvX + (size_t)k * M->nproc);
  }
}

// gradS <- fvc::grad(x); lapSrc <- explicit non-orthogonal laplacian source
// of that gradient (two gathers, stream-ordered).  Across processor patches:
// the halo of x before the gradient, the halo of the gradient before the
// correction (the coupled faces interpolate with the neighbour rank's values).
void correction_source(lf_mesh *M, const MeshDev &md, double DT, const double *x) {
  lf_context *ctx = M->ctx;
  field_halo(M, x);
  ctx->launch(LF_K_NONORTH,
              [&] { launch_grad(ctx->stream, M->Lasm, md, M->geo, x, M->haloT(), M->gradS, nullptr); });
  vector_halo(M, M->gradS, M->n, 3);
  ctx->launch(LF_K_NONORTH, [&] {
    launch_lap_corr(ctx->stream, M->Lasm, md, M->geo, DT, M->gradS, M->ws.recvX, M->nproc, M->lapSrc);
  });
}

const MeshDev &mesh_for(const lf_mesh *M, const lf_laplacian_params *p) {
  if (p && p->variable_DT) {
    if (!M->dtSet) throw Error{LF_ERR_STATE, "variable_DT: set the DT field first (field_set LF_FIELD_DT)"};
    return M->mdVar;
  }
  return M->md;
}

void solve_loop(lf_mesh *M, const lf_solver_controls *c, double *psi, bool fromAssembly,
                const lf_laplacian_params *p, lf_solver_perf *out, const double *T0, const double *lapSrc) {
  lf_context *ctx = M->ctx;
  cudaStream_t s = ctx->stream;
  const Workspace &ws = M->ws;
  const bool psiIsT = (psi == M->T);
  if (M->hctl->precond == LF_PRECOND_GAMG)
    ensure_gamg(M);  // hierarchy + level-0 rows, before the assembly writes the rows
  else if (M->hctl->precond != LF_PRECOND_DIAGONAL)
    ensure_dic(M);  // before the assembly writes the rows
  // sum(psi) for normFactor; with the peer-memory transport the same launch
  // puts psi at the processor-face cells into the neighbours' recvT
  if (!(psiIsT && M->sumPsiValid) || M->p2pConnected) sum_psi(M, psi);
  if (host_halo(M)) exchange_field(M, psi, ws.recvT);
  if (fromAssembly) {
    ctx->launch(LF_K_ASSEMBLE, [&] {
      M->upperStale = !M->ld.writeUpper;
      launch_assemble(s, M->Lasm, mesh_for(M, p), M->ld, p->DT, 1.0 / p->dt, psi, M->haloT(), true, ws, T0,
                      lapSrc);
    });
  } else {
    ctx->launch(LF_K_SETUP, [&] { launch_pcg_setup(s, M->Lsetup, M->md, M->ld, M->haloT(), ws); });
  }
  if (overlap_halo(M))
    start_w_halo(M);  // w of the setup for iteration 0, on the comm stream
  else if (host_halo(M))
    exchange_field(M, ws.w, ws.recvW);  // w of the setup for iteration 0
  allreduce(M, ws.lsum->setup, ws.gsum->setup, 3);
  run_iterations(M, out);
  // gsum->p1[1] now holds sum(psi) of the final psi (last phase-1 launch)
  M->sumPsiValid = psiIsT;
}

}  // namespace lf
