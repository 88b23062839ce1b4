// C ABI entry points (include/lfoam.h).  Every call catches everything and
// maps it to an lf_status; nothing throws or aborts across the boundary.
#include <cmath>
#include <cstdio>

#include "host.h"

using namespace lf;

namespace lf {
void mesh_create_impl(lf_context *ctx, const lf_mesh_desc *d, lf_mesh **out);
}

static thread_local std::string g_last_error;

template <class F>
static lf_status guard(F &&fn, lf_mesh *M = nullptr) {
  try {
    if (M && M->broken) throw Error{LF_ERR_STATE, "mesh unusable after an earlier CUDA/NCCL error"};
    if (M && M->ctx) LF_CUDA(cudaSetDevice(M->ctx->device));  // the mesh's device, whatever the caller's current one
    fn();
    return LF_OK;
  } catch (const Error &e) {
    g_last_error = e.msg;
    if (M && (e.st == LF_ERR_CUDA || e.st == LF_ERR_NCCL)) M->broken = true;
    return e.st;
  } catch (const std::bad_alloc &) {
    g_last_error = "host allocation failed";
    return LF_ERR_OOM;
  } catch (const std::exception &e) {
    g_last_error = e.what();
    return LF_ERR_INTERNAL;
  } catch (...) {
    g_last_error = "unknown exception";
    return LF_ERR_INTERNAL;
  }
}

// ------------------------------------------------------------- context
void lf_context::launch(int kind, const std::function<void()> &fn) {
  if (capturing) {  // recorded into a graph; counted when the graph is launched
    fn();
    LF_CUDA(cudaGetLastError());
    return;
  }
  if (instrument) {
    cudaEvent_t a = event(), b = event();
    LF_CUDA(cudaEventRecord(a, stream));
    fn();
    LF_CUDA(cudaGetLastError());
    LF_CUDA(cudaEventRecord(b, stream));
    pending.push_back({kind, a, b});
  } else {
    fn();
    LF_CUDA(cudaGetLastError());
  }
  ++launches;
  ++kLaunches[kind];
}

cudaEvent_t lf_context::event() {
  if (!evFree.empty()) {
    cudaEvent_t e = evFree.back();
    evFree.pop_back();
    return e;
  }
  cudaEvent_t e;
  LF_CUDA(cudaEventCreate(&e));
  return e;
}

void lf_context::harvest() {
  for (const Pending &p : pending) {
    float ms = 0.f;
    LF_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
    kMs[p.kind] += ms;
    evFree.push_back(p.a);
    evFree.push_back(p.b);
  }
  pending.clear();
}

lf_context::~lf_context() {
  if (stream) cudaStreamSynchronize(stream);
  for (auto &p : pending) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : evFree) cudaEventDestroy(e);
  if (commStream) cudaStreamSynchronize(commStream);
  if (commHalo) nccl_comm_destroy(commHalo);
  if (comm) nccl_comm_destroy(comm);
  if (commStream) cudaStreamDestroy(commStream);
  if (evPacked) cudaEventDestroy(evPacked);
  if (evHalo) cudaEventDestroy(evHalo);
  if (ownStream && stream) cudaStreamDestroy(stream);
}

extern "C" {

const char *lf_status_string(lf_status s) {
  switch (s) {
    case LF_OK: return "LF_OK";
    case LF_ERR_INVALID_ARG: return "LF_ERR_INVALID_ARG";
    case LF_ERR_STATE: return "LF_ERR_STATE";
    case LF_ERR_OOM: return "LF_ERR_OOM";
    case LF_ERR_CUDA: return "LF_ERR_CUDA";
    case LF_ERR_NCCL: return "LF_ERR_NCCL";
    case LF_ERR_INTERNAL: return "LF_ERR_INTERNAL";
  }
  return "LF_ERR_UNKNOWN";
}

const char *lf_last_error(void) { return g_last_error.c_str(); }

int lf_version(void) { return LF_VERSION; }

lf_status lf_context_create(int device, void *cuda_stream, lf_context **out) {
  return guard([&] {
    LF_REQUIRE(out != nullptr, "out is NULL");
    int ndev = 0;
    LF_CUDA(cudaGetDeviceCount(&ndev));
    LF_REQUIRE(device >= 0 && device < ndev, "device ordinal out of range");
    LF_CUDA(cudaSetDevice(device));
    std::unique_ptr<lf_context> c(new lf_context());
    c->device = device;
    LF_CUDA(cudaDeviceGetAttribute(&c->smCount, cudaDevAttrMultiProcessorCount, device));
    if (cuda_stream) {
      c->stream = static_cast<cudaStream_t>(cuda_stream);
    } else {
      LF_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->ownStream = true;
    }
    *out = c.release();
  });
}

lf_status lf_context_destroy(lf_context *ctx) {
  return guard([&] { delete ctx; });
}

lf_status lf_comm_unique_id(void *out) {
  return guard([&] {
    LF_REQUIRE(out != nullptr, "out is NULL");
    nccl_unique_id(out);
  });
}

lf_status lf_comm_init(lf_context *ctx, const void *uid, int nranks, int rank) {
  return guard([&] {
    LF_REQUIRE(ctx && uid, "NULL argument");
    LF_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "bad nranks/rank");
    LF_REQUIRE(ctx->comm == nullptr, "communicator already initialised");
    LF_REQUIRE(!ctx->p2p, "context already uses the peer-memory transport");
    ctx->comm = nccl_comm_init(uid, nranks, rank, ctx->device);
    ctx->nranks = nranks;
    ctx->rank = rank;
    ctx->commHalo = nccl_comm_split(ctx->comm, rank);
    LF_CUDA(cudaStreamCreateWithFlags(&ctx->commStream, cudaStreamNonBlocking));
    LF_CUDA(cudaEventCreateWithFlags(&ctx->evPacked, cudaEventDisableTiming));
    LF_CUDA(cudaEventCreateWithFlags(&ctx->evHalo, cudaEventDisableTiming));
  });
}

lf_status lf_p2p_init(lf_context *ctx, int nranks, int rank) {
  return guard([&] {
    LF_REQUIRE(ctx != nullptr, "ctx is NULL");
    p2p_init(ctx, nranks, rank);
  });
}

lf_status lf_p2p_export(lf_mesh *M, void *handle) {
  return guard([&] {
    LF_REQUIRE(M && handle, "NULL argument");
    p2p_export(M, handle);
  }, M);
}

lf_status lf_p2p_connect(lf_mesh *M, int nranks, int rank, const void *handles) {
  return guard([&] {
    LF_REQUIRE(M && handles, "NULL argument");
    p2p_connect(M, nranks, rank, handles);
  }, M);
}

lf_status lf_comm_info(const lf_context *ctx, int *nranks, int *rank) {
  return guard([&] {
    LF_REQUIRE(ctx != nullptr, "ctx is NULL");
    if (nranks) *nranks = ctx->nranks;
    if (rank) *rank = ctx->rank;
  });
}

// ---------------------------------------------------------------- mesh
lf_status mesh_create(lf_context *ctx, const lf_mesh_desc *desc, lf_mesh **out) {
  return guard([&] { mesh_create_impl(ctx, desc, out); });
}

lf_status mesh_destroy(lf_mesh *mesh) {
  return guard([&] {
    if (mesh) cudaStreamSynchronize(mesh->ctx->stream);
    delete mesh;
  });
}

lf_status lf_mesh_info(const lf_mesh *M, int32_t *n, int32_t *F, int32_t *B, int64_t *bytes) {
  return guard([&] {
    LF_REQUIRE(M != nullptr, "mesh is NULL");
    if (n) *n = M->n;
    if (F) *F = M->F;
    if (B) *B = M->B;
    if (bytes) *bytes = M->arena.bytes;
  });
}

lf_status lf_mesh_layout(const lf_mesh *M, int32_t *ell_width, int32_t *row_width, int32_t *label_escapes) {
  return guard([&] {
    LF_REQUIRE(M != nullptr, "mesh is NULL");
    if (ell_width) *ell_width = M->md.K;
    if (row_width) *row_width = M->md.KS;
    if (label_escapes) *label_escapes = M->md.codeE ? M->ell16Escapes : -1;
  });
}

lf_status lf_mesh_export_addressing(const lf_mesh *M, int32_t *owner_start, int32_t *losort,
                                    int32_t *losort_start, int32_t *face_order, int32_t *cell_order) {
  return guard([&] {
    LF_REQUIRE(M != nullptr, "mesh is NULL");
    cudaStream_t s = M->ctx->stream;
    auto cp = [&](int32_t *dst, const int32_t *src, size_t cnt) {
      if (dst && cnt) LF_CUDA(cudaMemcpyAsync(dst, src, sizeof(int32_t) * cnt, cudaMemcpyDeviceToHost, s));
    };
    cp(owner_start, M->md.ownerStart, M->n + 1);
    cp(losort, M->md.losort, M->F);
    cp(losort_start, M->md.losortStart, M->n + 1);
    cp(face_order, M->facePerm, M->F);
    if (cell_order) {
      if (M->renumbered)
        cp(cell_order, M->cellPerm, M->n);
      else
        for (int32_t i = 0; i < M->n; ++i) cell_order[i] = i;
    }
    LF_CUDA(cudaStreamSynchronize(s));
  }, const_cast<lf_mesh *>(M));
}

lf_status lf_permute(const lf_mesh *M, int to_internal, const double *in, double *out) {
  return guard([&] {
    LF_REQUIRE(M && in && out, "NULL argument");
    LF_REQUIRE(in != out, "in and out must not alias");
    cudaStream_t s = M->ctx->stream;
    if (!M->renumbered) {
      LF_CUDA(cudaMemcpyAsync(out, in, sizeof(double) * M->n, cudaMemcpyDeviceToDevice, s));
    } else {
      // internal[i] = caller[cellPerm[i]]  /  caller[cellPerm[i]] = internal[i]
      launch_permute(s, M->n, M->cellPerm, in, out, !to_internal);
      LF_CUDA(cudaGetLastError());
    }
  }, const_cast<lf_mesh *>(M));
}

// --------------------------------------------------------------- fields
lf_status field_set(lf_mesh *M, lf_field f, int32_t patch, const double *v, int64_t n, int on_device) {
  return guard([&] {
    LF_REQUIRE(M && v, "NULL argument");
    cudaStream_t s = M->ctx->stream;
    const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (f == LF_FIELD_T) {
      LF_REQUIRE(patch == -1, "patch must be -1 for LF_FIELD_T");
      LF_REQUIRE(n == M->n, "n must equal n_cells");
      if (!M->renumbered) {
        LF_CUDA(cudaMemcpyAsync(M->T, v, sizeof(double) * n, kind, s));
      } else {
        LF_CUDA(cudaMemcpyAsync(M->scratch, v, sizeof(double) * n, kind, s));
        launch_permute(s, M->n, M->cellPerm, M->scratch, M->T, false);
      }
      M->sumPsiValid = false;
    } else if (f == LF_FIELD_DT) {
      LF_REQUIRE(patch == -1, "patch must be -1 for LF_FIELD_DT");
      LF_REQUIRE(n == M->n, "n must equal n_cells");
      LF_REQUIRE(M->hasGeom, "a DT field needs the full geometry (interpolation weights)");
      LF_REQUIRE(M->nproc == 0 || M->procGeom, "a DT field across processor patches needs the patches' cf and cn");
      {
        // validated on the host either way (a device field is copied back once:
        // DT is set once per case, not per step)
        std::vector<double> hv;
        const double *chk = v;
        if (on_device) {
          hv.resize(n);
          LF_CUDA(cudaMemcpyAsync(hv.data(), v, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
          LF_CUDA(cudaStreamSynchronize(s));
          chk = hv.data();
        }
        for (int64_t i = 0; i < n; ++i)
          LF_REQUIRE(chk[i] > 0.0 && std::isfinite(chk[i]), "DT must be > 0 and finite");
      }
      if (!M->DTc) {
        M->DTc = M->arena.alloc<double>(M->n);
        M->gammaF = M->arena.alloc<double>(M->F);
        M->gammaB = M->arena.alloc<double>(M->B);
      }
      if (!M->renumbered) {
        LF_CUDA(cudaMemcpyAsync(M->DTc, v, sizeof(double) * n, kind, s));
      } else {
        LF_CUDA(cudaMemcpyAsync(M->scratch, v, sizeof(double) * n, kind, s));
        launch_permute(s, M->n, M->cellPerm, M->scratch, M->DTc, false);
      }
      vector_halo(M, M->DTc, M->n, 1);  // the coupled cells' DT (collective)
      M->ctx->launch(LF_K_NONORTH, [&] {
        launch_face_gamma(s, M->md, M->geo, M->ownerInt, M->bCell, M->DTc, M->ws.recvX, M->gammaF, M->gammaB);
      });
      M->mdVar = M->md;
      M->mdVar.gammaF = M->gammaF;
      M->mdVar.gammaB = M->gammaB;
      M->dtSet = true;
    } else if (f == LF_FIELD_PATCH_VALUE) {
      LF_REQUIRE(patch >= 0 && patch < M->nPatches, "patch out of range");
      const int32_t off = M->patchStart[patch], cnt = M->patchStart[patch + 1] - off;
      LF_REQUIRE(n == cnt, "n must equal the patch's n_faces");
      if (M->patchType[patch] == LF_PATCH_FIXED_VALUE)
        LF_CUDA(cudaMemcpyAsync(M->bValue + off, v, sizeof(double) * n, kind, s));
    } else {
      throw Error{LF_ERR_INVALID_ARG, "unknown field"};
    }
    if (!on_device) LF_CUDA(cudaStreamSynchronize(s));
    LF_CUDA(cudaGetLastError());
  }, M);
}

lf_status field_get(const lf_mesh *Mc, lf_field f, int32_t patch, double *v, int64_t n, int on_device) {
  lf_mesh *M = const_cast<lf_mesh *>(Mc);
  return guard([&] {
    LF_REQUIRE(M && v, "NULL argument");
    cudaStream_t s = M->ctx->stream;
    const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (f == LF_FIELD_T) {
      LF_REQUIRE(patch == -1, "patch must be -1 for LF_FIELD_T");
      LF_REQUIRE(n == M->n, "n must equal n_cells");
      if (!M->renumbered) {
        LF_CUDA(cudaMemcpyAsync(v, M->T, sizeof(double) * n, kind, s));
      } else {
        launch_permute(s, M->n, M->cellPerm, M->T, M->scratch, true);
        LF_CUDA(cudaMemcpyAsync(v, M->scratch, sizeof(double) * n, kind, s));
      }
    } else if (f == LF_FIELD_DT) {
      LF_REQUIRE(patch == -1, "patch must be -1 for LF_FIELD_DT");
      LF_REQUIRE(n == M->n, "n must equal n_cells");
      if (!M->dtSet) throw Error{LF_ERR_STATE, "the DT field was never set"};
      if (!M->renumbered) {
        LF_CUDA(cudaMemcpyAsync(v, M->DTc, sizeof(double) * n, kind, s));
      } else {
        launch_permute(s, M->n, M->cellPerm, M->DTc, M->scratch, true);
        LF_CUDA(cudaMemcpyAsync(v, M->scratch, sizeof(double) * n, kind, s));
      }
    } else if (f == LF_FIELD_PATCH_VALUE) {
      LF_REQUIRE(patch >= 0 && patch < M->nPatches, "patch out of range");
      const int32_t off = M->patchStart[patch], cnt = M->patchStart[patch + 1] - off;
      LF_REQUIRE(n == cnt, "n must equal the patch's n_faces");
      const int t = M->patchType[patch];
      if (cnt > 0) {
        if (t == LF_PATCH_FIXED_VALUE) {
          LF_CUDA(cudaMemcpyAsync(v, M->bValue + off, sizeof(double) * n, kind, s));
        } else if (t == LF_PATCH_ZERO_GRADIENT) {  // correctBoundaryConditions: T_b = T[faceCells]
          launch_gather_f64(s, cnt, M->bCell + off, M->T, M->scratch);
          LF_CUDA(cudaMemcpyAsync(v, M->scratch, sizeof(double) * n, kind, s));
        } else {
          LF_CUDA(cudaMemsetAsync(M->scratch, 0, sizeof(double) * n, s));
          LF_CUDA(cudaMemcpyAsync(v, M->scratch, sizeof(double) * n, kind, s));
        }
      }
    } else {
      throw Error{LF_ERR_INVALID_ARG, "unknown field"};
    }
    if (!on_device) LF_CUDA(cudaStreamSynchronize(s));
    LF_CUDA(cudaGetLastError());
  }, M);
}

// -------------------------------------------------------------- assembly
lf_status laplacian_assemble(lf_mesh *M, const lf_laplacian_params *p, lf_ldu **sys) {
  return guard([&] {
    LF_REQUIRE(M && p, "NULL argument");
    LF_REQUIRE(p->DT > 0.0 && p->dt > 0.0, "DT and dt must be > 0");
    lf_context *ctx = M->ctx;
    cudaStream_t s = ctx->stream;
    const MeshDev &md = mesh_for(M, p);
    const double *lapSrc = nullptr;
    if (p->corrected) {
      require_corrected(M);
      correction_source(M, md, p->DT, M->T);
      lapSrc = M->lapSrc;
    }
    field_halo(M, M->T);
    ctx->launch(LF_K_ASSEMBLE, [&] {
      M->upperStale = !M->ld.writeUpper;
      launch_assemble(s, M->Lasm, md, M->ld, p->DT, 1.0 / p->dt, M->T, M->haloT(), false, M->ws, nullptr,
                      lapSrc);
    });
    M->ldu.assembled = true;
    if (sys) *sys = &M->ldu;
  }, M);
}

lf_status lf_ldu_export(const lf_ldu *sys, double *diag, double *upper, double *source,
                        double *internal_coeffs, double *boundary_coeffs) {
  lf_mesh *M = sys ? sys->mesh : nullptr;
  return guard([&] {
    LF_REQUIRE(sys && M, "NULL ldu");
    LF_REQUIRE(sys->assembled, "ldu not assembled");
    cudaStream_t s = M->ctx->stream;
    auto cell = [&](double *dst, const double *src) {
      if (!dst) return;
      if (M->renumbered) {
        launch_permute(s, M->n, M->cellPerm, src, M->scratch, true);
        src = M->scratch;
      }
      LF_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * M->n, cudaMemcpyDeviceToHost, s));
      LF_CUDA(cudaStreamSynchronize(s));
    };
    cell(diag, M->ld.diag);
    cell(source, M->ld.source);
    if (upper && M->F > 0) {
      std::vector<double> tmp(M->F);
      std::vector<int32_t> perm(M->F);
      ensure_upper(M);
      LF_CUDA(cudaMemcpyAsync(tmp.data(), M->ld.upper, sizeof(double) * M->F, cudaMemcpyDeviceToHost, s));
      LF_CUDA(cudaMemcpyAsync(perm.data(), M->facePerm, sizeof(int32_t) * M->F, cudaMemcpyDeviceToHost, s));
      LF_CUDA(cudaStreamSynchronize(s));
      for (int32_t i = 0; i < M->F; ++i) upper[perm[i]] = tmp[i];
    }
    if (internal_coeffs && M->B)
      LF_CUDA(cudaMemcpyAsync(internal_coeffs, M->ld.bInt, sizeof(double) * M->B, cudaMemcpyDeviceToHost, s));
    if (boundary_coeffs && M->B)
      LF_CUDA(cudaMemcpyAsync(boundary_coeffs, M->ld.bBnd, sizeof(double) * M->B, cudaMemcpyDeviceToHost, s));
    LF_CUDA(cudaStreamSynchronize(s));
  }, M);
}

lf_status ldu_amul(const lf_ldu *sys, const double *x, double *y) {
  lf_mesh *M = sys ? sys->mesh : nullptr;
  return guard([&] {
    LF_REQUIRE(sys && M && x && y, "NULL argument");
    LF_REQUIRE(x != y, "x and y must not alias");
    LF_REQUIRE(sys->assembled, "ldu not assembled");
    lf_context *ctx = M->ctx;
    cudaStream_t s = ctx->stream;
    field_halo(M, x);
    ctx->launch(LF_K_AMUL, [&] { launch_amul(s, M->Lamul, M->md, M->ld, M->haloT(), x, y); });
  }, M);
}

// ------------------------------------------------------------- fvc::grad
lf_status lf_fvc_grad(lf_mesh *M, const double *x, double *grad, double *bgrad) {
  return guard([&] {
    LF_REQUIRE(M && x && grad, "NULL argument");
    require_corrected(M);
    lf_context *ctx = M->ctx;
    cudaStream_t s = ctx->stream;
    field_halo(M, x);
    ctx->launch(LF_K_NONORTH, [&] { launch_grad(s, M->Lasm, M->md, M->geo, x, M->haloT(), M->gradS, grad); });
    if (bgrad)
      ctx->launch(LF_K_NONORTH, [&] { launch_grad_bc(s, M->md, M->geo, M->bCell, x, M->gradS, bgrad); });
  }, M);
}

// ------------------------------------------------------------------- PCG
lf_status ldu_precondition(const lf_ldu *sys, int32_t precond, const double *r, double *w, double *rD) {
  lf_mesh *M = sys ? sys->mesh : nullptr;
  return guard([&] {
    LF_REQUIRE(sys && M && r && w, "NULL argument");
    LF_REQUIRE(r != w && r != rD && w != rD, "r, w and rD must not alias");
    LF_REQUIRE(sys->assembled, "ldu not assembled");
    LF_REQUIRE(precond >= LF_PRECOND_DIAGONAL && precond <= LF_PRECOND_GAMG, "unknown preconditioner");
    if (precond == LF_PRECOND_GAMG)
      gamg_precondition(M, r, w, rD);
    else
      precondition(M, precond, r, w, rD);
  }, M);
}

// ------------------------------------------------------------------ GAMG
lf_status lf_gamg_hierarchy(lf_mesh *M, int32_t *n_levels, int32_t *cells, int32_t *faces, int32_t *agg) {
  return guard([&] {
    LF_REQUIRE(M != nullptr, "mesh is NULL");
    gamg_hierarchy(M, n_levels, cells, faces, agg);
  }, M);
}

lf_status lf_gamg_export(const lf_ldu *sys, int32_t level, double *D, double *U, int32_t *face_l,
                         int32_t *face_u) {
  lf_mesh *M = sys ? sys->mesh : nullptr;
  return guard([&] {
    LF_REQUIRE(sys && M, "NULL ldu");
    if (!M->gamgFormed) throw Error{LF_ERR_STATE, "no GAMG solve or application yet"};
    LF_CUDA(cudaStreamSynchronize(M->ctx->stream));
    gamg_export(M, level, D, U, face_l, face_u);
  }, M);
}

lf_status pcg_solve(lf_ldu *sys, double *psi, const lf_solver_controls *c, lf_solver_perf *out) {
  lf_mesh *M = sys ? sys->mesh : nullptr;
  return guard([&] {
    LF_REQUIRE(sys && M && psi && c, "NULL argument");
    LF_REQUIRE(sys->assembled, "ldu not assembled");
    upload_controls(M, c, psi);
    solve_loop(M, c, psi, false, nullptr, out);
  }, M);
}

lf_status laplacianFoam_step(lf_mesh *M, const lf_laplacian_params *p, const lf_solver_controls *c,
                             int32_t n_steps, lf_solver_perf *per_step) {
  return guard([&] {
    LF_REQUIRE(M && p && c, "NULL argument");
    LF_REQUIRE(p->DT > 0.0 && p->dt > 0.0, "DT and dt must be > 0");
    LF_REQUIRE(n_steps >= 0, "n_steps must be >= 0");
    if (p->corrected) {
      require_corrected(M);
      LF_REQUIRE(p->n_non_orth_correctors >= 0, "n_non_orth_correctors must be >= 0");
    }
    const MeshDev &md = mesh_for(M, p);  // validates variable_DT up front
    if (n_steps == 0) return;
    upload_controls(M, c, M->T);
    if (!p->corrected) {
      for (int32_t st = 0; st < n_steps; ++st) {
        solve_loop(M, c, M->T, true, p, per_step ? per_step + st : nullptr);
        M->ldu.assembled = true;
      }
      return;
    }
    // simple.correctNonOrthogonal() loop: ddt keeps T0 of the step,
    // each pass re-evaluates the explicit correction from the current T
    const int32_t passes = 1 + p->n_non_orth_correctors;
    const bool keepT0 = passes > 1;
    for (int32_t st = 0; st < n_steps; ++st) {
      if (keepT0)
        LF_CUDA(cudaMemcpyAsync(M->T0, M->T, sizeof(double) * M->n, cudaMemcpyDeviceToDevice, M->ctx->stream));
      for (int32_t k = 0; k < passes; ++k) {
        correction_source(M, md, p->DT, M->T);
        solve_loop(M, c, M->T, true, p, per_step ? per_step + (int64_t)st * passes + k : nullptr,
                   keepT0 ? M->T0 : nullptr, M->lapSrc);
        M->ldu.assembled = true;
      }
    }
  }, M);
}

// -------------------------------------------------------- instrumentation
lf_status lf_set_instrumentation(lf_context *ctx, int enable) {
  return guard([&] {
    LF_REQUIRE(ctx != nullptr, "ctx is NULL");
    LF_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->harvest();
    ctx->instrument = enable != 0;
    ctx->kLaunches.fill(0);
    ctx->kMs.fill(0.0);
    ctx->launches = 0;
  });
}

lf_status lf_kernel_stats(const lf_context *ctx, lf_kernel_kind k, int64_t *launches, double *ms) {
  return guard([&] {
    LF_REQUIRE(ctx != nullptr, "ctx is NULL");
    LF_REQUIRE(k >= 0 && k < LF_K_COUNT, "bad kernel kind");
    LF_CUDA(cudaStreamSynchronize(ctx->stream));
    const_cast<lf_context *>(ctx)->harvest();
    if (launches) *launches = ctx->kLaunches[k];
    if (ms) *ms = ctx->kMs[k];
  });
}

lf_status lf_set_option(lf_context *ctx, lf_option opt, int value) {
  return guard([&] {
    LF_REQUIRE(ctx != nullptr, "ctx is NULL");
    if (opt == LF_OPT_PERSISTENT)
      ctx->persistent = value != 0;
    else if (opt == LF_OPT_GRAPHS)
      ctx->useGraphs = value != 0;
    else if (opt == LF_OPT_SOLVE_VARIANT) {
      LF_REQUIRE(value >= 0 && value <= 2, "solve variant must be 0, 1 or 2");
      ctx->solveVariant = value;
    } else if (opt == LF_OPT_COMPRESSED_LABELS)
      ctx->compressedLabels = value != 0;
    else if (opt == LF_OPT_OVERLAP_HALO)
      ctx->overlapHalo = value != 0;
    else if (opt == LF_OPT_DYNAMIC_TRIPS) {
      LF_REQUIRE(value >= -1 && value <= 100, "dynamic trips must be -1 (default) or a percentage 0..100");
      ctx->dynPct = value;
    } else if (opt == LF_OPT_L2_PREFETCH) {
      LF_REQUIRE(value >= 0 && value <= 2, "l2 prefetch must be 0 (by mesh), 1 (on) or 2 (off)");
      ctx->l2Prefetch = value;
    }
    else
      throw Error{LF_ERR_INVALID_ARG, "unknown option"};
  });
}

lf_status lf_launch_count(const lf_context *ctx, int64_t *n) {
  return guard([&] {
    LF_REQUIRE(ctx && n, "NULL argument");
    *n = ctx->launches;
  });
}

}  // extern "C"
