// Non-orthogonal correction path: the gradient kernels
// the paper ported to the GPU (§5.2) and the explicit part of the Gauss
// linear corrected laplacian.
//
// Every kernel is an atomic-free per-item GATHER over the same lists the
// assembly uses (ownerStart/nbr for owned faces, losort/losortOwner for
// neighbour-side faces, abStart/abFace for boundary faces) — the paper's
// replacement of the serial owner/neighbour scatter by
// ownerStart / neighbourList loops and of the boundary scatter by
// facePatchIndex/facePatchStart.  A cell visits its faces in the
// order a serial face loop would reach it (neighbour-side faces have a lower
// owner, hence come first in upper-triangular order; then owned faces; then
// boundary faces in patch order), and every operation is an explicitly
// rounded _rn intrinsic (no FMA contraction), so on an upper-triangular mesh
// the results equal the serial scatter bit for bit.
//
// These run once per corrector pass, outside the PCG loop; they are plain
// HBM-bound FP64 sweeps.
#include "lfoam_internal.h"

namespace lf {

namespace {
constexpr int NB = 256;
constexpr double ROOTVSMALL = 1e-150;  // OpenFOAM's ROOTVSMALL (double)

__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dvd(double a, double b) { return __ddiv_rn(a, b); }

// surfaceInterpolation::makeWeights (Listing "weights parallel loop",
// P:321-334) and nonOrthCorrectionVectors (n - d*deltaCoeffs), per internal
// face.  Inputs AoS [F][3] in internal face order and orientation, cell
// centres AoS [n][3] internal numbering; outputs SoA [3][F].
__global__ void __launch_bounds__(NB) k_weights_corr(int32_t F, const int32_t *__restrict__ owner,
                                                     const int32_t *__restrict__ nbr,
                                                     const double *__restrict__ SfA,
                                                     const double *__restrict__ CfA,
                                                     const double *__restrict__ CA,
                                                     const double *__restrict__ magSf,
                                                     const double *__restrict__ delta, double *__restrict__ w,
                                                     double *__restrict__ corr, double *__restrict__ SfS) {
  for (int32_t f = blockIdx.x * blockDim.x + threadIdx.x; f < F; f += gridDim.x * blockDim.x) {
    const int32_t P = owner[f], N = nbr[f];
    double so = 0.0, sn = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double s = SfA[3 * (size_t)f + k], cf = CfA[3 * (size_t)f + k];
      so = add(so, mul(s, sub(cf, CA[3 * (size_t)P + k])));
      sn = add(sn, mul(s, sub(CA[3 * (size_t)N + k], cf)));
    }
    so = fabs(so);
    sn = fabs(sn);
    const double sum = add(so, sn);
    w[f] = fabs(sum) > ROOTVSMALL ? dvd(sn, sum) : 0.5;
    const double m = magSf[f], dl = delta[f];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double s = SfA[3 * (size_t)f + k];
      const double nk = dvd(s, m);
      const double dk = sub(CA[3 * (size_t)N + k], CA[3 * (size_t)P + k]);
      corr[(size_t)k * F + f] = sub(nk, mul(dk, dl));
      SfS[(size_t)k * F + f] = s;
    }
  }
}

// gaussGrad::gradf with linear interpolation, per cell: sum over faces of
// Sf * (lambda (x_P - x_N) + x_N) (P:293-299 interpolation, P:435-452 gradf
// gathers), + boundary Sf * x_b, / V.
__global__ void __launch_bounds__(NB) k_grad(MeshDev m, GeomDev g, const double *__restrict__ x,
                                             const double *__restrict__ halo, double *__restrict__ gradS,
                                             double *__restrict__ gradA) {
  const int32_t n = m.n, F = g.F, B = g.B;
  for (int32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    const double xc = x[c];
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    for (int32_t j = m.losortStart[c], e = m.losortStart[c + 1]; j < e; ++j) {
      const int32_t f = m.losort[j], P = m.losortOwner[j];
      const double ssf = add(mul(g.w[f], sub(x[P], xc)), xc);
      a0 = sub(a0, mul(g.Sf[f], ssf));
      a1 = sub(a1, mul(g.Sf[(size_t)F + f], ssf));
      a2 = sub(a2, mul(g.Sf[2 * (size_t)F + f], ssf));
    }
    for (int32_t f = m.ownerStart[c], e = m.ownerStart[c + 1]; f < e; ++f) {
      const double xN = x[m.nbr[f]];
      const double ssf = add(mul(g.w[f], sub(xc, xN)), xN);
      a0 = add(a0, mul(g.Sf[f], ssf));
      a1 = add(a1, mul(g.Sf[(size_t)F + f], ssf));
      a2 = add(a2, mul(g.Sf[2 * (size_t)F + f], ssf));
    }
    for (int32_t j = g.abStart[c], e = g.abStart[c + 1]; j < e; ++j) {
      const int32_t i = g.abFace[j];
      const int t = m.bType[i];
      double pssf;
      if (t == LF_PATCH_FIXED_VALUE) {
        pssf = m.bValue[i];
      } else if (t == LF_PATCH_PROCESSOR && g.bW) {
        // coupled face: linear interpolation with the neighbour rank's cell
        // value (halo), the internal-face formula with this cell as owner
        const double xN = halo[m.bSlot[i]];
        pssf = add(mul(g.bW[i], sub(xc, xN)), xN);
      } else {
        pssf = xc;
      }
      a0 = add(a0, mul(g.bSf[i], pssf));
      a1 = add(a1, mul(g.bSf[(size_t)B + i], pssf));
      a2 = add(a2, mul(g.bSf[2 * (size_t)B + i], pssf));
    }
    const double V = m.V[c];
    a0 = dvd(a0, V);
    a1 = dvd(a1, V);
    a2 = dvd(a2, V);
    if (gradS) {
      gradS[c] = a0;
      gradS[(size_t)n + c] = a1;
      gradS[2 * (size_t)n + c] = a2;
    }
    if (gradA) {
      gradA[3 * (size_t)c] = a0;
      gradA[3 * (size_t)c + 1] = a1;
      gradA[3 * (size_t)c + 2] = a2;
    }
  }
}

// correctBoundaryConditions of the gradient (Listing P:539-556), per
// boundary face: gb = grad[faceCell] + n (snGrad - n.grad[faceCell]) on
// non-coupled patches.  Output AoS [B][3].
__global__ void __launch_bounds__(NB) k_grad_bc(MeshDev m, GeomDev g, const int32_t *__restrict__ bCell,
                                                const double *__restrict__ x, const double *__restrict__ gradS,
                                                double *__restrict__ bgradA) {
  const int32_t n = m.n, B = g.B;
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < B; i += gridDim.x * blockDim.x) {
    const int32_t c = bCell[i];
    double gb[3], nv[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      gb[k] = gradS[(size_t)k * n + c];
      nv[k] = dvd(g.bSf[(size_t)k * B + i], m.bMagSf[i]);
    }
    const int t = m.bType[i];
    if (t != LF_PATCH_PROCESSOR) {
      double ng = 0.0;
#pragma unroll
      for (int k = 0; k < 3; ++k) ng = add(ng, mul(nv[k], gb[k]));
      const double sng = t == LF_PATCH_FIXED_VALUE ? mul(m.bDelta[i], sub(m.bValue[i], x[c])) : 0.0;
      const double dn = sub(sng, ng);
#pragma unroll
      for (int k = 0; k < 3; ++k) gb[k] = add(gb[k], mul(nv[k], dn));
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) bgradA[3 * (size_t)i + k] = gb[k];
  }
}

__device__ __forceinline__ double face_flux(const GeomDev &g, const MeshDev &m, double DT, int32_t f,
                                            const double *__restrict__ gradS, int32_t P, int32_t N) {
  const int32_t n = m.n, F = g.F;
  const double w = g.w[f];
  double cs = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {  // dotInterpolate(corrVecs, grad)
    const double gP = gradS[(size_t)k * n + P], gN = gradS[(size_t)k * n + N];
    cs = add(cs, mul(g.corr[(size_t)k * F + f], add(mul(w, sub(gP, gN)), gN)));
  }
  return mul(mul(m.gammaF ? m.gammaF[f] : DT, m.magSf[f]), cs);
}

// Explicit non-orthogonal part of gaussLaplacianScheme::fvmLaplacian:
// lapSrc = -V * div(DT |Sf| corrVecs . interpolate(grad T)), per cell
// (surfaceIntegrate: owner +, neighbour -; non-coupled boundary faces carry
// no correction).
__global__ void __launch_bounds__(NB) k_lap_corr(MeshDev m, GeomDev g, double DT,
                                                 const double *__restrict__ gradS,
                                                 const double *__restrict__ haloG, int32_t nproc,
                                                 double *__restrict__ lapSrc) {
  const int32_t n = m.n, B = g.B;
  for (int32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int32_t j = m.losortStart[c], e = m.losortStart[c + 1]; j < e; ++j)
      acc = sub(acc, face_flux(g, m, DT, m.losort[j], gradS, m.losortOwner[j], c));
    for (int32_t f = m.ownerStart[c], e = m.ownerStart[c + 1]; f < e; ++f)
      acc = add(acc, face_flux(g, m, DT, f, gradS, c, m.nbr[f]));
    if (m.hasProc && g.bW) {
      // coupled faces (outward from this cell): corrVec . (w grad_P + (1-w)
      // grad_N) with the neighbour rank's gradient (halo)
      for (int32_t kk = m.pcStart[c], e = m.pcStart[c + 1]; kk < e; ++kk) {
        const int32_t i = m.pcFace[kk], sl = m.bSlot[i];
        const double w = g.bW[i];
        double cs = 0.0;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const double gP = gradS[(size_t)k * n + c], gN = haloG[(size_t)k * nproc + sl];
          cs = add(cs, mul(g.bCorr[(size_t)k * B + i], add(mul(w, sub(gP, gN)), gN)));
        }
        acc = add(acc, mul(mul(m.gammaB ? m.gammaB[i] : DT, m.bMagSf[i]), cs));
      }
    }
    const double V = m.V[c];
    lapSrc[c] = -mul(V, dvd(acc, V));
  }
}

// Face diffusivity of a cell DT field (§8(f) row 2): linear interpolation
// gamma_f = w (DT_P - DT_N) + DT_N (P:293-299 with the weights of P:321-334),
// boundary faces DT[faceCell].
__global__ void __launch_bounds__(NB) k_face_gamma(MeshDev m, GeomDev g, const int32_t *__restrict__ owner,
                                                   const int32_t *__restrict__ bCell,
                                                   const double *__restrict__ DTc,
                                                   const double *__restrict__ haloDT,
                                                   double *__restrict__ gammaF, double *__restrict__ gammaB) {
  const int32_t F = g.F, B = g.B;
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < F + B; i += gridDim.x * blockDim.x) {
    if (i < F) {
      const double dN = DTc[m.nbr[i]];
      gammaF[i] = add(mul(g.w[i], sub(DTc[owner[i]], dN)), dN);
    } else {
      const int32_t b = i - F;
      if (g.bW && m.bType[b] == LF_PATCH_PROCESSOR) {  // the coupled cell's DT (halo)
        const double dN = haloDT[m.bSlot[b]];
        gammaB[b] = add(mul(g.bW[b], sub(DTc[bCell[b]], dN)), dN);
      } else {
        gammaB[b] = DTc[bCell[b]];
      }
    }
  }
}

int grid_for(int64_t items) {
  const int64_t b = (items + NB - 1) / NB;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 16));
}
}  // namespace

void launch_weights_corr(cudaStream_t s, int32_t F, const int32_t *owner, const int32_t *nbr,
                         const double *SfA, const double *CfA, const double *CA, const double *magSf,
                         const double *delta, double *w, double *corr, double *SfS) {
  if (F <= 0) return;
  k_weights_corr<<<grid_for(F), NB, 0, s>>>(F, owner, nbr, SfA, CfA, CA, magSf, delta, w, corr, SfS);
}

void launch_grad(cudaStream_t s, const Launch &L, const MeshDev &m, const GeomDev &g, const double *x,
                 const double *halo, double *gradS, double *gradA) {
  k_grad<<<L.grid, NB, 0, s>>>(m, g, x, halo, gradS, gradA);
}

void launch_grad_bc(cudaStream_t s, const MeshDev &m, const GeomDev &g, const int32_t *bCell,
                    const double *x, const double *gradS, double *bgradA) {
  if (g.B <= 0) return;
  k_grad_bc<<<grid_for(g.B), NB, 0, s>>>(m, g, bCell, x, gradS, bgradA);
}

void launch_face_gamma(cudaStream_t s, const MeshDev &m, const GeomDev &g, const int32_t *owner,
                       const int32_t *bCell, const double *DTc, const double *haloDT, double *gammaF,
                       double *gammaB) {
  if (g.F + g.B <= 0) return;
  k_face_gamma<<<grid_for((int64_t)g.F + g.B), NB, 0, s>>>(m, g, owner, bCell, DTc, haloDT, gammaF, gammaB);
}

void launch_lap_corr(cudaStream_t s, const Launch &L, const MeshDev &m, const GeomDev &g, double DT,
                     const double *gradS, const double *haloG, int32_t nproc, double *lapSrc) {
  k_lap_corr<<<L.grid, NB, 0, s>>>(m, g, DT, gradS, haloG, nproc, lapSrc);
}

}  // namespace lf
