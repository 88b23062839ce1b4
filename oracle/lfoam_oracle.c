/*
 * lfoam_oracle.c — CPU ORACLE for the laplacianFoam hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py (its cpu_baseline leg and --impl reference arm) may load this
 * library.  The product (paper_2507_18268_b200, liblfoam.so) never links,
 * loads or calls it, and shares no code, header or table with it.
 *
 * Plain C99, IEEE double, single-threaded, built with -O2 -ffp-contract=off
 * (no FMA contraction), loops in the order the definitions state them.
 *
 * What it computes (PAPER.md = P):
 *   - laplacianFoam step, P:233-261 (Listing 1): TEqn = fvm::ddt(T) -
 *     fvm::laplacian(DT,T) == fvOptions(T) (= 0, reading A2); TEqn.solve().
 *   - Euler ddt (reading A3): diag += rDeltaT*V, source += (rDeltaT*T0)*V.
 *   - Gauss laplacian, orthogonal two-point flux (reading A4):
 *     u_f = deltaCoeffs_f*(DT*magSf_f); upper = -u; negSumDiag.
 *   - boundary coefficients (reading A5; OpenFOAM fvMatrix addBoundaryDiag /
 *     addBoundarySource): fixedValue diag += a, source += (DT*magSf)*(delta*Tb);
 *     zeroGradient nothing; processor diag += a, interface coeff = a.
 *   - lduMatrix::Amul with processor interfaces (y -= bc*x_remote).
 *   - OpenFOAM PCG + diagonal preconditioner (§5.1, §6): L1
 *     residual / normFactor, strict '<' (reading A9), singularity 1e-300.
 *   - OpenFOAM DIC preconditioner, face-loop form over
 *     the upper-triangular face order (reading A39).
 *   - GAMG preconditioner: pairwise face
 *     agglomeration, Galerkin coarse LDU matrices, symmetric Jacobi V-cycle
 *     with an exact coarsest solve (reading A43).
 *   - CSR cell->face grouping (§5.2): the plain definition — a
 *     stable counting sort (items grouped by key, ties in input order,
 *     starts = exclusive scan of counts with the total appended, A13/A14).
 *
 * Parity pins for every function live in tests/test_oracle_*.py (closed
 * forms, SPEC worked examples, dense brute force, invariants).  The PCG
 * iteration count, normFactor and residuals after step 0 have no closed
 * form: "parity unpinned" beyond the pins listed in DESIGN.md §Parity.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_FIXED_VALUE 0
#define ORC_ZERO_GRADIENT 1
#define ORC_PROCESSOR 2

typedef struct {
    int32_t n_cells, n_faces, n_patches, n_bfaces;
    const int32_t *owner, *neighbour;      /* [n_faces] */
    const double *mag_sf, *delta, *V;      /* [n_faces], [n_faces], [n_cells] */
    const int32_t *patch_type;             /* [n_patches] */
    const int32_t *patch_start;            /* [n_patches+1] into the flat boundary arrays */
    const int32_t *b_cells;                /* [n_bfaces] faceCells */
    const double *b_mag_sf, *b_delta;      /* [n_bfaces] */
    /* full geometry (optional, NULL if absent): non-orthogonal correction */
    const double *Sf, *Cf;                 /* [n_faces][3] */
    const double *C;                       /* [n_cells][3] */
    const double *b_Sf;                    /* [n_bfaces][3] */
    /* spatially varying DT (optional, NULL = the scalar DT argument): the
     * face diffusivity gamma_f (linear interpolation of the cell field,
     * orc_face_gamma) and its boundary values */
    const double *gamma;                   /* [n_faces] */
    const double *b_gamma;                 /* [n_bfaces] */
} orc_mesh;

typedef struct {
    double initial_residual, final_residual;
    int32_t n_iterations, converged, singular, pad;
} orc_perf;

/* gsum: in-place global sum of k doubles over all ranks (NULL = one rank).
 * halo: x_remote[i] := value of x across processor boundary face i
 *       (flat boundary index; non-processor entries untouched). */
typedef void (*orc_gsum_fn)(void *ctx, double *vals, int32_t k);
typedef void (*orc_halo_fn)(void *ctx, const double *x, double *x_remote);

/* ------------------------------------------------------------------ CSR */
/* P:401-429 (§5.2, "List of List", "Sorting owner list", "Starting index"):
 * group face ids by key.  Definition: starts[g] = #keys < g (n_groups+1
 * entries, A14); items lists, for each group in ascending order, the input
 * positions with that key in input order (stable, A13). */
int orc_group(const int32_t *keys, int64_t m, int32_t n_groups,
              int32_t *items, int32_t *starts)
{
    int64_t i;
    int32_t g;
    int32_t *fill;
    for (g = 0; g <= n_groups; g++) starts[g] = 0;
    for (i = 0; i < m; i++) {
        if (keys[i] < 0 || keys[i] >= n_groups) return 1;
        starts[keys[i] + 1] += 1;
    }
    for (g = 0; g < n_groups; g++) starts[g + 1] += starts[g];
    fill = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n_groups > 0 ? n_groups : 1));
    if (!fill) return 2;
    for (g = 0; g < n_groups; g++) fill[g] = starts[g];
    for (i = 0; i < m; i++) items[fill[keys[i]]++] = (int32_t)i;
    free(fill);
    return 0;
}

/* ------------------------------------------------------------- assembly */
/* SURVEY §8(c.1) lines 1-4 (OpenFOAM EulerDdtScheme::fvmDdt,
 * gaussLaplacianScheme::fvmLaplacianUncorrected + negSumDiag, fvMatrix
 * operator-, addBoundaryDiag/addBoundarySource).
 *   b_int[i]  = internalCoeffs of boundary face i (a; 0 for zeroGradient)
 *   b_bnd[i]  = boundaryCoeffs of boundary face i ((DT*magSf)*(delta*Tb)
 *               for fixedValue, a for processor (interfaceBouCoeffs), 0 zeroGradient)
 */
int orc_assemble(const orc_mesh *m, double DT, double dt, const double *T0,
                 const double *b_value, double *diag, double *upper,
                 double *source, double *b_int, double *b_bnd)
{
    int32_t c, f, p, i;
    double rDeltaT = 1.0 / dt;
    double *L = (double *)calloc((size_t)(m->n_cells > 0 ? m->n_cells : 1), sizeof(double));
    if (!L) return 2;
    for (c = 0; c < m->n_cells; c++) {
        diag[c] = rDeltaT * m->V[c];                    /* D[c] */
        source[c] = (rDeltaT * T0[c]) * m->V[c];        /* S[c] */
    }
    for (f = 0; f < m->n_faces; f++) {                 /* file order */
        double g = m->gamma ? m->gamma[f] : DT;         /* gammaMagSf = gamma_f*magSf */
        double u = m->delta[f] * (g * m->mag_sf[f]);
        upper[f] = -u;
        L[m->owner[f]] -= u;
        L[m->neighbour[f]] -= u;
    }
    for (c = 0; c < m->n_cells; c++) diag[c] = diag[c] - L[c];
    free(L);
    for (p = 0; p < m->n_patches; p++) {
        int32_t t = m->patch_type[p];
        for (i = m->patch_start[p]; i < m->patch_start[p + 1]; i++) {
            int32_t cc = m->b_cells[i];
            double gms = (m->b_gamma ? m->b_gamma[i] : DT) * m->b_mag_sf[i];
            double a = gms * m->b_delta[i];
            if (t == ORC_FIXED_VALUE) {
                double bc = gms * (m->b_delta[i] * b_value[i]);
                diag[cc] += a;
                source[cc] += bc;
                b_int[i] = a;
                b_bnd[i] = bc;
            } else if (t == ORC_PROCESSOR) {
                diag[cc] += a;
                b_int[i] = a;
                b_bnd[i] = a;
            } else {
                b_int[i] = 0.0;
                b_bnd[i] = 0.0;
            }
        }
    }
    return 0;
}

/* ----------------------------------------------------------------- Amul */
/* lduMatrix::Amul (SURVEY §8(c.1) "Amul(x)"): y = diag*x; face loop in
 * file order; then processor interfaces y[c] -= bc*x_remote. */
void orc_amul(const orc_mesh *m, const double *diag, const double *upper,
              const double *b_bnd, const double *x, const double *x_remote,
              double *y)
{
    int32_t c, f, p, i;
    for (c = 0; c < m->n_cells; c++) y[c] = diag[c] * x[c];
    for (f = 0; f < m->n_faces; f++) {
        y[m->neighbour[f]] += upper[f] * x[m->owner[f]];
        y[m->owner[f]] += upper[f] * x[m->neighbour[f]];
    }
    for (p = 0; p < m->n_patches; p++) {
        if (m->patch_type[p] != ORC_PROCESSOR) continue;
        for (i = m->patch_start[p]; i < m->patch_start[p + 1]; i++)
            y[m->b_cells[i]] -= b_bnd[i] * x_remote[i];
    }
}

/* lduMatrix::sumA: row sums incl. interface boundary coeffs. */
void orc_sumA(const orc_mesh *m, const double *diag, const double *upper,
              const double *b_bnd, double *sumA)
{
    int32_t c, f, p, i;
    for (c = 0; c < m->n_cells; c++) sumA[c] = diag[c];
    for (f = 0; f < m->n_faces; f++) {
        sumA[m->neighbour[f]] += upper[f];
        sumA[m->owner[f]] += upper[f];
    }
    for (p = 0; p < m->n_patches; p++) {
        if (m->patch_type[p] != ORC_PROCESSOR) continue;
        for (i = m->patch_start[p]; i < m->patch_start[p + 1]; i++)
            sumA[m->b_cells[i]] -= b_bnd[i];
    }
}

static void gsum(orc_gsum_fn fn, void *ctx, double *v, int32_t k)
{
    if (fn) fn(ctx, v, k);
}

static void amul_halo(const orc_mesh *m, const double *diag, const double *upper,
                      const double *b_bnd, const double *x, double *xr, double *y,
                      orc_halo_fn halo, void *ctx)
{
    if (halo) halo(ctx, x, xr);
    orc_amul(m, diag, upper, b_bnd, x, xr, y);
}

static int converged(double res, double init, double tol, double rel_tol)
{
    return res < tol || (rel_tol > 0.0 && res < rel_tol * init);
}

/* ------------------------------------------------------------------ DIC */
/* DIC preconditioner ("DIC/DILU (the usual laplacianFoam
 * fvSolution choice [OF])"; OpenFOAM DICPreconditioner), in OpenFOAM's own
 * face-loop form.  lduAddressing keeps faces in upper-triangular order
 * (lower address l < upper address u, sorted by l then u); the loops below
 * run over that order (reading A39: the oracle sorts a copy of the faces,
 * so any input face order/orientation gives the OpenFOAM result).
 *   calcReciprocalD:  rD = diag; for f: rD[u] -= upper_f*upper_f/rD[l];
 *                     rD = 1/rD
 *   precondition:     wA = rD*rA;
 *                     for f ascending:  wA[u] -= rD[u]*upper_f*wA[l];
 *                     for f descending: wA[l] -= rD[l]*upper_f*wA[u]
 * i.e. wA = M^-1 rA with M = (D*+L) D*^-1 (D*+U), D* = 1/rD (incomplete
 * Cholesky with no fill: diag(M) = diag(A), M = A on A's pattern).
 * Processor interfaces do not enter (OpenFOAM's DIC is processor-local). */
typedef struct {
    int32_t l, u, f;
} orc_face3;

static int face3_cmp(const void *a, const void *b)
{
    const orc_face3 *x = (const orc_face3 *)a, *y = (const orc_face3 *)b;
    if (x->l != y->l) return x->l < y->l ? -1 : 1;
    if (x->u != y->u) return x->u < y->u ? -1 : 1;
    return x->f < y->f ? -1 : (x->f > y->f);
}

static orc_face3 *upper_triangular_faces(const orc_mesh *m)
{
    int32_t f, F = m->n_faces;
    orc_face3 *t = (orc_face3 *)malloc(sizeof(orc_face3) * (size_t)(F > 0 ? F : 1));
    if (!t) return NULL;
    for (f = 0; f < F; f++) {
        int32_t a = m->owner[f], b = m->neighbour[f];
        t[f].l = a < b ? a : b;
        t[f].u = a < b ? b : a;
        t[f].f = f;
    }
    qsort(t, (size_t)F, sizeof(orc_face3), face3_cmp);
    return t;
}

static void dic_rD(const orc_mesh *m, const orc_face3 *t, const double *diag,
                   const double *upper, double *rD)
{
    int32_t c, k;
    for (c = 0; c < m->n_cells; c++) rD[c] = diag[c];
    for (k = 0; k < m->n_faces; k++) {
        double a = upper[t[k].f];
        rD[t[k].u] -= a * a / rD[t[k].l];
    }
    for (c = 0; c < m->n_cells; c++) rD[c] = 1.0 / rD[c];
}

static void dic_precondition(const orc_mesh *m, const orc_face3 *t, const double *rD,
                             const double *upper, const double *rA, double *wA)
{
    int32_t c, k;
    for (c = 0; c < m->n_cells; c++) wA[c] = rD[c] * rA[c];
    for (k = 0; k < m->n_faces; k++)
        wA[t[k].u] -= rD[t[k].u] * upper[t[k].f] * wA[t[k].l];
    for (k = m->n_faces - 1; k >= 0; k--)
        wA[t[k].l] -= rD[t[k].l] * upper[t[k].f] * wA[t[k].u];
}

/* rD_out[n] (reciprocal DIC diagonal) and, if rA != NULL, wA = M^-1 rA. */
int orc_dic(const orc_mesh *m, const double *diag, const double *upper,
            const double *rA, double *rD_out, double *wA)
{
    orc_face3 *t = upper_triangular_faces(m);
    if (!t) return 2;
    dic_rD(m, t, diag, upper, rD_out);
    if (rA) dic_precondition(m, t, rD_out, upper, rA, wA);
    free(t);
    return 0;
}

/* ----------------------------------------------------------------- GAMG */
/* GAMG preconditioner ("GAMG/AmgX (the paper's
 * suggested alternative)"; §7 names an AMG preconditioner "a better
 * alternative").  The paper gives no algorithm; the reading (A43)
 * follows OpenFOAM's GAMG with pairwise face agglomeration:
 *   agglomeration (once per mesh, geometric weights w_f = magSf_f*delta_f):
 *     one PAIRING PASS over a graph (cells, faces (l,u,w) upper-triangular):
 *       for c in order (ascending; DESCENDING on odd passes), unassigned:
 *         j = the unassigned neighbour with the largest w (first in ascending
 *             neighbour label on ties); if any: c and j form a new aggregate;
 *         else j = the neighbour with the largest w: c joins j's aggregate;
 *         else (no neighbour) c is a singleton aggregate.
 *       aggregates are numbered in creation order; the coarse graph has one
 *       face per pair of adjacent aggregates (I < J, sorted), weight = sum of
 *       the fine weights in ascending fine-face order.
 *     a LEVEL = two pairing passes (OpenFOAM mergeLevels 2); levels are added
 *     while the current one has more than GAMG_NMIN cells and the new one has
 *     at most 90% of its cells (at most GAMG_MAXL levels).
 *   coarse matrices (per solve, Galerkin A_{l+1} = P^T A_l P with P the
 *     piecewise-constant aggregation): D_{l+1}[I] = sum over members c of I
 *     (ascending) of D_l[c], then over the faces internal to I (ascending)
 *     of (U_f + U_f); U_{l+1}[F] = sum of U_f over the faces of F (ascending).
 *   V-cycle (one per application, zero initial guess, symmetric: one Jacobi
 *     sweep x += omega*rD*(b - A x) before and after the coarse correction,
 *     omega = GAMG_OMEGA; the coarsest level solved exactly with the inverse
 *     from a Cholesky factorisation):
 *       b_0 = r
 *       l = 0..L-1:  x_l = omega*(rD_l*b_l);  b_{l+1} = P^T (b_l - A_l x_l)
 *       x_L = A_L^-1 b_L
 *       l = L-1..0:  z = x_l + P x_{l+1};  x_l = z + omega*(rD_l*(b_l - A_l z))
 *       M^-1 r = x_0
 *   A_l x uses the face loop of lduMatrix::Amul over the level's
 *   upper-triangular faces (a cell's terms in ascending neighbour label).
 * Single rank (no processor interfaces on the coarse levels). */
#define GAMG_NMIN 64
#define GAMG_MAXL 30
#define GAMG_OMEGA 0.9
#define GAMG_MAXCOARSEST 2048

typedef struct {
    int32_t n, nf;
    int32_t *l, *u;       /* [nf] faces, upper-triangular, sorted by (l, u) */
    double *w;            /* [nf] agglomeration weights */
    int32_t *agg;         /* [n] cell -> cell of the next level (not on the coarsest) */
    int32_t *cface;       /* [nf] face -> face of the next level, -1 inside an aggregate */
    double *D, *U, *rD;   /* per solve */
    double *x, *b, *y;    /* work */
} orc_glevel;

typedef struct {
    int32_t L;            /* index of the coarsest level (levels 0..L) */
    orc_glevel lv[GAMG_MAXL + 1];
    int32_t *fmap;        /* level-0 face k = mesh face fmap[k] */
    double *inv;          /* [nL*nL] inverse of the coarsest matrix (row major) */
} orc_gamg_t;

/* neighbours of every cell in ascending label: CSR over the faces */
static int graph_rows(int32_t n, int32_t nf, const int32_t *l, const int32_t *u, const double *w,
                      int32_t **start, int32_t **nb, double **wt)
{
    int32_t c, f, *cnt = (int32_t *)calloc((size_t)n + 1, sizeof(int32_t));
    if (!cnt) return 2;
    for (f = 0; f < nf; f++) { cnt[l[f] + 1]++; cnt[u[f] + 1]++; }
    for (c = 0; c < n; c++) cnt[c + 1] += cnt[c];
    *start = cnt;
    *nb = (int32_t *)malloc(sizeof(int32_t) * (size_t)(2 * nf + 1));
    *wt = (double *)malloc(sizeof(double) * (size_t)(2 * nf + 1));
    int32_t *pos = (int32_t *)malloc(sizeof(int32_t) * ((size_t)n + 1));
    if (!*nb || !*wt || !pos) return 2;
    memcpy(pos, cnt, sizeof(int32_t) * (size_t)n);
    /* faces sorted by (l, u): for cell c the faces (l', c) come in ascending
     * l' < c, then the faces (c, u') in ascending u' -> ascending labels
     * when both sides are appended in face order, lower side first */
    for (f = 0; f < nf; f++) { (*nb)[pos[u[f]]] = l[f]; (*wt)[pos[u[f]]++] = w[f]; }
    for (f = 0; f < nf; f++) { (*nb)[pos[l[f]]] = u[f]; (*wt)[pos[l[f]]++] = w[f]; }
    free(pos);
    return 0;
}

typedef struct { int32_t l, u, f; } orc_cf;
static int cf_cmp(const void *a, const void *b)
{
    const orc_cf *x = (const orc_cf *)a, *y = (const orc_cf *)b;
    if (x->l != y->l) return x->l < y->l ? -1 : 1;
    if (x->u != y->u) return x->u < y->u ? -1 : 1;
    return x->f < y->f ? -1 : (x->f > y->f);
}

/* one pairing pass on (n, nf, l, u, w): agg[n], *nc, and the coarse graph
 * (*cl, *cu, *cw, *ncf) with cface[nf] (-1 inside an aggregate) */
static int pair_pass(int32_t n, int32_t nf, const int32_t *l, const int32_t *u, const double *w,
                     int reverse, int32_t *agg, int32_t *nc, int32_t *cface,
                     int32_t **cl, int32_t **cu, double **cw, int32_t *ncf)
{
    int32_t *st, *nb, i, k, f, m = 0;
    double *wt;
    if (graph_rows(n, nf, l, u, w, &st, &nb, &wt)) return 2;
    for (i = 0; i < n; i++) agg[i] = -1;
    *nc = 0;
    for (i = 0; i < n; i++) {
        int32_t c = reverse ? n - 1 - i : i, best = -1;
        double bw = -1.0;
        if (agg[c] >= 0) continue;
        for (k = st[c]; k < st[c + 1]; k++)
            if (agg[nb[k]] < 0 && wt[k] > bw) { bw = wt[k]; best = nb[k]; }
        if (best >= 0) {
            agg[c] = agg[best] = (*nc)++;
        } else {
            bw = -1.0;
            for (k = st[c]; k < st[c + 1]; k++)
                if (wt[k] > bw) { bw = wt[k]; best = nb[k]; }
            agg[c] = best >= 0 ? agg[best] : (*nc)++;
        }
    }
    free(st); free(nb); free(wt);
    /* coarse faces: distinct (I, J), I < J, sorted; weights summed in fine order */
    orc_cf *t = (orc_cf *)malloc(sizeof(orc_cf) * (size_t)(nf > 0 ? nf : 1));
    if (!t) return 2;
    for (f = 0; f < nf; f++) {
        int32_t a = agg[l[f]], b = agg[u[f]];
        cface[f] = -1;
        if (a == b) continue;
        t[m].l = a < b ? a : b; t[m].u = a < b ? b : a; t[m].f = f; m++;
    }
    qsort(t, (size_t)m, sizeof(orc_cf), cf_cmp);
    *cl = (int32_t *)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
    *cu = (int32_t *)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
    *cw = (double *)calloc((size_t)(m > 0 ? m : 1), sizeof(double));
    if (!*cl || !*cu || !*cw) return 2;
    *ncf = 0;
    for (k = 0; k < m; k++) {
        if (k == 0 || t[k].l != t[k - 1].l || t[k].u != t[k - 1].u) {
            (*cl)[*ncf] = t[k].l; (*cu)[*ncf] = t[k].u; (*ncf)++;
        }
        cface[t[k].f] = *ncf - 1;
    }
    /* weights in ascending fine-face order (t is sorted by face within a pair) */
    for (f = 0; f < nf; f++)
        if (cface[f] >= 0) (*cw)[cface[f]] += w[f];
    free(t);
    return 0;
}

static void gamg_free(orc_gamg_t *g)
{
    int32_t i;
    for (i = 0; i <= g->L; i++) {
        orc_glevel *v = &g->lv[i];
        free(v->l); free(v->u); free(v->w); free(v->agg); free(v->cface);
        free(v->D); free(v->U); free(v->rD); free(v->x); free(v->b); free(v->y);
    }
    free(g->fmap); free(g->inv);
    memset(g, 0, sizeof(*g));
}

/* the level hierarchy of a mesh (agglomeration only) */
static int gamg_build(const orc_mesh *m, orc_gamg_t *g)
{
    int32_t f, k;
    memset(g, 0, sizeof(*g));
    orc_face3 *t = upper_triangular_faces(m);
    if (!t) return 2;
    orc_glevel *v = &g->lv[0];
    v->n = m->n_cells; v->nf = m->n_faces;
    size_t F1 = (size_t)(m->n_faces > 0 ? m->n_faces : 1);
    v->l = (int32_t *)malloc(sizeof(int32_t) * F1); v->u = (int32_t *)malloc(sizeof(int32_t) * F1);
    v->w = (double *)malloc(sizeof(double) * F1); g->fmap = (int32_t *)malloc(sizeof(int32_t) * F1);
    if (!v->l || !v->u || !v->w || !g->fmap) return 2;
    for (k = 0; k < m->n_faces; k++) {
        f = t[k].f;
        v->l[k] = t[k].l; v->u[k] = t[k].u; g->fmap[k] = f;
        v->w[k] = m->mag_sf[f] * m->delta[f];
    }
    free(t);
    int32_t pass = 0;
    while (g->L < GAMG_MAXL && g->lv[g->L].n > GAMG_NMIN) {
        orc_glevel *a = &g->lv[g->L];
        /* two pairing passes: a -> mid -> coarse */
        int32_t n1, nf1, n2, nf2, *l1, *u1, *l2, *u2;
        double *w1, *w2;
        int32_t *agg1 = (int32_t *)malloc(sizeof(int32_t) * (size_t)(a->n > 0 ? a->n : 1));
        int32_t *cf1 = (int32_t *)malloc(sizeof(int32_t) * (size_t)(a->nf > 0 ? a->nf : 1));
        if (!agg1 || !cf1) return 2;
        if (pair_pass(a->n, a->nf, a->l, a->u, a->w, pass & 1, agg1, &n1, cf1, &l1, &u1, &w1, &nf1)) return 2;
        int32_t *agg2 = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n1 > 0 ? n1 : 1));
        int32_t *cf2 = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nf1 > 0 ? nf1 : 1));
        if (!agg2 || !cf2) return 2;
        if (pair_pass(n1, nf1, l1, u1, w1, (pass + 1) & 1, agg2, &n2, cf2, &l2, &u2, &w2, &nf2)) return 2;
        pass += 2;
        free(l1); free(u1); free(w1);
        if ((double)n2 > 0.9 * (double)a->n) {  /* coarsening stalled: a is the coarsest */
            free(agg1); free(cf1); free(agg2); free(cf2); free(l2); free(u2); free(w2);
            break;
        }
        a->agg = agg1; a->cface = cf1;
        for (k = 0; k < a->n; k++) a->agg[k] = agg2[agg1[k]];
        for (f = 0; f < a->nf; f++) a->cface[f] = cf1[f] < 0 ? -1 : cf2[cf1[f]];
        free(agg2); free(cf2);
        orc_glevel *c = &g->lv[++g->L];
        c->n = n2; c->nf = nf2; c->l = l2; c->u = u2; c->w = w2;
    }
    if (g->lv[g->L].n > GAMG_MAXCOARSEST) return 3;
    for (k = 0; k <= g->L; k++) {
        orc_glevel *a = &g->lv[k];
        size_t nn = (size_t)(a->n > 0 ? a->n : 1), ff = (size_t)(a->nf > 0 ? a->nf : 1);
        a->D = (double *)calloc(nn, sizeof(double)); a->rD = (double *)calloc(nn, sizeof(double));
        a->U = (double *)calloc(ff, sizeof(double));
        a->x = (double *)calloc(nn, sizeof(double)); a->b = (double *)calloc(nn, sizeof(double));
        a->y = (double *)calloc(nn, sizeof(double));
        if (!a->D || !a->rD || !a->U || !a->x || !a->b || !a->y) return 2;
    }
    int32_t nL = g->lv[g->L].n;
    g->inv = (double *)calloc((size_t)nL * (size_t)nL + 1, sizeof(double));
    return g->inv ? 0 : 2;
}

/* y = A_l x, face loop (lduMatrix::Amul) */
static void glevel_amul(const orc_glevel *a, const double *x, double *y)
{
    int32_t c, f;
    for (c = 0; c < a->n; c++) y[c] = a->D[c] * x[c];
    for (f = 0; f < a->nf; f++) {
        y[a->u[f]] += a->U[f] * x[a->l[f]];
        y[a->l[f]] += a->U[f] * x[a->u[f]];
    }
}

/* coarse matrices of the current fine matrix and the coarsest inverse */
static int gamg_setup(orc_gamg_t *g, const double *diag, const double *upper)
{
    int32_t l, c, f, i, j, k;
    orc_glevel *a0 = &g->lv[0];
    for (c = 0; c < a0->n; c++) a0->D[c] = diag[c];
    for (f = 0; f < a0->nf; f++) a0->U[f] = upper[g->fmap[f]];
    for (l = 0; l < g->L; l++) {
        orc_glevel *a = &g->lv[l], *b = &g->lv[l + 1];
        for (c = 0; c < b->n; c++) b->D[c] = 0.0;
        for (f = 0; f < b->nf; f++) b->U[f] = 0.0;
        for (c = 0; c < a->n; c++) b->D[a->agg[c]] += a->D[c];
        for (f = 0; f < a->nf; f++)
            if (a->cface[f] < 0) b->D[a->agg[a->l[f]]] += a->U[f] + a->U[f];
        for (f = 0; f < a->nf; f++)
            if (a->cface[f] >= 0) b->U[a->cface[f]] += a->U[f];
    }
    for (l = 0; l <= g->L; l++)
        for (c = 0; c < g->lv[l].n; c++) g->lv[l].rD[c] = 1.0 / g->lv[l].D[c];
    /* coarsest: dense A, Cholesky (row by row), inverse column by column */
    orc_glevel *z = &g->lv[g->L];
    int32_t n = z->n;
    double *A = (double *)calloc((size_t)n * (size_t)n + 1, sizeof(double));
    double *Lm = (double *)calloc((size_t)n * (size_t)n + 1, sizeof(double));
    double *yv = (double *)calloc((size_t)n + 1, sizeof(double));
    if (!A || !Lm || !yv) return 2;
    for (c = 0; c < n; c++) A[c * n + c] = z->D[c];
    for (f = 0; f < z->nf; f++) { A[z->l[f] * n + z->u[f]] = z->U[f]; A[z->u[f] * n + z->l[f]] = z->U[f]; }
    for (i = 0; i < n; i++)
        for (j = 0; j <= i; j++) {
            double s = A[i * n + j];
            for (k = 0; k < j; k++) s -= Lm[i * n + k] * Lm[j * n + k];
            if (i == j) {
                if (!(s > 0.0)) { free(A); free(Lm); free(yv); return 4; }  /* not SPD */
                Lm[i * n + i] = sqrt(s);
            } else {
                Lm[i * n + j] = s / Lm[j * n + j];
            }
        }
    for (k = 0; k < n; k++) {  /* column k of the inverse: L L^T x = e_k */
        for (i = 0; i < n; i++) {
            double s = i == k ? 1.0 : 0.0;
            for (j = 0; j < i; j++) s -= Lm[i * n + j] * yv[j];
            yv[i] = s / Lm[i * n + i];
        }
        for (i = n - 1; i >= 0; i--) {
            double s = yv[i];
            for (j = i + 1; j < n; j++) s -= Lm[j * n + i] * g->inv[j * n + k];
            g->inv[i * n + k] = s / Lm[i * n + i];
        }
    }
    free(A); free(Lm); free(yv);
    return 0;
}

/* wA = M^-1 rA: one V-cycle */
static void gamg_precondition(orc_gamg_t *g, const double *rA, double *wA)
{
    int32_t l, c, k;
    orc_glevel *a0 = &g->lv[0];
    for (c = 0; c < a0->n; c++) a0->b[c] = rA[c];
    for (l = 0; l < g->L; l++) {
        orc_glevel *a = &g->lv[l], *b = &g->lv[l + 1];
        for (c = 0; c < a->n; c++) a->x[c] = GAMG_OMEGA * (a->rD[c] * a->b[c]);
        glevel_amul(a, a->x, a->y);
        for (c = 0; c < b->n; c++) b->b[c] = 0.0;
        for (c = 0; c < a->n; c++) b->b[a->agg[c]] += a->b[c] - a->y[c];
    }
    orc_glevel *z = &g->lv[g->L];
    for (c = 0; c < z->n; c++) {
        double s = 0.0;
        for (k = 0; k < z->n; k++) s += g->inv[c * z->n + k] * z->b[k];
        z->x[c] = s;
    }
    for (l = g->L - 1; l >= 0; l--) {
        orc_glevel *a = &g->lv[l], *b = &g->lv[l + 1];
        for (c = 0; c < a->n; c++) a->x[c] = a->x[c] + b->x[a->agg[c]];   /* z = x + P x_c */
        glevel_amul(a, a->x, a->y);
        for (c = 0; c < a->n; c++) a->x[c] = a->x[c] + GAMG_OMEGA * (a->rD[c] * (a->b[c] - a->y[c]));
    }
    for (c = 0; c < a0->n; c++) wA[c] = a0->x[c];
}

/* Test access: level sizes, agglomeration maps and coarse matrices of the
 * hierarchy for (diag, upper); and w = M^-1 r.  out_n[GAMG_MAXL+1] cell
 * counts, out_nf[...] face counts, returns L (>= 0) or -error.  If
 * agg_out != NULL it receives the level-0 -> level-1 ... maps concatenated
 * (sum of n_l for l < L); if r != NULL, w = M^-1 r. */
int orc_gamg(const orc_mesh *m, const double *diag, const double *upper, int32_t *out_n,
             int32_t *out_nf, int32_t *agg_out, const double *r, double *w)
{
    orc_gamg_t g;
    int32_t l, off = 0, rc = gamg_build(m, &g);
    if (rc) { gamg_free(&g); return -rc; }
    if (diag && (rc = gamg_setup(&g, diag, upper))) { gamg_free(&g); return -rc; }
    for (l = 0; l <= g.L; l++) {
        if (out_n) out_n[l] = g.lv[l].n;
        if (out_nf) out_nf[l] = g.lv[l].nf;
        if (agg_out && l < g.L) {
            memcpy(agg_out + off, g.lv[l].agg, sizeof(int32_t) * (size_t)g.lv[l].n);
            off += g.lv[l].n;
        }
    }
    if (r && w) gamg_precondition(&g, r, w);
    l = g.L;
    gamg_free(&g);
    return l;
}

/* coarse matrix of level lev (1..L): D[n_lev], U[nf_lev], faces l/u */
int orc_gamg_level(const orc_mesh *m, const double *diag, const double *upper, int32_t lev,
                   double *D, double *U, int32_t *fl, int32_t *fu)
{
    orc_gamg_t g;
    int32_t rc = gamg_build(m, &g);
    if (rc || lev < 0 || lev > g.L) { gamg_free(&g); return rc ? -rc : -1; }
    if ((rc = gamg_setup(&g, diag, upper))) { gamg_free(&g); return -rc; }
    orc_glevel *a = &g.lv[lev];
    memcpy(D, a->D, sizeof(double) * (size_t)a->n);
    memcpy(U, a->U, sizeof(double) * (size_t)a->nf);
    memcpy(fl, a->l, sizeof(int32_t) * (size_t)a->nf);
    memcpy(fu, a->u, sizeof(int32_t) * (size_t)a->nf);
    gamg_free(&g);
    return 0;
}

#define ORC_PRECOND_DIAGONAL 0
#define ORC_PRECOND_DIC 1
#define ORC_PRECOND_GAMG 3

/* ------------------------------------------------------------------ PCG */
/* OpenFOAM PCG::scalarSolve, SURVEY §8(c.1) "PCG" block, step by step in
 * its order; precond = ORC_PRECOND_DIAGONAL (diagonalPreconditioner, the
 * paper's choice P:608), ORC_PRECOND_GAMG (one V-cycle, above) or
 * ORC_PRECOND_DIC (DICPreconditioner, above; built
 * where OpenFOAM constructs the preconditioner, once per solve). */
int orc_pcg_p(const orc_mesh *m, const double *diag, const double *upper,
              const double *b_bnd, const double *source, double *psi,
              double tol, double rel_tol, int32_t max_iter, int32_t min_iter,
              int32_t precond,
              orc_gsum_fn gsum_fn, orc_halo_fn halo_fn, void *ctx, orc_perf *perf)
{
    orc_face3 *t = NULL;
    int32_t n = m->n_cells, c;
    size_t nn = (size_t)(n > 0 ? n : 1), nb = (size_t)(m->n_bfaces > 0 ? m->n_bfaces : 1);
    double *wA = (double *)calloc(nn, sizeof(double));
    double *rA = (double *)calloc(nn, sizeof(double));
    double *pA = (double *)calloc(nn, sizeof(double));
    double *rD = (double *)calloc(nn, sizeof(double));
    double *tmp = (double *)calloc(nn, sizeof(double));
    double *xr = (double *)calloc(nb, sizeof(double));
    double s[2], normFactor, psibar, wArA, wArAold, wApA, alpha, beta;
    int32_t it = 0;
    orc_gamg_t gamg;
    int have_gamg = 0;
    if (!wA || !rA || !pA || !rD || !tmp || !xr) return 2;

    memset(perf, 0, sizeof(*perf));
    /* wA = A psi ; rA = source - wA */
    amul_halo(m, diag, upper, b_bnd, psi, xr, wA, halo_fn, ctx);
    for (c = 0; c < n; c++) rA[c] = source[c] - wA[c];

    /* normFactor: psibar = gAverage(psi); tmp = sumA*psibar;
     * gSum(|wA - tmp| + |source - tmp|) + 1e-20 */
    s[0] = 0.0;
    for (c = 0; c < n; c++) s[0] += psi[c];
    s[1] = (double)n;
    gsum(gsum_fn, ctx, s, 2);
    psibar = s[1] > 0.0 ? s[0] / s[1] : 0.0;
    orc_sumA(m, diag, upper, b_bnd, tmp);
    for (c = 0; c < n; c++) tmp[c] *= psibar;
    s[0] = 0.0;
    for (c = 0; c < n; c++) s[0] += fabs(wA[c] - tmp[c]) + fabs(source[c] - tmp[c]);
    gsum(gsum_fn, ctx, s, 1);
    normFactor = s[0] + 1e-20;

    s[0] = 0.0;
    for (c = 0; c < n; c++) s[0] += fabs(rA[c]);
    gsum(gsum_fn, ctx, s, 1);
    perf->initial_residual = s[0] / normFactor;
    perf->final_residual = perf->initial_residual;

    if (min_iter > 0 || !converged(perf->final_residual, perf->initial_residual, tol, rel_tol)) {
        if (precond == ORC_PRECOND_DIC) {
            t = upper_triangular_faces(m);
            if (!t) return 2;
            dic_rD(m, t, diag, upper, rD);
        } else if (precond == ORC_PRECOND_GAMG) {
            int rc = gamg_build(m, &gamg);
            if (!rc) rc = gamg_setup(&gamg, diag, upper);
            if (rc) { gamg_free(&gamg); return rc; }
            have_gamg = 1;
        } else {
            for (c = 0; c < n; c++) rD[c] = 1.0 / diag[c];
        }
        wArA = 1e20; /* OpenFOAM solverPerformance::great_ */
        do {
            wArAold = wArA;
            if (precond == ORC_PRECOND_DIC)                           /* precondition */
                dic_precondition(m, t, rD, upper, rA, wA);
            else if (precond == ORC_PRECOND_GAMG)
                gamg_precondition(&gamg, rA, wA);
            else
                for (c = 0; c < n; c++) wA[c] = rD[c] * rA[c];
            s[0] = 0.0;
            for (c = 0; c < n; c++) s[0] += wA[c] * rA[c];
            gsum(gsum_fn, ctx, s, 1);
            wArA = s[0];
            if (it == 0) {
                for (c = 0; c < n; c++) pA[c] = wA[c];
            } else {
                beta = wArA / wArAold;
                for (c = 0; c < n; c++) pA[c] = wA[c] + beta * pA[c];
            }
            amul_halo(m, diag, upper, b_bnd, pA, xr, wA, halo_fn, ctx);
            s[0] = 0.0;
            for (c = 0; c < n; c++) s[0] += wA[c] * pA[c];
            gsum(gsum_fn, ctx, s, 1);
            wApA = s[0];
            if (fabs(wApA) / normFactor < 1e-300) {              /* checkSingularity */
                perf->singular = 1;
                break;
            }
            alpha = wArA / wApA;
            for (c = 0; c < n; c++) {
                psi[c] += alpha * pA[c];
                rA[c] -= alpha * wA[c];
            }
            s[0] = 0.0;
            for (c = 0; c < n; c++) s[0] += fabs(rA[c]);
            gsum(gsum_fn, ctx, s, 1);
            perf->final_residual = s[0] / normFactor;
        } while ((++it < max_iter &&
                  !converged(perf->final_residual, perf->initial_residual, tol, rel_tol)) ||
                 it < min_iter);
    }
    perf->n_iterations = it;
    perf->converged = converged(perf->final_residual, perf->initial_residual, tol, rel_tol);
    free(wA); free(rA); free(pA); free(rD); free(tmp); free(xr); free(t);
    if (have_gamg) gamg_free(&gamg);
    return 0;
}

int orc_pcg(const orc_mesh *m, const double *diag, const double *upper,
            const double *b_bnd, const double *source, double *psi,
            double tol, double rel_tol, int32_t max_iter, int32_t min_iter,
            orc_gsum_fn gsum_fn, orc_halo_fn halo_fn, void *ctx, orc_perf *perf)
{
    return orc_pcg_p(m, diag, upper, b_bnd, source, psi, tol, rel_tol, max_iter, min_iter,
                     ORC_PRECOND_DIAGONAL, gsum_fn, halo_fn, ctx, perf);
}

/* correctBoundaryConditions for the patch values (a6): zeroGradient
 * Tb = T[faceCells]; fixedValue unchanged. */
void orc_patch_values(const orc_mesh *m, const double *T, double *b_value)
{
    int32_t p, i;
    for (p = 0; p < m->n_patches; p++) {
        if (m->patch_type[p] != ORC_ZERO_GRADIENT) continue;
        for (i = m->patch_start[p]; i < m->patch_start[p + 1]; i++)
            b_value[i] = T[m->b_cells[i]];
    }
}

/* ------------------------------------------------------- laplacianFoam */
/* Listing 1: for each step: assemble TEqn from T0 = T, solve
 * with psi = T (initial guess = old T), correct boundary values. */
int orc_laplacian_foam_p(const orc_mesh *m, double DT, double dt, double *T,
                         double *b_value, int32_t n_steps, double tol,
                         double rel_tol, int32_t max_iter, int32_t min_iter,
                         int32_t precond, orc_gsum_fn gsum_fn, orc_halo_fn halo_fn,
                         void *ctx, orc_perf *perf)
{
    size_t nn = (size_t)(m->n_cells > 0 ? m->n_cells : 1);
    size_t nf = (size_t)(m->n_faces > 0 ? m->n_faces : 1);
    size_t nb = (size_t)(m->n_bfaces > 0 ? m->n_bfaces : 1);
    double *diag = (double *)malloc(nn * sizeof(double));
    double *source = (double *)malloc(nn * sizeof(double));
    double *upper = (double *)malloc(nf * sizeof(double));
    double *b_int = (double *)malloc(nb * sizeof(double));
    double *b_bnd = (double *)malloc(nb * sizeof(double));
    int32_t s;
    int rc = 0;
    if (!diag || !source || !upper || !b_int || !b_bnd) return 2;
    for (s = 0; s < n_steps && rc == 0; s++) {
        rc = orc_assemble(m, DT, dt, T, b_value, diag, upper, source, b_int, b_bnd);
        if (rc == 0)
            rc = orc_pcg_p(m, diag, upper, b_bnd, source, T, tol, rel_tol, max_iter,
                           min_iter, precond, gsum_fn, halo_fn, ctx, &perf[s]);
        orc_patch_values(m, T, b_value);
    }
    free(diag); free(source); free(upper); free(b_int); free(b_bnd);
    return rc;
}

int orc_laplacian_foam(const orc_mesh *m, double DT, double dt, double *T,
                       double *b_value, int32_t n_steps, double tol,
                       double rel_tol, int32_t max_iter, int32_t min_iter,
                       orc_gsum_fn gsum_fn, orc_halo_fn halo_fn, void *ctx,
                       orc_perf *perf)
{
    return orc_laplacian_foam_p(m, DT, dt, T, b_value, n_steps, tol, rel_tol, max_iter,
                                min_iter, ORC_PRECOND_DIAGONAL, gsum_fn, halo_fn, ctx, perf);
}

/* ================================================================ *
 * Non-orthogonal correction path: the gradient *
 * kernels the paper ported (§5.2) and the corrected Gauss laplacian. *
 * ================================================================ */
#define ORC_ROOTVSMALL 1e-150

/* weights, Listing "weights parallel loop": the owner weight
 * lambda = SfdNei / (SfdOwn + SfdNei), 0.5 if the sum is below ROOTVSMALL. */
void orc_weights(const orc_mesh *m, double *w)
{
    int32_t f, k;
    for (f = 0; f < m->n_faces; f++) {
        const double *s = m->Sf + 3 * f, *cf = m->Cf + 3 * f;
        const double *cp = m->C + 3 * m->owner[f], *cn = m->C + 3 * m->neighbour[f];
        double so = 0.0, sn = 0.0;
        for (k = 0; k < 3; k++) {
            so += s[k] * (cf[k] - cp[k]);
            sn += s[k] * (cn[k] - cf[k]);
        }
        so = fabs(so);
        sn = fabs(sn);
        w[f] = fabs(so + sn) > ORC_ROOTVSMALL ? sn / (so + sn) : 0.5;
    }
}

/* surfaceInterpolation::nonOrthCorrectionVectors: n - d * deltaCoeffs with
 * n = Sf/|Sf| and d = C_N - C_P (deltaCoeffs = the mesh's nonOrthDeltaCoeffs). */
void orc_corr_vectors(const orc_mesh *m, double *corr)
{
    int32_t f, k;
    for (f = 0; f < m->n_faces; f++) {
        const double *cp = m->C + 3 * m->owner[f], *cn = m->C + 3 * m->neighbour[f];
        for (k = 0; k < 3; k++) {
            double nk = m->Sf[3 * f + k] / m->mag_sf[f];
            double dk = cn[k] - cp[k];
            corr[3 * f + k] = nk - dk * m->delta[f];
        }
    }
}

/* Boundary value of x on boundary face i (the patch field after evaluate):
 * fixedValue T_b, zeroGradient x[faceCell]. */
static double orc_patch_value(const orc_mesh *m, int32_t p, int32_t i, const double *x, const double *b_value)
{
    return m->patch_type[p] == ORC_FIXED_VALUE ? b_value[i] : x[m->b_cells[i]];
}

/* gaussGrad::gradf with linear interpolation, as the SERIAL scatter loops the
 * paper starts from: Listing "First cycle in the gradf routine" (P:375-382:
 * igGrad[owner] += Sf*ssf, igGrad[neighbour] -= Sf*ssf), Listing "Second cycle
 * gradient" (igGrad[faceCells] += pSf*pssf) and "Field division"
 * (igGrad /= V).  ssf = lambda*(x_P - x_N) + x_N (Listing
 * "dotInterpolate loop" form). */
void orc_grad(const orc_mesh *m, const double *w, const double *x, const double *b_value, double *grad)
{
    int32_t c, f, p, i, k;
    for (c = 0; c < 3 * m->n_cells; c++) grad[c] = 0.0;
    for (f = 0; f < m->n_faces; f++) {
        const int32_t P = m->owner[f], N = m->neighbour[f];
        const double ssf = w[f] * (x[P] - x[N]) + x[N];
        for (k = 0; k < 3; k++) {
            const double sfssf = m->Sf[3 * f + k] * ssf;
            grad[3 * P + k] += sfssf;
            grad[3 * N + k] -= sfssf;
        }
    }
    for (p = 0; p < m->n_patches; p++)
        for (i = m->patch_start[p]; i < m->patch_start[p + 1]; i++) {
            const double pssf = orc_patch_value(m, p, i, x, b_value);
            for (k = 0; k < 3; k++) grad[3 * m->b_cells[i] + k] += m->b_Sf[3 * i + k] * pssf;
        }
    for (c = 0; c < m->n_cells; c++)
        for (k = 0; k < 3; k++) grad[3 * c + k] /= m->V[c];
}

/* correctBoundaryConditions of the gradient (Listing "CorrectBoundaryConditions",
 * P:539-556): gb = grad[faceCell] (extrapolated), then on non-coupled patches
 * gb += n*(snGrad - n.gb) with snGrad = deltaCoeffs*(T_b - T_c) (fixedValue),
 * 0 (zeroGradient). */
void orc_grad_bc(const orc_mesh *m, const double *x, const double *b_value, const double *grad, double *bgrad)
{
    int32_t p, i, k;
    for (p = 0; p < m->n_patches; p++)
        for (i = m->patch_start[p]; i < m->patch_start[p + 1]; i++) {
            const int32_t c = m->b_cells[i];
            double n[3], ng = 0.0, sng;
            for (k = 0; k < 3; k++) {
                bgrad[3 * i + k] = grad[3 * c + k];
                n[k] = m->b_Sf[3 * i + k] / m->b_mag_sf[i];
            }
            if (m->patch_type[p] == ORC_PROCESSOR) continue;  /* coupled: untouched */
            for (k = 0; k < 3; k++) ng += n[k] * bgrad[3 * i + k];
            sng = m->patch_type[p] == ORC_FIXED_VALUE ? m->b_delta[i] * (b_value[i] - x[c]) : 0.0;
            for (k = 0; k < 3; k++) bgrad[3 * i + k] += n[k] * (sng - ng);
        }
}

/* Explicit non-orthogonal part of the corrected Gauss laplacian
 * (gaussLaplacianScheme::fvmLaplacian): fvm.source() -= V*fvc::div(gammaMagSf *
 * (corrVecs & interpolate(grad T))).  Returns that source contribution
 * lapSrc[c] = -(V * div)[c]; boundary corrections are zero (non-coupled). */
void orc_lap_correction(const orc_mesh *m, double DT, const double *w, const double *corr,
                        const double *grad, double *lapSrc)
{
    int32_t c, f, k;
    for (c = 0; c < m->n_cells; c++) lapSrc[c] = 0.0;
    for (f = 0; f < m->n_faces; f++) {
        const int32_t P = m->owner[f], N = m->neighbour[f];
        double cs = 0.0, flux;
        for (k = 0; k < 3; k++) {  /* dotInterpolate(corr, grad) */
            const double gf = w[f] * (grad[3 * P + k] - grad[3 * N + k]) + grad[3 * N + k];
            cs += corr[3 * f + k] * gf;
        }
        flux = ((m->gamma ? m->gamma[f] : DT) * m->mag_sf[f]) * cs;
        lapSrc[P] += flux;   /* surfaceIntegrate: owner +, neighbour - */
        lapSrc[N] -= flux;
    }
    for (c = 0; c < m->n_cells; c++) lapSrc[c] = -(m->V[c] * (lapSrc[c] / m->V[c]));
}

/* Listing 1 with the non-orthogonal corrector loop: every step keeps
 * T0 (old time) for ddt, and runs n_corr + 1 passes, each assembling with
 * the explicit correction of the CURRENT T and solving from it.
 * perf: [n_steps * (n_corr + 1)]. */
int orc_laplacian_foam_corrected_p(const orc_mesh *m, double DT, double dt, double *T,
                                   double *b_value, int32_t n_steps, int32_t n_corr, double tol,
                                   double rel_tol, int32_t max_iter, int32_t min_iter,
                                   int32_t precond, orc_perf *perf)
{
    size_t nn = (size_t)(m->n_cells > 0 ? m->n_cells : 1);
    size_t nf = (size_t)(m->n_faces > 0 ? m->n_faces : 1);
    size_t nb = (size_t)(m->n_bfaces > 0 ? m->n_bfaces : 1);
    double *diag = (double *)malloc(nn * sizeof(double)), *source = (double *)malloc(nn * sizeof(double));
    double *upper = (double *)malloc(nf * sizeof(double)), *w = (double *)malloc(nf * sizeof(double));
    double *corr = (double *)malloc(3 * nf * sizeof(double)), *grad = (double *)malloc(3 * nn * sizeof(double));
    double *lapSrc = (double *)malloc(nn * sizeof(double)), *T0 = (double *)malloc(nn * sizeof(double));
    double *b_int = (double *)malloc(nb * sizeof(double)), *b_bnd = (double *)malloc(nb * sizeof(double));
    int32_t s, k, c;
    int rc = 0;
    if (!diag || !source || !upper || !w || !corr || !grad || !lapSrc || !T0 || !b_int || !b_bnd) return 2;
    orc_weights(m, w);
    orc_corr_vectors(m, corr);
    for (s = 0; s < n_steps && rc == 0; s++) {
        for (c = 0; c < m->n_cells; c++) T0[c] = T[c];
        for (k = 0; k <= n_corr && rc == 0; k++) {
            orc_patch_values(m, T, b_value);
            orc_grad(m, w, T, b_value, grad);
            orc_lap_correction(m, DT, w, corr, grad, lapSrc);
            rc = orc_assemble(m, DT, dt, T0, b_value, diag, upper, source, b_int, b_bnd);
            /* TEqn = ddt - laplacian: source -= lapSrc, before the boundary
             * source (added in solveSegregated): rebuild in that order */
            if (rc == 0) {
                double rDeltaT = 1.0 / dt;
                int32_t p, i;
                for (c = 0; c < m->n_cells; c++) source[c] = (rDeltaT * T0[c]) * m->V[c] - lapSrc[c];
                for (p = 0; p < m->n_patches; p++)
                    if (m->patch_type[p] == ORC_FIXED_VALUE)
                        for (i = m->patch_start[p]; i < m->patch_start[p + 1]; i++)
                            source[m->b_cells[i]] += b_bnd[i];
                rc = orc_pcg_p(m, diag, upper, b_bnd, source, T, tol, rel_tol, max_iter, min_iter,
                               precond, NULL, NULL, NULL, &perf[s * (n_corr + 1) + k]);
            }
        }
        orc_patch_values(m, T, b_value);
    }
    free(diag); free(source); free(upper); free(w); free(corr); free(grad); free(lapSrc); free(T0);
    free(b_int); free(b_bnd);
    return rc;
}

int orc_laplacian_foam_corrected(const orc_mesh *m, double DT, double dt, double *T,
                                 double *b_value, int32_t n_steps, int32_t n_corr, double tol,
                                 double rel_tol, int32_t max_iter, int32_t min_iter, orc_perf *perf)
{
    return orc_laplacian_foam_corrected_p(m, DT, dt, T, b_value, n_steps, n_corr, tol, rel_tol,
                                          max_iter, min_iter, ORC_PRECOND_DIAGONAL, perf);
}

/* Spatially varying DT: the laplacian's face
 * diffusivity is the linear interpolate of the cell field,
 * gamma_f = lambda*(DT_P - DT_N) + DT_N (Listing "dotInterpolate loop" form,
 * P:293-299, with the weights of P:321-334); on boundary faces the field's
 * patch value, DT[faceCell] (zeroGradient DT, reading A38). */
void orc_face_gamma(const orc_mesh *m, const double *w, const double *DTc, double *gamma, double *b_gamma)
{
    int32_t f, i;
    for (f = 0; f < m->n_faces; f++)
        gamma[f] = w[f] * (DTc[m->owner[f]] - DTc[m->neighbour[f]]) + DTc[m->neighbour[f]];
    for (i = 0; i < m->n_bfaces; i++) b_gamma[i] = DTc[m->b_cells[i]];
}
