// Hot-path CUDA kernels for sm_100a (B200).
//
// All kernels are memory-bound FP64 work (Amul ~0.18 flop/B
// against a ~5 flop/B FP64 ridge) — no tensor cores.  One thread per cell,
// grid-stride over a RESIDENT grid (numSMs x blocks/SM), so every SM sweeps
// the cell range in lock-step and the neighbour-side re-reads (N^2 cells
// behind on a cube) hit in the 126 MB L2.
//
// Two row layouts for the off-diagonal gather:
//  * CSR (the paper's atomic-free lists, §5.2): ownerStart/nbr for
//    the owner side, losortStart/losort/losortOwner for the neighbour side.
//    Used by the assembly and as the general fallback.
//  * ELL slices derived from the CSR lists at mesh_create (DESIGN.md "Data
//    layout"): slot k of cell c at k*n + c (coalesced, no start offsets):
//      upperE[k*n+c]  coefficient of c's k-th owned face (0 if none)
//      nbrE[k*n+c]    its neighbour cell (-1 if none)
//      loE[k*n+c]     c's k-th neighbour-side face (losort order) as the
//                     packed owner-slot (kk<<29 | owner): its coefficient is
//                     upperE[kk*n + owner] (an L2 re-read), -1 if none.
//    This reads exactly the algorithmic 16 B/face (coefficient + 2 labels)
//    instead of the CSR's 28 B/face + 8 B/cell, with dependency depth 2
//    (index -> value) instead of 3 (start -> index -> value).
//
// Determinism: no float atomics anywhere.  Reductions are fixed-order
// (grid-stride partial per thread -> xor-shuffle tree -> per-block partial
// -> the last block, chosen by an integer ticket, sums the block partials in
// block order).  Same grid => bitwise-identical results run to run.
#include <cub/device/device_radix_sort.cuh>

#include "lfoam_internal.h"

namespace lf {

// ---- tuning knobs (defaults = the shipped configuration; variants are built
// with -D for measurements, see scripts/variants.py and profiles/)
#ifndef LF_BS
#define LF_BS 512        // threads per block (r1u sweep: 512 beats 256 by 2.4% at 100^3, 1.6% at
#endif                   // 200^3 in the persistent solve — fewer arrivals per grid barrier)
#ifndef LF_MINB
#define LF_MINB 2        // __launch_bounds__ min blocks/SM (register cap 65536/(BS*MINB))
#endif
#ifndef LF_MINB_G
#define LF_MINB_G 2      // same, for the row-gather kernels (phase 1, Amul, PCG setup)
#endif
#ifndef LF_P2_UNROLL
#define LF_P2_UNROLL 4   // cells per thread per grid-stride trip in phase 2
#endif
#ifndef LF_NO_ELL
#define LF_NO_ELL 0      // 1: force the CSR gather (ablation)
#endif
#ifndef LF_UNI
#define LF_UNI 0         // 1: ELL gathers take the labels of uniform 32-cell groups from one
#endif                   // descriptor per (slot, group) (MeshDev.uniE, k_build_uni)

constexpr int BS = LF_BS;
constexpr unsigned FULL = 0xffffffffu;
enum { T_SUM = 0, T_ASM = 1, T_SETUP = 2, T_P1 = 3, T_P2 = 4, T_P1I = 5, T_DYN = 8 };
constexpr int ELL_SHIFT = 29;  // slot kk <= 3 in bits 29-30: the packed label stays >= 0
constexpr int ELL_MASK = (1 << ELL_SHIFT) - 1;

int kernel_block_size() { return BS; }

// ------------------------------------------------------------ reductions
template <int NV>
__device__ __forceinline__ void warp_sum(double (&v)[NV]) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] += __shfl_xor_sync(FULL, v[k], o);
}

template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double (*sm)[32]) {
  warp_sum<NV>(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) sm[k][wid] = v[k];
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = lane < nw ? sm[k][lane] : 0.0;
    warp_sum<NV>(v);
  }
}

// ------------------------------------------------ peer-memory allreduce
// Executed by every thread of ONE block per rank (the last block of a
// launch / grid barrier).  Rank r stores its NV local totals into slot r of
// every rank's mailbox (P2P stores over NVLink, or plain stores when the
// mailbox is on the same GPU), publishes them with a system-scope release
// of the slot flag = seq, waits until all P slots of its own mailbox carry
// seq, and sums the P slots in rank order: bit-identical on every rank.
// Mailboxes are double-buffered by seq parity (a rank can be at most one
// allreduce ahead of any other).
__device__ __forceinline__ void st_release_sys(unsigned *p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed_sys_u32(const unsigned *p) {
  unsigned v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Spin-waits poll with RELAXED loads and acquire once after the flag moved
// (LF_SPIN_RELAXED): an ld.acquire compiles to LDG.STRONG + CCTL.IVALL, so
// polling with it invalidates the SM's L1 on every poll — under the block
// that is still computing on the same SM (its neighbour gathers then miss
// L1).  ncu r6c, 200^3: 39M polls per solve at the alpha barrier, 23% of the
// warp samples waiting there.
#ifndef LF_SPIN_RELAXED
#define LF_SPIN_RELAXED 1
#endif
__device__ __forceinline__ double ld_relaxed_sys(const double *p) {
  double v;
  asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}

// Blocks that stored halo values into peer memory (push_halo) note it here;
// only they issue the system-scope fence before arriving at a reduction.
__shared__ int lf_blockPushed;  // per block; may start as garbage (then one extra fence)
// thread 0, after the block's bar.sync: make this block's peer stores
// visible system-wide if it made any (and reset the note)
#ifndef LF_PUSH_FENCE
#define LF_PUSH_FENCE 1  // 0: no per-block system fence; the peer stores are ordered by the
#endif                   // block's gpu-scope release at arrival and the last block's system-
                         // scope fence + release.sys flag store in p2p_allreduce (cumulativity)
__device__ __forceinline__ void fence_pushed() {
  if (LF_PUSH_FENCE && lf_blockPushed) {
    __threadfence_system();
    lf_blockPushed = 0;
  }
}

// Spin-wait watchdog: a rank that never arrives must not hang the GPU —
// after LF_SPIN_TIMEOUT_S seconds the kernel traps (the call returns
// LF_ERR_CUDA) instead of spinning forever.
#ifndef LF_SPIN_TIMEOUT_S
#define LF_SPIN_TIMEOUT_S 30
#endif
__device__ __forceinline__ unsigned long long gtime_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void spin_check(unsigned long long t0, unsigned &tries) {
  if ((++tries & 1023u) == 0u && gtime_ns() - t0 > (unsigned long long)LF_SPIN_TIMEOUT_S * 1000000000ull)
    __trap();
}

template <int NV>
__device__ void p2p_allreduce(const P2PDev &P, double (&tot)[NV] /* valid in thread 0 */) {
  __shared__ double sv[NV];
  __shared__ unsigned sseq;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) sv[k] = tot[k];
    sseq = *P.seq + 1u;
    *P.seq = sseq;
  }
  __syncthreads();
  const unsigned seq = sseq, par = seq & 1u;
  const int q = threadIdx.x;
  if (q < P.P) {
    double *dst = P.vals[q] + ((int)par * LF_MAXP + P.rank) * 4;
#pragma unroll
    for (int k = 0; k < NV; ++k) dst[k] = sv[k];
    __threadfence_system();
    st_release_sys(P.flags[q] + par * LF_MAXP + P.rank, seq);
    const unsigned *mine = P.flags[P.rank] + par * LF_MAXP + q;
    const unsigned long long t0 = gtime_ns();
    unsigned tries = 0;
    while ((int)((LF_SPIN_RELAXED ? ld_relaxed_sys_u32(mine) : ld_acquire_sys(mine)) - seq) < 0) {
      __nanosleep(64);
      spin_check(t0, tries);
    }
    if (LF_SPIN_RELAXED) (void)ld_acquire_sys(mine);  // synchronises with the peers' releases
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double *box = P.vals[P.rank] + (int)par * LF_MAXP * 4;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = 0.0;
      for (int r = 0; r < P.P; ++r) s += ld_relaxed_sys(box + r * 4 + k);
      tot[k] = s;
    }
  }
}

// Block partial -> partials[k*grid + block]; the last block (ticket) sums
// the partials in block order (and, with the peer-memory transport, over
// the ranks) and writes out[0..NV).  Returns true in every thread of the
// last block; its thread 0 then holds the totals in v.
template <int NV>
__device__ bool reduce_grid(double (&v)[NV], double *partials, unsigned *ticket, double *out,
                            const P2PDev &P) {
  __shared__ double sm[NV][32];
  __shared__ int amLast;
  block_sum<NV>(v, sm);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) partials[k * gridDim.x + blockIdx.x] = v[k];
    if (P.P > 0) fence_pushed();  // this block's peer-memory halo stores precede the ticket
    __threadfence();
    const unsigned t = atomicAdd(ticket, 1u);
    amLast = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!amLast) return false;
  __threadfence();
  double s[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) s[k] = 0.0;
  // all partial loads of a trip in flight at once (one L2 round trip for
  // grids up to 4*blockDim); summation order per thread: b, b+BS, b+2BS, ...
  constexpr int U = 4;
  for (int b0 = threadIdx.x; b0 < (int)gridDim.x; b0 += blockDim.x * U) {
    double t[U][NV];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int b = b0 + u * blockDim.x;
#pragma unroll
      for (int k = 0; k < NV; ++k) t[u][k] = b < (int)gridDim.x ? __ldcg(&partials[k * gridDim.x + b]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < NV; ++k) s[k] += t[u][k];
  }
  block_sum<NV>(s, sm);
  if (P.P > 0) p2p_allreduce<NV>(P, s);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      out[k] = s[k];
      v[k] = s[k];
    }
    *ticket = 0u;
  }
  return true;
}

// ------------------------------------------------------------ row gathers
// Off-diagonal part of row c: the neighbour side (faces whose neighbour is
// c, in losort order) then the owner side (faces owned by c) — for
// upper-triangular face order exactly the face-loop order of
// lduMatrix::Amul.  Returns acc + sum upper_f x_other(f);
// sU (optional) receives sum upper_f (row sum for sumA).
// KE > 0: half ELL slices with KE slots per side; KE < 0: full-row ELL with
// -KE slots (the DIC rows; meshes with more than 4 faces on a side), each
// row in ascending neighbour label = the same summation order; KE == 0: CSR.
template <int KE, class XF, bool E16 = false>
__device__ __forceinline__ double row_offdiag(const MeshDev &m, const LduDev &a, int c, double acc,
                                              XF xval, double *sU = nullptr) {
  if constexpr (KE < 0) {
    constexpr int KS = -KE;
    int lab[KS];
    double u[KS], x[KS];
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      lab[k] = __ldg(m.symN + k * m.ldS + c);
      u[k] = __ldg(a.symU + k * m.ldS + c);
    }
#pragma unroll
    for (int k = 0; k < KS; ++k) x[k] = lab[k] >= 0 ? xval(lab[k] & (DIC_L0BIT - 1)) : 0.0;
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < KS; ++k)
      if (lab[k] >= 0) {
        acc = fma(u[k], x[k], acc);
        s += u[k];
      }
    if (sU) *sU = s;
    return acc;
  } else if constexpr (KE > 0) {
    const int n = m.ldE;  // slab stride
    int lo[KE], nb[KE];
    double uo[KE];
    if constexpr (E16) {  // compressed labels (see k_build_ell16), decoded to the same values
      const int g = c >> 5;
#pragma unroll
      for (int k = 0; k < KE; ++k) {
        const unsigned cw = __ldg(m.codeE + k * n + c);
        const int2 o = __ldg(m.offE + k * m.ngE + g);
        const unsigned nd = cw & 0xFFFFu, ldv = cw >> 16;
        nb[k] = nd == 0xFFFFu ? -1 : nd == 0xFFFEu ? __ldg(m.nbrE + k * n + c) : c + o.x + (int)nd - 0x8000;
        lo[k] = ldv == 0xFFFFu ? -1
                : ldv == 0xFFFEu ? __ldg(m.loE + k * n + c)
                                 : (int)((ldv >> 14) << ELL_SHIFT) | (c - o.y - (int)(ldv & 0x3FFFu) + 0x2000);
        uo[k] = a.upperE[k * n + c];
      }
    } else if (LF_UNI && m.uniE) {
      // uniform groups: the labels follow from one broadcast descriptor per
      // slot (no per-cell label bytes); other groups read them
      const int g = c >> 5;
#pragma unroll
      for (int k = 0; k < KE; ++k) {
        const int2 u = __ldg(m.uniE + k * m.ngE + g);
        nb[k] = u.x > 0 ? c + u.x : (u.x == 0 ? -1 : __ldg(m.nbrE + k * n + c));
        lo[k] = u.y > 0 ? ((u.y & ~ELL_MASK) | (c - (u.y & ELL_MASK))) : (u.y == 0 ? -1 : __ldg(m.loE + k * n + c));
        uo[k] = a.upperE[k * n + c];
      }
    } else {
#pragma unroll
      for (int k = 0; k < KE; ++k) {
        lo[k] = __ldg(m.loE + k * n + c);
        nb[k] = __ldg(m.nbrE + k * n + c);
        uo[k] = a.upperE[k * n + c];
      }
    }
    double lu[KE], lx[KE], ox[KE];
#pragma unroll
    for (int k = 0; k < KE; ++k) {
      const int oc = lo[k] & ELL_MASK;
      lu[k] = lo[k] >= 0 ? a.upperE[(lo[k] >> ELL_SHIFT) * n + oc] : 0.0;
      lx[k] = lo[k] >= 0 ? xval(oc) : 0.0;
      ox[k] = nb[k] >= 0 ? xval(nb[k]) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < KE; ++k)
      if (lo[k] >= 0) acc = fma(lu[k], lx[k], acc);
#pragma unroll
    for (int k = 0; k < KE; ++k)
      if (nb[k] >= 0) acc = fma(uo[k], ox[k], acc);
    if (sU) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < KE; ++k) s += lu[k];
#pragma unroll
      for (int k = 0; k < KE; ++k) s += uo[k];
      *sU = s;
    }
    return acc;
  } else {
    const int l0 = m.losortStart[c], l1 = m.losortStart[c + 1];
    const int o0 = m.ownerStart[c], o1 = m.ownerStart[c + 1];
    double s = 0.0;
    for (int j = l0; j < l1; ++j) {
      const double u = a.upper[m.losort[j]];
      acc = fma(u, xval(m.losortOwner[j]), acc);
      s += u;
    }
    for (int i = o0; i < o1; ++i) {
      const double u = a.upper[i];
      acc = fma(u, xval(m.nbr[i]), acc);
      s += u;
    }
    if (sU) *sU = s;
    return acc;
  }
}

__device__ __forceinline__ bool has_proc(const MeshDev &m, int c) {
  return m.hasProc && ((__ldg(m.procMask + (c >> 5)) >> (c & 31)) & 1u);
}

// Processor-interface term  sum_i bc_i * x_remote_i  (subtracted by callers);
// sBc (optional) receives sum_i bc_i.
__device__ __forceinline__ double row_proc(const MeshDev &m, const double *__restrict__ bBnd,
                                           const double *__restrict__ halo, int c,
                                           double *sBc = nullptr) {
  double s = 0.0, sb = 0.0;
  if (has_proc(m, c)) {
    const int k0 = m.pcStart[c], k1 = m.pcStart[c + 1];
    for (int k = k0; k < k1; ++k) {
      const int i = m.pcFace[k];
      s = fma(bBnd[i], halo[m.bSlot[i]], s);
      sb += bBnd[i];
    }
  }
  if (sBc) *sBc = sb;
  return s;
}

// PCG interface term with halo p recomputed locally from the neighbour's w:
// p_halo = w_halo (first iteration) or fma(beta, p_halo_old, w_halo) — the
// same operands and operation the owning rank uses for that cell, so both
// ranks hold bitwise the same p.  The new halo p is kept for the next
// iteration (written by the thread that owns the face's cell).
__device__ __forceinline__ double row_proc_p(const MeshDev &m, const double *__restrict__ bBnd,
                                             const Workspace &ws, bool first, double beta, int k,
                                             int c, int flag = -1 /* has_proc(m, c) if known */) {
  double s = 0.0;
  if (flag < 0 ? has_proc(m, c) : flag != 0) {
    const double *phOld = (k & 1) ? ws.pH[0] : ws.pH[1];
    double *phNew = (k & 1) ? ws.pH[1] : ws.pH[0];
    const int k0 = m.pcStart[c], k1 = m.pcStart[c + 1];
    for (int kk = k0; kk < k1; ++kk) {
      const int i = m.pcFace[kk], sl = m.bSlot[i];
      const double wh = ws.recvW[sl];
      const double ph = first ? wh : fma(beta, phOld[sl], wh);
      phNew[sl] = ph;
      s = fma(bBnd[i], ph, s);
    }
  }
  return s;
}

// Peer-memory halo: store a cell's new value into the neighbour's halo slot
// of each of its processor faces (remote store over NVLink; own buffer for
// self pairs): segment base + offset.  The block notes that it pushed
// (lf_blockPushed); only such blocks issue the system-scope fence before
// their arrival at the next reduction.
enum { HALO_W = 0, HALO_T = 1 };
template <int WHICH>
__device__ __forceinline__ void push_halo(const MeshDev &m, const P2PDev &P, int c, double val, int flag = -1) {
  if (flag < 0 ? has_proc(m, c) : flag != 0) {
    const int k0 = m.pcStart[c], k1 = m.pcStart[c + 1];
    for (int kk = k0; kk < k1; ++kk) {
      const int sl = m.bSlot[m.pcFace[kk]];
      int g = 0;
      while (g + 1 < P.nseg && sl >= P.segBeg[g + 1]) ++g;
      double *base = WHICH == HALO_W ? P.dstW[g] : P.dstT[P.tPar][g];
      base[sl - P.segBeg[g]] = val;
    }
    if (k1 > k0) lf_blockPushed = 1;
  }
}


// ------------------------------------------------------ L2 bulk prefetch
// cp.async.bulk.prefetch.L2 (sm_90+ TMA engine): one instruction pulls a
// contiguous byte range into L2 without occupying registers.  Each block
// prefetches the streamed arrays of its NEXT grid-stride trip, so DRAM
// latency overlaps the current trip and the demand loads hit L2.
#ifndef LF_PF
#define LF_PF 0          // trips ahead (0 = off).  Measured r1h: PF=1 slows phase 1 at
#endif                   // 200^3 from 181 to 246 us (profiles/variants_r1h.log) -> off
__device__ __forceinline__ void l2_prefetch(const void *p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
template <class T>
__device__ __forceinline__ void pf_range(const T *base, long off, int cnt) {
  const unsigned bytes = (unsigned)(cnt * (int)sizeof(T)) & ~15u;  // 16-byte multiple
  if (bytes) l2_prefetch(base + off, bytes);
}

__device__ __forceinline__ bool conv(double res, double init, const PcgCtl *ctl) {
  return res < ctl->tol || (ctl->relTol > 0.0 && res < ctl->relTol * init);
}

// Dispatch a KE-templated kernel on the mesh's ELL width.
#define LF_DISPATCH_KE(m, KERNEL, ...)                                     \
  do {                                                                     \
    if (!LF_NO_ELL && (m).K > 0 && (m).K <= 3) KERNEL<3> __VA_ARGS__;       \
    else if (!LF_NO_ELL && (m).K == 4) KERNEL<4> __VA_ARGS__;               \
    else if ((m).KS == 6) KERNEL<-6> __VA_ARGS__;                          \
    else if ((m).KS == 8) KERNEL<-8> __VA_ARGS__;                          \
    else KERNEL<0> __VA_ARGS__;                                            \
  } while (0)

// ------------------------------------------------------------------ sum
// sum(x) (gAverage numerator); with the peer-memory transport it also puts x
// at the processor-face cells into the neighbours' recvT (the halo of T/psi
// the next assembly / PCG setup reads), ordered before the allreduce.
__global__ void __launch_bounds__(BS, LF_MINB)
    k_sum(MeshDev m, const double *__restrict__ x, double *partials, unsigned *ticket, double *out,
          Workspace ws) {
  double v[1] = {0.0};
  const bool push = ws.p2p.P > 0;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < m.n; c += gridDim.x * blockDim.x) {
    const double xc = x[c];
    v[0] += xc;
    if (push) push_halo<HALO_T>(m, ws.p2p, c, xc);
  }
  reduce_grid<1>(v, partials, ticket, out, ws.p2p);
}

// Vector halo over the peer-memory transport (the gradient and the DT field
// of the corrected / variable-DT paths): component k of every send slot's
// cell into the neighbour's recvX, then an (empty) allreduce that orders the
// stores before the neighbour's next kernel.
__global__ void __launch_bounds__(BS, LF_MINB)
    k_push_x(MeshDev m, const double *__restrict__ x, int64_t stride, int ncomp, double *partials,
             unsigned *ticket, double *out, Workspace ws) {
  const P2PDev &P = ws.p2p;
  const int nslot = P.segBeg[P.nseg];
  for (int sl = blockIdx.x * blockDim.x + threadIdx.x; sl < nslot; sl += gridDim.x * blockDim.x) {
    const int cell = ws.sendCell[sl];
    int g = 0;
    while (g + 1 < P.nseg && sl >= P.segBeg[g + 1]) ++g;
    for (int k = 0; k < ncomp; ++k) P.dstX[g][(size_t)k * P.xStr[g] + (sl - P.segBeg[g])] = x[k * stride + cell];
    lf_blockPushed = 1;
  }
  double v[1] = {0.0};
  reduce_grid<1>(v, partials, ticket, out, ws.p2p);
}

void launch_push_x(cudaStream_t s, const Launch &L, const MeshDev &m, const double *x, int64_t stride, int ncomp,
                   const Workspace &ws, double *out) {
  k_push_x<<<L.grid, BS, 0, s>>>(m, x, stride, ncomp, ws.partials, ws.tickets + T_SUM, out, ws);
}

void launch_sum(cudaStream_t s, const Launch &L, const MeshDev &m, const double *x, const Workspace &ws,
                double *out) {
  k_sum<<<L.grid, BS, 0, s>>>(m, x, ws.partials, ws.tickets + T_SUM, out, ws);
}

// -------------------------------------------------------------- assembly
// fvm::ddt(T) - fvm::laplacian(DT,T) (SURVEY §8(c.1) lines 1-4, readings
// A3-A5) as a per-cell gather over the CSR lists.  Every coefficient is
// formed with the same rounded operations, in the same order, as the face
// loop of the definition (explicit _rn intrinsics: no FMA contraction), so
// diag/upper/source are bitwise those of the definition on upper-triangular
// meshes.  The owner side also writes the ELL copy upperE.
// SETUP additionally fuses the PCG prologue for psi = T0 = T: A psi (from
// the just-formed coefficients), r = b - A psi, normFactor terms with
// psibar = gSum(psi)/nTotal, sum|r|, w = r/diag and sum w.r.
template <bool SETUP>
__global__ void __launch_bounds__(BS, LF_MINB)
    k_assemble(MeshDev m, LduDev a, double DT, double rDeltaT, const double *__restrict__ T,
               const double *__restrict__ halo, Workspace ws, const double *__restrict__ T0,
               const double *__restrict__ lapSrc) {
  // T: psi (current T, initial guess); T0: old-time T for ddt (== T unless
  // non-orthogonal correctors run); lapSrc: explicit non-orthogonal part of
  // the corrected laplacian's source (null = orthogonal scheme)
  double psibar = 0.0;
  if (SETUP) psibar = ws.gsum->p1[1] / ws.ctl->nTotal;
  double v[3] = {0.0, 0.0, 0.0};
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < m.n; c += gridDim.x * blockDim.x) {
    double L = 0.0, sOff = 0.0, sU = 0.0;
    const int l0 = m.losortStart[c], l1 = m.losortStart[c + 1];
    for (int j = l0; j < l1; ++j) {
      const int f = m.losort[j];
      const double u = __dmul_rn(m.delta[f], __dmul_rn(m.gammaF ? m.gammaF[f] : DT, m.magSf[f]));
      if (a.symU) a.symU[(j - l0) * a.ldS + c] = -u;  // full-row copy (DIC)
      L = __dsub_rn(L, u);
      if (SETUP) {
        sOff = fma(-u, T[m.losortOwner[j]], sOff);
        sU -= u;
      }
    }
    const int o0 = m.ownerStart[c], o1 = m.ownerStart[c + 1];
    for (int i = o0; i < o1; ++i) {
      const double u = __dmul_rn(m.delta[i], __dmul_rn(m.gammaF ? m.gammaF[i] : DT, m.magSf[i]));
      if (a.writeUpper) a.upper[i] = -u;
      if (m.K > 0) a.upperE[(i - o0) * m.ldE + c] = -u;
      if (a.symU) a.symU[((l1 - l0) + (i - o0)) * a.ldS + c] = -u;
      L = __dsub_rn(L, u);
      if (SETUP) {
        sOff = fma(-u, T[m.nbr[i]], sOff);
        sU -= u;
      }
    }
    const double Tc = T[c];
    double d = __dsub_rn(__dmul_rn(rDeltaT, m.V[c]), L);
    double b = __dmul_rn(__dmul_rn(rDeltaT, T0[c]), m.V[c]);
    if (lapSrc) b = __dsub_rn(b, lapSrc[c]);  // TEqn = ddt - laplacian: source -= lap source
    double sP = 0.0, sBc = 0.0;
    const int b0 = m.bcStart[c], b1 = m.bcStart[c + 1];
    for (int k = b0; k < b1; ++k) {
      const int i = m.bcFace[k];
      const double gms = __dmul_rn(m.gammaB ? m.gammaB[i] : DT, m.bMagSf[i]);
      const double aa = __dmul_rn(gms, m.bDelta[i]);
      d = __dadd_rn(d, aa);
      a.bInt[i] = aa;
      if (m.bType[i] == LF_PATCH_FIXED_VALUE) {
        const double bb = __dmul_rn(gms, __dmul_rn(m.bDelta[i], m.bValue[i]));
        b = __dadd_rn(b, bb);
        a.bBnd[i] = bb;
      } else {  // processor: interfaceBouCoeffs = a, coupled via Amul
        a.bBnd[i] = aa;
        if (SETUP) {
          sP = fma(aa, halo[m.bSlot[i]], sP);
          sBc += aa;
        }
      }
    }
    a.diag[c] = d;
    a.source[c] = b;
    if (SETUP) {
      const double Ap = fma(d, Tc, sOff) - sP;
      const double sumA = d + sU - sBc;
      const double r = b - Ap;
      const double tmp = sumA * psibar;
      v[0] += fabs(Ap - tmp) + fabs(b - tmp);
      v[1] += fabs(r);
      const double w = (1.0 / d) * r;
      v[2] = fma(w, r, v[2]);
      ws.r[c] = r;
      ws.w[c] = w;
      if (ws.p2p.P > 0) push_halo<HALO_W>(m, ws.p2p, c, w);
    }
  }
  if (SETUP) {
    if (reduce_grid<3>(v, ws.partials, ws.tickets + T_ASM, ws.lsum->setup, ws.p2p) && threadIdx.x == 0) {
      PcgCtl *ctl = ws.ctl;
      ctl->it = 0;
      ctl->stop = 0;
      ctl->converged = 0;
      ctl->singular = 0;
    }
  }
}

void launch_assemble(cudaStream_t s, const Launch &L, const MeshDev &m, const LduDev &a, double DT,
                     double rDeltaT, const double *T, const double *halo, bool setup,
                     const Workspace &ws, const double *T0, const double *lapSrc) {
  if (!T0) T0 = T;
  if (setup)
    k_assemble<true><<<L.grid, BS, 0, s>>>(m, a, DT, rDeltaT, T, halo, ws, T0, lapSrc);
  else
    k_assemble<false><<<L.grid, BS, 0, s>>>(m, a, DT, rDeltaT, T, halo, ws, T0, lapSrc);
}

// ------------------------------------------------------------- PCG setup
// Prologue of a standalone pcg_solve: A psi from the stored coefficients,
// r = source - A psi, normFactor terms, sum|r|, w = r/diag, sum w.r.
template <int KE>
__global__ void __launch_bounds__(BS, LF_MINB_G)
    k_pcg_setup(MeshDev m, LduDev a, const double *__restrict__ halo, Workspace ws) {
  const double *psi = ws.ctl->psi;
  const double psibar = ws.gsum->p1[1] / ws.ctl->nTotal;
  double v[3] = {0.0, 0.0, 0.0};
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < m.n; c += gridDim.x * blockDim.x) {
    const double d = a.diag[c];
    double sU = 0.0, sBc = 0.0;
    const double sOff = row_offdiag<KE>(m, a, c, 0.0, [&](int j) { return psi[j]; }, &sU);
    const double Ap = fma(d, psi[c], sOff) - row_proc(m, a.bBnd, halo, c, &sBc);
    const double b = a.source[c];
    const double sumA = d + sU - sBc;
    const double r = b - Ap;
    const double tmp = sumA * psibar;
    v[0] += fabs(Ap - tmp) + fabs(b - tmp);
    v[1] += fabs(r);
    const double w = (1.0 / d) * r;
    v[2] = fma(w, r, v[2]);
    ws.r[c] = r;
    ws.w[c] = w;
    if (ws.p2p.P > 0) push_halo<HALO_W>(m, ws.p2p, c, w);
  }
  if (reduce_grid<3>(v, ws.partials, ws.tickets + T_SETUP, ws.lsum->setup, ws.p2p) && threadIdx.x == 0) {
    PcgCtl *ctl = ws.ctl;
    ctl->it = 0;
    ctl->stop = 0;
    ctl->converged = 0;
    ctl->singular = 0;
  }
}

void launch_pcg_setup(cudaStream_t s, const Launch &L, const MeshDev &m, const LduDev &a,
                      const double *halo, const Workspace &ws) {
  LF_DISPATCH_KE(m, k_pcg_setup, <<<L.grid, BS, 0, s>>>(m, a, halo, ws));
}

// ------------------------------------------------------ iteration state
// Everything a launch of iteration k derives from the previous launch's
// global sums (identical on every rank and every block).
struct IterState {
  int k;
  bool cont;
  double nf, initRes, finRes, wArA, beta;
};

__device__ __forceinline__ IterState derive_phase1(const Workspace &ws) {
  const PcgCtl *ctl = ws.ctl;
  IterState s;
  s.k = ctl->it;
  s.beta = 0.0;
  if (s.k == 0) {
    // OpenFOAM: normFactor = gSum(...) + small_; initRes = gSumMag(r)/normFactor;
    // iterate if minIter > 0 || !checkConvergence
    s.nf = ws.gsum->setup[0] + 1e-20;
    s.initRes = ws.gsum->setup[1] / s.nf;
    s.finRes = s.initRes;
    s.cont = ctl->minIter > 0 || !conv(s.finRes, s.initRes, ctl);
    s.wArA = ws.gsum->setup[2];
  } else {
    // while ((++it < maxIter && !converged) || it < minIter)
    s.nf = ctl->normFactor;
    s.initRes = ctl->initRes;
    s.finRes = ws.gsum->p2[0] / s.nf;
    s.cont = (s.k < ctl->maxIter && !conv(s.finRes, s.initRes, ctl)) || s.k < ctl->minIter;
    s.wArA = ws.gsum->p2[1];
    s.beta = s.wArA / ctl->wArA;
  }
  return s;
}

// p = w (first iteration) or w + beta*p_old — evaluated identically for a
// cell's own value and for the same cell seen as a neighbour (recomputed
// there instead of a third kernel / extra HBM pass), so A p uses exactly
// the stored p.
__device__ __forceinline__ double pval(const double *__restrict__ w, const double *__restrict__ pold,
                                       double beta, bool first, int j) {
  return first ? w[j] : fma(beta, pold[j], w[j]);
}

// ---------------------------------------------------------------- phase 1
// Deferred psi += alpha_{k-1} p_{k-1}; stopping test on the previous
// iteration's residual; p_k = w + beta p_{k-1}; q = A p_k; sum p.q, sum psi.
template <int KE, int PART = 0>
__global__ void __launch_bounds__(BS, LF_MINB_G)
    k_phase1(MeshDev m, LduDev a, Workspace ws, const int32_t *__restrict__ cells = nullptr, int32_t count = 0) {
  const PcgCtl *ctl = ws.ctl;
  if (ctl->stop) return;
  const IterState s = derive_phase1(ws);
  const bool first = (s.k == 0);
  const double alpha = ctl->alpha;
  double *psi = ctl->psi;
  const double *__restrict__ pold = (s.k & 1) ? ws.p[0] : ws.p[1];
  double *__restrict__ pnew = (s.k & 1) ? ws.p[1] : ws.p[0];
  const double *__restrict__ w = ws.w;
  double v[2] = {0.0, 0.0};
  const int nIt = PART == 0 ? m.n : count;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nIt; t += gridDim.x * blockDim.x) {
    const int c = PART == 0 ? t : cells[t];
#if LF_PF > 0
    if (KE > 0 && s.cont && threadIdx.x < 4 + 3 * KE) {
      const int cb = c - threadIdx.x + LF_PF * gridDim.x * blockDim.x;
      if (cb < m.n) {
        const int cnt = min((int)blockDim.x, m.n - cb), L = threadIdx.x;
        const long ld = m.ldE;
        if (L == 0) pf_range(w, cb, cnt);
        else if (L == 1) { if (!first) pf_range(pold, cb, cnt); }
        else if (L == 2) pf_range(psi, cb, cnt);
        else if (L == 3) pf_range(a.diag, cb, cnt);
        else if (L < 4 + KE) pf_range(a.upperE, (L - 4) * ld + cb, cnt);
        else if (L < 4 + 2 * KE) pf_range(m.nbrE, (L - 4 - KE) * ld + cb, cnt);
        else pf_range(m.loE, (L - 4 - 2 * KE) * ld + cb, cnt);
      }
    }
#endif
    double ps = psi[c];
    if (!first) {
      ps = fma(alpha, pold[c], ps);
      psi[c] = ps;
    }
    v[1] += ps;
    if (s.cont) {
      const double pc = pval(w, pold, s.beta, first, c);
      pnew[c] = pc;
      double q = a.diag[c] * pc;
      q = row_offdiag<KE>(m, a, c, q, [&](int j) { return pval(w, pold, s.beta, first, j); });
      q -= row_proc_p(m, a.bBnd, ws, first, s.beta, s.k, c);
      ws.q[c] = q;
      v[0] = fma(pc, q, v[0]);
    }
  }
  if constexpr (PART == 1) {  // interior cells: partial sums only
    reduce_grid<2>(v, ws.partials, ws.tickets + T_P1I, ws.lsum->p1x, ws.p2p);
    return;
  }
  if (reduce_grid<2>(v, ws.partials, ws.tickets + T_P1, ws.lsum->p1, ws.p2p) && threadIdx.x == 0) {
    PcgCtl *c = ws.ctl;
    if (PART == 2) {  // + the interior cells' sums (fixed order: deterministic)
      ws.lsum->p1[0] = v[0] + ws.lsum->p1x[0];
      ws.lsum->p1[1] = v[1] + ws.lsum->p1x[1];
    }
    if (first) {
      c->normFactor = s.nf;
      c->initRes = s.initRes;
    }
    c->finRes = s.finRes;
    c->wArA = s.wArA;
    if (!s.cont) {
      c->stop = 1;
      c->converged = conv(s.finRes, s.initRes, c) ? 1 : 0;
    }
  }
}

void launch_phase1(cudaStream_t s, const Launch &L, const MeshDev &m, const LduDev &a,
                   const Workspace &ws) {
  LF_DISPATCH_KE(m, k_phase1, <<<L.grid, BS, 0, s>>>(m, a, ws));
}

template <int KE>
static void phase1_part(cudaStream_t s, const Launch &L, const MeshDev &m, const LduDev &a, const Workspace &ws,
                        int part, const int32_t *cells, int32_t count) {
  if (part == 1)
    k_phase1<KE, 1><<<L.grid, BS, 0, s>>>(m, a, ws, cells, count);
  else
    k_phase1<KE, 2><<<L.grid, BS, 0, s>>>(m, a, ws, cells, count);
}

void launch_phase1_part(cudaStream_t s, const Launch &L, const MeshDev &m, const LduDev &a, const Workspace &ws,
                        int part, const int32_t *cells, int32_t count) {
  if (!LF_NO_ELL && m.K > 0 && m.K <= 3) phase1_part<3>(s, L, m, a, ws, part, cells, count);
  else if (!LF_NO_ELL && m.K == 4) phase1_part<4>(s, L, m, a, ws, part, cells, count);
  else if (m.KS == 6) phase1_part<-6>(s, L, m, a, ws, part, cells, count);
  else if (m.KS == 8) phase1_part<-8>(s, L, m, a, ws, part, cells, count);
  else phase1_part<0>(s, L, m, a, ws, part, cells, count);
}

// ---------------------------------------------------------------- phase 2
// checkSingularity(|wApA|/normFactor); alpha = wArA/wApA; r -= alpha q;
// w = rD r (diagonal preconditioner, rD = 1/diag); sum|r|, sum w.r.
__global__ void __launch_bounds__(BS, LF_MINB)
    k_phase2(MeshDev m, LduDev a, Workspace ws) {
  const int n = m.n;
  const bool push = ws.p2p.P > 0;
  const PcgCtl *ctl = ws.ctl;
  if (ctl->stop) return;
  const int k = ctl->it;
  const double pq = ws.gsum->p1[0];
  const bool singular = fabs(pq) / ctl->normFactor < 1e-300;
  const double alpha = ctl->wArA / pq;
  double v[2] = {0.0, 0.0};
  if (!singular) {
    // LF_P2_UNROLL cells per trip: all loads of the trip issued first
    constexpr int U = LF_P2_UNROLL;
    const int stride = gridDim.x * blockDim.x;
    for (int c0 = blockIdx.x * blockDim.x + threadIdx.x; c0 < n; c0 += stride * U) {
#if LF_PF > 0
      if (threadIdx.x < 3 * U) {
        const int cb = c0 - threadIdx.x + LF_PF * stride * U + (threadIdx.x / 3) * stride;
        if (cb < n) {
          const int cnt = min((int)blockDim.x, n - cb), L = threadIdx.x % 3;
          pf_range(L == 0 ? ws.q : (L == 1 ? ws.r : a.diag), cb, cnt);
        }
      }
#endif
      double q[U], r[U], d[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + u * stride;
        const bool ok = c < n;
        q[u] = ok ? ws.q[c] : 0.0;
        r[u] = ok ? ws.r[c] : 0.0;
        d[u] = ok ? a.diag[c] : 1.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + u * stride;
        if (c < n) {
          const double rn = fma(-alpha, q[u], r[u]);
          const double w = (1.0 / d[u]) * rn;
          ws.r[c] = rn;
          ws.w[c] = w;
          if (push) push_halo<HALO_W>(m, ws.p2p, c, w);
          v[0] += fabs(rn);
          v[1] = fma(w, rn, v[1]);
        }
      }
    }
  }
  if (reduce_grid<2>(v, ws.partials, ws.tickets + T_P2, ws.lsum->p2, ws.p2p) && threadIdx.x == 0) {
    PcgCtl *c = ws.ctl;
    if (singular) {
      c->stop = 1;
      c->singular = 1;
      c->converged = conv(c->finRes, c->initRes, c) ? 1 : 0;
    } else {
      c->alpha = alpha;
      c->it = k + 1;
    }
  }
}

void launch_phase2(cudaStream_t s, const Launch &L, const MeshDev &m, const LduDev &a, const Workspace &ws) {
  k_phase2<<<L.grid, BS, 0, s>>>(m, a, ws);
}

// ------------------------------------------------- persistent PCG (1 GPU)
// The whole solve in ONE cooperative launch (resident grid, all blocks
// co-scheduled): the two phases of every iteration are separated by grid
// barriers instead of kernel boundaries.  At a barrier each block publishes
// its partial sums; the last block to arrive (integer ticket) sums them in
// block order (same order as reduce_grid: results bitwise equal to the
// launch-per-phase path for the same grid), publishes the totals and
// releases the barrier.  Scalars (alpha, beta, stopping rule) live in
// registers, identical in every block.  Data written by other blocks during
// the launch (w, p at neighbour cells, the totals) is read with ld.global.cg
// (L2) because L1 is not coherent within a launch; everything else is
// either read-only or written and re-read by the same thread.
#ifndef LF_PERSIST_LDCG
#define LF_PERSIST_LDCG 0  // 1: neighbour reads via ld.cg instead of L1 invalidation at barriers
#endif
__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned *p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

#ifndef LF_SPIN_NS
#define LF_SPIN_NS 32  // grid-barrier poll back-off (ns)
#endif
// wait until the barrier generation moves past gen: relaxed polls, then one
// acquire (orders the later loads; the single L1 invalidation they need)
__device__ __forceinline__ void wait_generation(const unsigned *gp, unsigned gen) {
  const unsigned long long t0 = gtime_ns();
  unsigned tries = 0;
  while ((LF_SPIN_RELAXED ? ld_relaxed(gp) : ld_acquire(gp)) == gen) {
    if (LF_SPIN_NS > 0) __nanosleep(LF_SPIN_NS);
    spin_check(t0, tries);
  }
  if (LF_SPIN_RELAXED) (void)ld_acquire(gp);
}
#ifndef LF_BAR_ACQREL
#define LF_BAR_ACQREL 1  // grid barrier with acq_rel atomics instead of fence + atomic
#endif
#if LF_TIMING
#define LF_DBG_ARG(x) , (x)
#else
#define LF_DBG_ARG(x)
#endif
#if LF_TIMING
// barrier anatomy snapshot (debug builds): arrival / release / wake times
constexpr int LF_DBG_N = 64, LF_DBG_G = 1024;
__device__ unsigned long long g_dbg_arr[LF_DBG_N][LF_DBG_G], g_dbg_wake[LF_DBG_N][LF_DBG_G];
__device__ unsigned long long g_dbg_rel[LF_DBG_N];
__device__ int g_dbg_last[LF_DBG_N];
__device__ int g_dbg_smid[LF_DBG_G];
__device__ int g_dbg_i_dummy;
#define g_dbg_i dbg_i
#endif
// `idle` (all threads of a block) runs while the block waits for the
// release — after its arrival, or after the release in the last arriving
// block — so independent work fills the barrier's sync latency.
struct NoIdle {
  __device__ void operator()() const {}
};
// PEER = false compiles the cross-rank exchange out (single-rank variants).
template <int NV, bool PEER = true, class Idle = NoIdle>
__device__ void grid_reduce_sync(double (&v)[NV], double *partials, unsigned *bar, double *out,
                                 const P2PDev &P
#if LF_TIMING
                                 , int dbg_i
#endif
                                 , Idle idle = Idle(), const double *xtra = nullptr, int nx = 0,
                                 unsigned *rst = nullptr) {
  // xtra (nx > 0): per-unit sums of run-time scheduled work (xtra[k * nx +
  // u]), added after the gridDim.x block partials in index order: the totals
  // do not depend on which block ran a unit; rst: a counter the last block
  // zeroes before releasing
  __shared__ double sm[NV][32];
  __shared__ int amLast;
  block_sum<NV>(v, sm);
  unsigned gen = 0;  // thread 0: barrier generation before arriving
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) partials[k * gridDim.x + blockIdx.x] = v[k];
    gen = ld_relaxed(bar + 1);  // read before arriving (ordered by the release of the arrival)
#if LF_TIMING
    if (g_dbg_i < LF_DBG_N && blockIdx.x < LF_DBG_G) {
      g_dbg_arr[g_dbg_i][blockIdx.x] = gtime_ns();
      unsigned sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      g_dbg_smid[blockIdx.x] = (int)sm;
    }
#endif
    unsigned t;
    if (PEER && P.P > 0) {
      fence_pushed();  // peer-memory halo stores of this block (if any) precede the arrival
      // acq_rel: the last arriver also acquires every block's partials
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(t) : "l"(bar) : "memory");
    } else {
#if LF_BAR_ACQREL
      // release: the block's writes (ordered by the bar.sync above) precede the
      // arrival; acquire: the last arriver sees every block's partials
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(t) : "l"(bar) : "memory");
#else
      __threadfence();
      t = atomicAdd(bar, 1u);
#endif
    }
    amLast = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!amLast) idle();
  if (!amLast && threadIdx.x == 0) {
    {
      // ld.acquire.gpu orders the later loads and invalidates this SM's L1
      // (SASS CCTL.IVALL), so cached loads of other blocks' data are coherent
      wait_generation(bar + 1, gen);
#if LF_TIMING
      if (g_dbg_i < LF_DBG_N && blockIdx.x < LF_DBG_G) g_dbg_wake[g_dbg_i][blockIdx.x] = gtime_ns();
#endif
    }
  }
  __syncthreads();
  if (amLast) {
#if !LF_BAR_ACQREL
    __threadfence();
#endif
    double s[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) s[k] = 0.0;
    constexpr int U = 8;  // one L2 round trip for grids up to 8*blockDim
    const int G = (int)gridDim.x, NT = G + nx;
    for (int b0 = threadIdx.x; b0 < NT; b0 += blockDim.x * U) {
      double t[U][NV];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int b = b0 + u * blockDim.x;
#pragma unroll
        for (int k = 0; k < NV; ++k)
          t[u][k] = b < G ? __ldcg(&partials[k * G + b]) : (b < NT ? __ldcg(&xtra[(long)k * nx + (b - G)]) : 0.0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int k = 0; k < NV; ++k) s[k] += t[u][k];
    }
    block_sum<NV>(s, sm);
    if (PEER && P.P > 0) p2p_allreduce<NV>(P, s);  // ranks exchange totals before the local release
    if (threadIdx.x == 0) {
#pragma unroll
      for (int k = 0; k < NV; ++k) out[k] = s[k];
      if (rst) *rst = 0u;
      bar[0] = 0u;
#if LF_TIMING
      if (g_dbg_i < LF_DBG_N) {
        g_dbg_rel[g_dbg_i] = gtime_ns();
        g_dbg_last[g_dbg_i] = blockIdx.x;
      }
#endif
#if LF_BAR_ACQREL
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar + 1) : "memory");  // release
#else
      __threadfence();
      atomicAdd(bar + 1, 1u);  // release
#endif
    }
    __syncthreads();
    idle();  // the last arriver's own idle work, after releasing the others
    __syncthreads();
  }
}

// Plain grid barrier of the persistent kernels (no reduction): same
// protocol as grid_reduce_sync (acq_rel arrival, release by the last block,
// ld.acquire spin that also invalidates the SM's L1).
__device__ __forceinline__ void grid_barrier(unsigned *bar) {
  __shared__ int amLastB;
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned gen = ld_relaxed(bar + 1);
    unsigned t;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(t) : "l"(bar) : "memory");
    amLastB = (t == gridDim.x - 1);
    if (amLastB) {
      bar[0] = 0u;
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar + 1) : "memory");
    } else {
      wait_generation(bar + 1, gen);
    }
  }
  __syncthreads();
}

#ifndef LF_MINB_P
#define LF_MINB_P 2  // persistent kernel blocks/SM (x512 threads): 64 registers, no spills
                     // (r1o: 100^3 3.39 ms/step at 64 regs vs 3.71 with 60 B of spills)
#endif
#ifndef LF_TIMING
#define LF_TIMING 0  // 1: per-phase / per-barrier times printed by the persistent kernel
#endif
// default share (%) of phase-1 trips scheduled at run time (HBM-bound
// variant).  200^3 on boxes with slow SMs (r6n/r6r/r6s): 43.4-44.4 ->
// 41.2-41.5 ms/step at 25-40% (best 33%); on the others 38.9-39.3 at 0%,
// -1% at 25%, -2% at 40% (r6o/r6q); 400^3 658 -> 636 ms; permuted 200^3
// 199 -> 191 ms
#ifndef LF_DYN_PCT
#define LF_DYN_PCT 30
#endif
#ifndef LF_DYN
#define LF_DYN 0  // 1: run-time trips compiled into the persistent diagonal solve.  Off: the
#endif            // extra code costs the static trip loop spills (r6zb, one box: 200^3 217 ->
                  // 224-228 us/iteration, 400^3 1937 -> 2056) while the balancing gains
                  // 5-10% only on boxes with a slow TPC (r6n/r6r/r6s)
#ifndef LF_DYN_UT
#define LF_DYN_UT 2  // grid-stride trips per run-time scheduled unit (UT x one 512-cell block run)
#endif
#ifndef LF_DYN_MAXU
#define LF_DYN_MAXU 32  // run-time units a block may take per phase (shared-memory slots)
#endif
#ifndef LF_CHUNKED
#define LF_CHUNKED 0  // persistent kernel: contiguous cell chunk per block (vs grid stride).
#endif                // r1n: chunks raise the phase-1 arrival spread 6 -> 28 us at 100^3 -> off
bool persistent_chunked() { return LF_CHUNKED != 0; }
#ifndef LF_IDLE_FLUSH
#define LF_IDLE_FLUSH 1  // persistent kernel may do psi += alpha p while waiting at the beta
#endif                   // barrier (Workspace.idleFlush, set per mesh: L2-resident sizes)
#ifndef LF_REVERSE
#define LF_REVERSE 1  // persistent phase 2 sweeps the trips in reverse order (L2 reuse)
#endif
#ifndef LF_STASH_DIAG
#define LF_STASH_DIAG 1  // L2-resident variant: diag re-read from the stash after iteration 0
#endif
#ifndef LF_STASH_TRIPS
#define LF_STASH_TRIPS 8  // L2-resident variant: at most this many grid-stride trips per thread
#endif
#ifndef LF_TAIL
#define LF_TAIL 1  // persistent kernel: spread the last partial trip over all blocks
#endif
bool persistent_tail() { return LF_TAIL != 0; }
int stash_trips() { return LF_TAIL ? LF_STASH_TRIPS : 0; }
int dynamic_trips_pct() { return LF_DYN ? LF_DYN_PCT : 0; }
static size_t stash_bytes() { return (size_t)LF_STASH_TRIPS * BS * sizeof(double2); }
#ifndef LF_STASH_FIT
#define LF_STASH_FIT 1  // launch with only the stash slots the mesh's trips use (more L1 left)
#endif
// dynamic shared memory of an L2-resident launch: slot i * BS + thread for
// the trips i < ceil(n / (grid * BS)) (<= LF_STASH_TRIPS), times `per` bytes
static size_t stash_fit(int n, int grid, size_t per) {
  const long long cstep = (long long)grid * BS, trips = (n + cstep - 1) / cstep;
  const long long t = LF_STASH_FIT ? std::max(1LL, std::min<long long>(trips, LF_STASH_TRIPS)) : LF_STASH_TRIPS;
  return (size_t)t * BS * per;
}
#ifndef LF_P2P_UNROLL
#define LF_P2P_UNROLL 2  // persistent phase 2 cells per trip
#endif
// HALO = false: single rank without processor patches — the interface
// term, halo puts and peer allreduce are compiled out of the hot loop
// (they cost 13% at 100^3 even when branched around, r1o).
#ifndef LF_W88
#define LF_W88 0   // 1: HBM-bound variant does not store w (SURVEY's 88n + 16F iteration): phase 1
#endif             // recomputes w = (1/diag) r at the cell and its neighbours.  Measured (r4d,
                   // 200^3): 53.8 vs 40.5 ms/step — 7 FP64 divisions per cell cost more than 8n bytes.
                   // 2: the same with rD = 1/diag stored once per solve (ws.rDiag): neighbours
                   // form w = rD r (no division), the own cell (1/diag) r (one), phase 2 reads rD
                   // instead of diag: 80n + 16F per iteration
#ifndef LF_CPASYNC
#define LF_CPASYNC 0  // HBM-bound variant: phase 1 streams each thread's own-cell operands of the
#endif                // NEXT trip into shared memory with cp.async while the current trip gathers
constexpr int CPA_D = 9, CPA_I = 6;  // per-thread slots: 9 doubles, 6 labels (SoA over the block)
constexpr size_t CPA_BYTES = (size_t)BS * (CPA_D * sizeof(double) + CPA_I * sizeof(int));
__device__ __forceinline__ void cpa8(void *smem, const void *g) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void cpa4(void *smem, const void *g) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cpa_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// half-ELL row with the slot data already loaded (row_offdiag<KE > 0>)
template <int KE, class XF>
__device__ __forceinline__ double row_pre(const LduDev &a, int n, const int (&lo)[KE], const int (&nb)[KE],
                                          const double (&uo)[KE], double acc, XF xval) {
  double lu[KE], lx[KE], ox[KE];
#pragma unroll
  for (int k = 0; k < KE; ++k) {
    const int oc = lo[k] & ELL_MASK;
    lu[k] = lo[k] >= 0 ? a.upperE[(lo[k] >> ELL_SHIFT) * n + oc] : 0.0;
    lx[k] = lo[k] >= 0 ? xval(oc) : 0.0;
    ox[k] = nb[k] >= 0 ? xval(nb[k]) : 0.0;
  }
#pragma unroll
  for (int k = 0; k < KE; ++k)
    if (lo[k] >= 0) acc = fma(lu[k], lx[k], acc);
#pragma unroll
  for (int k = 0; k < KE; ++k)
    if (nb[k] >= 0) acc = fma(uo[k], ox[k], acc);
  return acc;
}

#ifndef LF_IDLE_PF
#define LF_IDLE_PF 0  // HBM-bound variant: trips whose own-cell streams a block prefetches into
#endif                // L2 (cp.async.bulk.prefetch.L2) while it waits at a grid barrier — phase 2's
                      // first trips at the alpha barrier, the next phase 1's at the beta barrier
#ifndef LF_QREC
#define LF_QREC 0  // HBM-bound variant: q = A p by the recurrence q_k = A w_k + beta q_{k-1}
#endif             // (p_k = w_k + beta p_{k-1}): ONE gather per neighbour (w) instead of two
                   // (w, p_old), for one more stream (q_{k-1}, 8n)
#ifndef LF_LPF
#define LF_LPF 1  // HBM-bound variant: each warp prefetches into L2 (prefetch.global.L2,
#endif            // lane-distributed: one or two instructions per thread, no registers held)
                  // the lines of its own-cell streams LF_LPF trips ahead in phase 1 when
                  // ws.l2pf (chosen per mesh, mesh.cpp; r6b 200^3: 40.8 -> 38.5 ms/step)
#ifndef LF_LPF_MASK
#define LF_LPF_MASK 15  // streams prefetched: 1 labels, 2 owner-side coefficients, 4 w / diag / p_old,
#endif                  // 8 psi / p_{k-2}
#ifndef LF_LPF_BULK
#define LF_LPF_BULK 0  // 1: the prefetch as one cp.async.bulk.prefetch.L2 per stream and block run
#endif
#ifndef LF_LPF2
#define LF_LPF2 0  // the same for phase 2's streams (r, q, diag), trips ahead in its order
#endif
__device__ __forceinline__ void l2_pf_line(const void *p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
struct PfEnt {
  const char *p;  // array base + byte offset of the point inside a warp's run
  int sh;         // log2 element size
};
#ifndef LF_PSI2
#define LF_PSI2 1  // HBM-bound variant: psi written every second iteration (two deferred
#endif             // updates applied in sequence: bitwise the one-at-a-time psi), -4n/iteration
                   // (r4d, 200^3: 40.13 vs 40.52 ms/step)
template <int KE, bool HALO, bool IDLE = false, bool E16 = false>
__global__ void __launch_bounds__(BS, LF_MINB_P)
    k_pcg_persistent(MeshDev m, LduDev a, Workspace ws, unsigned *bar) {
  constexpr int w88 = IDLE ? 0 : LF_W88;
  constexpr bool psi2 = LF_PSI2 && !IDLE;
  constexpr bool qrec = LF_QREC && !IDLE && !HALO && w88 == 0;
  constexpr bool cpa = LF_CPASYNC && LF_TAIL && !IDLE && KE > 0 && !E16 && w88 == 0;
  PcgCtl *ctl = ws.ctl;
  if (!HALO) ws.p2p.P = 0;
  if (ctl->stop) return;
  // block-uniform solver state lives in shared memory (thread 0 updates it
  // between barriers) so it does not occupy registers across the phases
  struct St {
    double nf, initRes, finRes, wArA, alpha, alphaPrev, beta;
    int k, cont, singular;
  };
  __shared__ St st;
  // run-time trips (phase 1, see below): claimed unit per slot (-1: not yet)
  // and each warp's sums per slot
  constexpr bool dyn = LF_DYN && LF_TAIL && !IDLE && !HALO && !qrec && w88 == 0 && !cpa;
  __shared__ int dynU[dyn ? LF_DYN_MAXU : 1];
  __shared__ double dynP[dyn ? LF_DYN_MAXU : 1][BS / 32][2];
  if (dyn && (int)threadIdx.x < LF_DYN_MAXU) dynU[threadIdx.x] = -1;
  if (threadIdx.x == 0) {
    st.k = ctl->it;
    st.nf = ctl->normFactor;
    st.initRes = ctl->initRes;
    st.finRes = ctl->finRes;
    st.wArA = ctl->wArA;
    st.alpha = ctl->alpha;
    st.alphaPrev = 0.0;
    st.singular = 0;
  }
  double *psi = ctl->psi;
  const double *__restrict__ w = ws.w;
  const double *__restrict__ rr = ws.r;
  // w at cell j: stored (w[j]) or, in the 88n variant, recomputed exactly as
  // phase 2 / the setup formed it: (1/diag_j) r_j
  const double *__restrict__ rDg = ws.rDiag;
  auto wv = [&](int j) -> double {
    if constexpr (w88 == 2) return rDg[j] * rr[j];
    else if constexpr (w88 == 1) return (1.0 / a.diag[j]) * rr[j];
    else return w[j];
  };
  double psiSum = 0.0;  // LF_IDLE_FLUSH: this thread's sum of psi after its last flush
  // IDLE (L2-resident sizes, <= LF_STASH_TRIPS trips per thread): phase 1
  // keeps each cell's {q, diag} in shared memory (slot = trip) for phase 2,
  // so q is never written to / read from global memory and diag is not
  // re-read: phase 2 streams r only (-24n bytes per iteration)
  extern __shared__ double2 lf_stash[];
#if LF_CHUNKED
  // block b owns the contiguous cells [b*C, (b+1)*C): equal work per block on
  // an SM-uniform grid (numSMs x blocks/SM), the same cells in both phases
  const int C = (((m.n + (int)gridDim.x - 1) / (int)gridDim.x) + 31) & ~31;
  const int cbeg = min((int)blockIdx.x * C, m.n), cend = min(cbeg + C, m.n);
  const int cstart = cbeg + threadIdx.x, cstep = blockDim.x;
#else
  const int cstart = blockIdx.x * blockDim.x + threadIdx.x, cend = m.n, cstep = gridDim.x * blockDim.x;
#endif
#if LF_TAIL
  // full grid-stride trips while every thread has a cell, then ONE tail trip
  // whose R leftover cells are spread evenly over all blocks (ceil(R/G)
  // consecutive cells each): every block handles the same number of cells
  // +-1 and all SMs still sweep the cell range together (L2 reuse of the
  // neighbour gathers).  Same mapping in both phases.
  const int nFull = m.n / cstep;
  int tailC;
  {
    const int base = nFull * cstep, R = m.n - base, per = (R + (int)gridDim.x - 1) / (int)gridDim.x;
    const int off = (int)blockIdx.x * per + (int)threadIdx.x;
    tailC = ((int)threadIdx.x < per && off < R) ? base + off : -1;
  }
#endif
#if LF_TIMING
  unsigned long long tprev = 0, tacc[4] = {0, 0, 0, 0};
#define LF_TSTAMP(i)                                   \
  do {                                                 \
    const unsigned long long tn_ = gtime_ns();         \
    if ((i) > 0) tacc[(i) - 1] += tn_ - tprev;         \
    tprev = tn_;                                       \
  } while (0)
#else
#define LF_TSTAMP(i) \
  do {               \
  } while (0)
#endif
  if constexpr (w88 == 2) {
    // rD = 1/diag once per solve (the value phase 2 / the setup divide by)
    for (int c = cstart; c < cend; c += cstep) ws.rDiag[c] = 1.0 / a.diag[c];
    grid_barrier(bar);
  }
  for (;;) {
    // ---- derive (OpenFOAM loop condition) from the previous totals
    if (threadIdx.x == 0) {
      if (st.k == 0) {
        st.nf = __ldcg(&ws.gsum->setup[0]) + 1e-20;
        st.initRes = __ldcg(&ws.gsum->setup[1]) / st.nf;
        st.finRes = st.initRes;
        st.cont = ctl->minIter > 0 || !conv(st.finRes, st.initRes, ctl);
        st.wArA = __ldcg(&ws.gsum->setup[2]);
        st.beta = 0.0;
      } else {
        st.finRes = __ldcg(&ws.gsum->p2[0]) / st.nf;
        st.cont = (st.k < ctl->maxIter && !conv(st.finRes, st.initRes, ctl)) || st.k < ctl->minIter;
        const double wn = __ldcg(&ws.gsum->p2[1]);
        st.beta = wn / st.wArA;
        st.wArA = wn;
      }
    }
    __syncthreads();
    const int k = st.k;
    const bool first = (k == 0), cont = st.cont != 0;
    const double beta = st.beta, alpha = st.alpha, alphaPrev = st.alphaPrev;
    const double *__restrict__ pold = (k & 1) ? ws.p[0] : ws.p[1];
    double *__restrict__ pnew = (k & 1) ? ws.p[1] : ws.p[0];
    // psi2: this pass writes psi when it is the last one or k is even (>= 2):
    // psi += alpha_{k-2} p_{k-2} (still in pnew) then alpha_{k-1} p_{k-1}
    const bool even2 = psi2 && k >= 2 && !(k & 1);
    const bool psiPass = !psi2 || !cont || even2 || first;  // k = 0: sum(psi) for a singular stop
    auto pnb = [&](int j) {  // p at a neighbour cell (written by another block)
#if LF_PERSIST_LDCG
      return first ? __ldcg(w + j) : fma(beta, __ldcg(pold + j), __ldcg(w + j));
#else  // L1 was invalidated by the barrier's ld.acquire.gpu: cached loads are coherent
      return first ? wv(j) : fma(beta, pold[j], wv(j));
#endif
    };
    // ---- phase 1: flush psi, p = w + beta p_old, q = A p, sums
    double v1[2] = {0.0, 0.0};
    LF_TSTAMP(0);
    constexpr bool idleF = IDLE;  // psi flush in the beta-barrier wait (Workspace.idleFlush)
    if (idleF) v1[1] = psiSum;  // sum psi after the flush done in the previous barrier's wait
    bool piped = false;  // phase 1 done by the cp.async pipeline
#if LF_TAIL
    if constexpr (cpa) if (cont) {
      piped = true;
      // cp.async pipeline: the own-cell operands of trip i+1 (labels, owner-
      // side coefficients, w, p_old, diag, psi, p_{k-2}, q_old) land in this
      // thread's shared-memory slots while trip i's neighbour gathers run
      // (per-thread groups: no block synchronisation)
      double *sD = reinterpret_cast<double *>(lf_stash);
      int *sI = reinterpret_cast<int *>(sD + CPA_D * BS);
      const int t = threadIdx.x, n = m.ldE;
      auto cell_of = [&](int i) { return i < nFull ? cstart + i * cstep : (i == nFull ? tailC : -1); };
      auto fetch = [&](int c) {
        if (c >= 0) {
#pragma unroll
          for (int kk = 0; kk < KE; ++kk) {
            cpa4(sI + kk * BS + t, m.loE + kk * n + c);
            cpa4(sI + (KE + kk) * BS + t, m.nbrE + kk * n + c);
            cpa8(sD + kk * BS + t, a.upperE + kk * n + c);
          }
          cpa8(sD + 3 * BS + t, w + c);
          cpa8(sD + 5 * BS + t, a.diag + c);
          if (!first) cpa8(sD + 4 * BS + t, pold + c);
          if (psiPass) cpa8(sD + 6 * BS + t, psi + c);
          if (even2) cpa8(sD + 7 * BS + t, pnew + c);
          if (qrec && !first) cpa8(sD + 8 * BS + t, ws.q + c);
        }
        cpa_commit();
      };
      fetch(cell_of(0));
      for (int i = 0; i <= nFull; ++i) {
        const int c = cell_of(i);
        cpa_wait_all();
        if (c < 0) break;
        int lo[KE], nb[KE];
        double uo[KE];
#pragma unroll
        for (int kk = 0; kk < KE; ++kk) {
          lo[kk] = sI[kk * BS + t];
          nb[kk] = sI[(KE + kk) * BS + t];
          uo[kk] = sD[kk * BS + t];
        }
        const double wc = sD[3 * BS + t], dc = sD[5 * BS + t];
        const double po = first ? 0.0 : sD[4 * BS + t];
        const double ps0 = psiPass ? sD[6 * BS + t] : 0.0, pn2 = even2 ? sD[7 * BS + t] : 0.0;
        const double qo = (qrec && !first) ? sD[8 * BS + t] : 0.0;
        fetch(cell_of(i + 1));
        if (psiPass) {
          double ps = ps0;
          if (even2) ps = fma(alphaPrev, pn2, ps);
          if (!first) {
            ps = fma(alpha, po, ps);
            psi[c] = ps;
          }
          v1[1] += ps;
        }
        const double pc = first ? wc : fma(beta, po, wc);
        pnew[c] = pc;
        double q;
        if constexpr (qrec) {
          q = row_pre<KE>(a, n, lo, nb, uo, dc * wc, [&](int j) { return w[j]; });
          if (!first) q = fma(beta, qo, q);
        } else {
          q = row_pre<KE>(a, n, lo, nb, uo, dc * pc, pnb);
        }
        if (HALO) q -= row_proc_p(m, a.bBnd, ws, first, beta, k, c);
        ws.q[c] = q;
        v1[0] = fma(pc, q, v1[0]);
      }
      cpa_wait_all();
    }
#if LF_TAIL
    constexpr bool lpf = LF_LPF > 0 && !IDLE && KE > 0 && !E16 && w88 == 0 && !qrec;
    // lane-distributed L2 prefetch table: entry e = one point (first / middle
    // / last byte) of one stream's 32-cell run; a warp covers every line of
    // its run with one or two prefetch instructions per lane
    __shared__ PfEnt pfTab[64];
    __shared__ int pfN;
    const int wbase = (int)blockIdx.x * BS + (int)(threadIdx.x & ~31u);
    const int lane = threadIdx.x & 31;
    // lane-distributed prefetch of the warp's 32-cell run starting at cell cb
    auto pf_cb = [&](long cb, int ne) {
      if (lane < ne) l2_pf_line(pfTab[lane].p + (cb << pfTab[lane].sh));
      if (lane + 32 < ne) l2_pf_line(pfTab[lane + 32].p + (cb << pfTab[lane + 32].sh));
    };
    auto pf_trip = [&](int ii, int ne) {
#if LF_LPF_BULK
      // one bulk L2 prefetch (TMA) per stream of the block's 512-cell run
      if (ii < nFull && (int)threadIdx.x < ne) {
        const PfEnt e = pfTab[threadIdx.x];
        const long cb = (long)blockIdx.x * BS + (long)ii * cstep;
        l2_prefetch(e.p + (cb << e.sh), (unsigned)BS << e.sh);
      }
      return;
#endif
      if (ii < nFull) {
        const long cb = (long)wbase + (long)ii * cstep;
        if (lane < ne) l2_pf_line(pfTab[lane].p + (cb << pfTab[lane].sh));
        if (lane + 32 < ne) l2_pf_line(pfTab[lane + 32].p + (cb << pfTab[lane + 32].sh));
      }
    };
    int pfn = 0;
    if constexpr (lpf) {
      if (cont && ws.l2pf && threadIdx.x == 0) {
        int e = 0;
        const long ld = m.ldE;
        auto addI = [&](const int32_t *b) {
          pfTab[e++] = {(const char *)b, 2};
          if (!LF_LPF_BULK) pfTab[e++] = {(const char *)b + 124, 2};
        };
        auto addD = [&](const double *b) {
          pfTab[e++] = {(const char *)b, 3};
          if (!LF_LPF_BULK) pfTab[e++] = {(const char *)b + 128, 3};
          if (!LF_LPF_BULK) pfTab[e++] = {(const char *)b + 248, 3};
        };
        for (int kk = 0; kk < KE; ++kk) {
          if (LF_LPF_MASK & 1) addI(m.loE + kk * ld);
          if (LF_LPF_MASK & 1) addI(m.nbrE + kk * ld);
          if (LF_LPF_MASK & 2) addD(a.upperE + kk * ld);
        }
        if (LF_LPF_MASK & 4) addD(w);
        if (LF_LPF_MASK & 4) addD(a.diag);
        if ((LF_LPF_MASK & 4) && !first) addD(pold);
        if ((LF_LPF_MASK & 8) && psiPass) addD(psi);
        if ((LF_LPF_MASK & 8) && even2) addD(pnew);
        pfN = e;
        e = 48;  // phase 2's streams
        addD(ws.q);
        addD(ws.r);
        addD(a.diag);
      }
      if (threadIdx.x == 0 && !(cont && ws.l2pf)) pfN = 0;
      __syncthreads();
      pfn = pfN;
      if (cont)
        for (int ii = 0; ii < LF_LPF; ++ii) pf_trip(ii, pfn);
    }
#endif
#endif  // LF_TAIL (cp.async pipeline)
    // one cell of phase 1 (i: its trip, the stash slot of the L2-resident variant)
    auto cell1 = [&](const int c, const int i, double (&acc)[2]) {
      const int pflag = HALO ? (int)has_proc(m, c) : 0;  // issued with the cell's own loads
      if (idleF) {
        if (first) acc[1] += psi[c];
      } else if (psiPass) {
        double ps = psi[c];
        if (even2) ps = fma(alphaPrev, pnew[c], ps);  // read before pnew[c] is overwritten below
        if (!first) {
          ps = fma(alpha, pold[c], ps);
          psi[c] = ps;
        }
        acc[1] += ps;
      }
      if (cont) {
#if LF_TAIL
        // the L2-resident variant reads diag from HBM once per solve: later
        // iterations take it from the stash slot it stays in
        const double dc = (IDLE && LF_STASH_DIAG && !first) ? lf_stash[i * BS + threadIdx.x].y : a.diag[c];
#else
        const double dc = a.diag[c];
#endif
        const double wc = w88 ? (1.0 / dc) * rr[c] : w[c];
        const double pc = first ? wc : fma(beta, pold[c], wc);
        pnew[c] = pc;
        double q;
        if constexpr (qrec) {
          auto wnb = [&](int j) { return w[j]; };
          const double qo = first ? 0.0 : ws.q[c];
          q = row_offdiag<KE, decltype(wnb), E16>(m, a, c, dc * wc, wnb);
          if (!first) q = fma(beta, qo, q);
        } else {
          q = dc * pc;
          q = row_offdiag<KE, decltype(pnb), E16>(m, a, c, q, pnb);
        }
        if (HALO) q -= row_proc_p(m, a.bBnd, ws, first, beta, k, c, pflag);
#if LF_TAIL
        if (IDLE)
          lf_stash[i * BS + threadIdx.x] = make_double2(q, dc);
        else
#endif
          ws.q[c] = q;
        acc[0] = fma(pc, q, acc[0]);
      }
    };
#if LF_TAIL
    // Run-time trips (HBM-bound variant, one rank; ws.dynTrips > 0): the
    // last trips are handed out by a global counter in units of LF_DYN_UT
    // trips x one block run (unit u: trip row u / G, block slot u % G — sweep
    // order), so SMs that run slower take fewer.  No block-wide barrier per
    // unit: thread 0 claims units two ahead into shared-memory slots the
    // warps poll; each warp stores its unit sums per slot, and after the
    // phase the block adds a unit's 16 warp sums in warp order and stores
    // them per unit -> totals independent of which block ran which unit.
    constexpr int UT = LF_DYN_UT, MAXU = LF_DYN_MAXU;
    auto n_dyn = [&]() { return dyn ? min(ws.dynTrips, nFull) : 0; };
    auto n_units = [&]() { return ((n_dyn() + UT - 1) / UT) * (int)gridDim.x; };
    if (!piped) {
      if constexpr (dyn) if (n_dyn() > 0 && threadIdx.x == 0) {
        dynU[0] = (int)atomicAdd(ws.tickets + T_DYN, 1u);
        dynU[1] = (int)atomicAdd(ws.tickets + T_DYN, 1u);
      }
      {
        // the static trips, then the spread tail trip (i == nStat: one loop,
        // one copy of the cell body, as before the run-time trips)
        const int nStat = nFull - n_dyn();
        for (int i = 0; i <= nStat; ++i) {
          const int c = i < nStat ? cstart + i * cstep : tailC;
          if (c < 0) break;
          if constexpr (lpf) if (pfn > 0 && i < nStat) {
            if (i + LF_LPF < nStat) {
              pf_trip(i + LF_LPF, pfn);
            } else if constexpr (dyn) {
              // last static trip: the block's first claimed unit instead
              const int u0 = ((volatile int *)dynU)[0], G = gridDim.x, UD = n_units();
              if (u0 >= 0 && u0 < UD) {
                const int r0 = u0 / G, s0 = u0 - r0 * G;
#pragma unroll
                for (int jj = 0; jj < UT; ++jj) {
                  const int ii = nStat + r0 * UT + jj;
                  if (ii < nFull) pf_cb((long)ii * cstep + (long)s0 * BS + (long)(threadIdx.x & ~31u), pfn);
                }
              }
            }
          }
          cell1(c, i < nStat ? i : nFull, v1);
        }
      }
      if constexpr (dyn) if (n_dyn() > 0) {
        const int G = gridDim.x, nStat = nFull - n_dyn(), UD = n_units(), wid = threadIdx.x >> 5;
        constexpr int ut = UT;
        volatile int *vU = dynU;
        for (;;) {  // rounds of up to MAXU units (slots flushed between rounds)
          int J = 0;
          bool done = false;
          for (; J < MAXU; ++J) {
            int u;
            while ((u = vU[J]) < 0) __nanosleep(32);  // thread 0 has not claimed slot J yet
            if (u >= UD) {
              done = true;
              break;
            }
            int nxt = 0;
            if (threadIdx.x == 0 && J + 2 < MAXU) nxt = (int)atomicAdd(ws.tickets + T_DYN, 1u);
            if constexpr (lpf) if (pfn > 0 && J + 1 < MAXU) {
              const int un = vU[J + 1];  // the next unit, if claimed: its lines into L2 now
              if (un >= 0 && un < UD) {
                const int rn = un / G, sn = un - rn * G;
#pragma unroll
                for (int jj = 0; jj < ut; ++jj) {
                  const int ii = nStat + rn * ut + jj;
                  if (ii < nFull) pf_cb((long)ii * cstep + (long)sn * BS + (long)(threadIdx.x & ~31u), pfn);
                }
              }
            }
            const int row = u / G, sl = u - row * G;
            double vu[2] = {0.0, 0.0};
#pragma unroll
            for (int jj = 0; jj < ut; ++jj) {
              const int ii = nStat + row * ut + jj;
              if (ii < nFull) cell1(ii * cstep + sl * BS + (int)threadIdx.x, ii, vu);
            }
            warp_sum<2>(vu);
            if (lane == 0) {
              dynP[J][wid][0] = vu[0];
              dynP[J][wid][1] = vu[1];
            }
            if (threadIdx.x == 0 && J + 2 < MAXU) vU[J + 2] = nxt;
          }
          __syncthreads();  // every warp is past its last slot read; dynP complete
          if ((int)threadIdx.x < J) {
            const int j = threadIdx.x, u = dynU[j];
            double s0 = 0.0, s1 = 0.0;
            for (int wv = 0; wv < BS / 32; ++wv) {  // warp order: deterministic
              s0 += dynP[j][wv][0];
              s1 += dynP[j][wv][1];
            }
            ws.partialsD[u] = s0;
            ws.partialsD[UD + u] = s1;
          }
          __syncthreads();  // slots read
          if ((int)threadIdx.x < MAXU) dynU[threadIdx.x] = -1;
          if (done) break;  // (the next phase's claims follow a grid barrier)
          __syncthreads();  // reset visible before the next round's claims
          if (threadIdx.x == 0) {
            vU[0] = (int)atomicAdd(ws.tickets + T_DYN, 1u);
            vU[1] = (int)atomicAdd(ws.tickets + T_DYN, 1u);
          }
        }
      }
    }
#else
    for (int c = cstart; c < cend; c += cstep) cell1(c, 0, v1);
#endif
    LF_TSTAMP(1);
    // idle-time prefetch (LF_IDLE_PF): r and diag of phase 2's first trips
    // (phase 2 walks the trips backwards, LF_REVERSE): this block's 512-cell
    // run of trip i starts at blockIdx.x * BS + i * cstep
    auto pf1 = [&]() {
      if constexpr (LF_IDLE_PF > 0 && !IDLE && LF_TAIL && LF_REVERSE) {
        const int j = threadIdx.x;
        if (j < 2 * LF_IDLE_PF) {
          const int i = nFull - 1 - (j >> 1);
          if (i >= 0) {
            const long c0 = (long)blockIdx.x * BS + (long)i * cstep;
            l2_prefetch((j & 1) ? (const void *)(a.diag + c0) : (const void *)(ws.r + c0), BS * sizeof(double));
          }
        }
      }
    };
#if LF_TAIL
    {
      const bool dy = n_dyn() > 0;
      grid_reduce_sync<2, HALO>(v1, ws.partials, bar, ws.gsum->p1, ws.p2p LF_DBG_ARG(2 * k), pf1,
                                dy ? ws.partialsD : nullptr, dy ? n_units() : 0, dy ? ws.tickets + T_DYN : nullptr);
    }
#else
    grid_reduce_sync<2, HALO>(v1, ws.partials, bar, ws.gsum->p1, ws.p2p LF_DBG_ARG(2 * k), pf1);
#endif
    LF_TSTAMP(2);
    if (!cont) break;
    // ---- phase 2: singularity, alpha, r -= alpha q, w = r/diag, sums
    if (threadIdx.x == 0) {
      const double pq = __ldcg(&ws.gsum->p1[0]);
      st.singular = fabs(pq) / st.nf < 1e-300;
      if (!st.singular) {
        st.alphaPrev = st.alpha;
        st.alpha = st.wArA / pq;
      }
    }
    __syncthreads();
    if (st.singular) break;
    const double alpha2 = st.alpha;
    double v2[2] = {0.0, 0.0};
    {
      constexpr int U = LF_P2P_UNROLL;  // cells per trip, loads issued first
      // U cells (c < 0: none): all loads first, then r, w and the sums
      auto p2cells = [&](const int (&cs)[U]) {
        double q[U], r[U], d[U];
        int pf[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int c = cs[u];
          const bool ok = c >= 0;
          pf[u] = (HALO && ok) ? (int)has_proc(m, c) : 0;
          q[u] = ok ? ws.q[c] : 0.0;
          r[u] = ok ? ws.r[c] : 0.0;
          d[u] = ok ? (w88 == 2 ? rDg[c] : a.diag[c]) : 1.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int c = cs[u];
          if (c >= 0) {
            const double rn = fma(-alpha2, q[u], r[u]);
            const double wc = (w88 == 2 ? d[u] : 1.0 / d[u]) * rn;
            ws.r[c] = rn;
            if (!w88) ws.w[c] = wc;
            if (HALO && ws.p2p.P > 0) push_halo<HALO_W>(m, ws.p2p, c, wc, pf[u]);
            v2[0] += fabs(rn);
            v2[1] = fma(wc, rn, v2[1]);
          }
        }
      };
#if LF_TAIL
      if (IDLE) {
        // {q, diag} from the stash, r streamed: all trips' loads issued first
        constexpr int T = LF_STASH_TRIPS;
        double rv[T];
#pragma unroll
        for (int i = 0; i < T; ++i) {
          const int c = i < nFull ? cstart + i * cstep : (i == nFull ? tailC : -1);
          rv[i] = (i <= nFull && c >= 0) ? ws.r[c] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < T; ++i) {
          const int c = i < nFull ? cstart + i * cstep : (i == nFull ? tailC : -1);
          if (i <= nFull && c >= 0) {
            const double2 qd = lf_stash[i * BS + threadIdx.x];
            const double rn = fma(-alpha2, qd.x, rv[i]);
            const double wc = (1.0 / qd.y) * rn;
            ws.r[c] = rn;
            ws.w[c] = wc;
            if (HALO && ws.p2p.P > 0) push_halo<HALO_W>(m, ws.p2p, c, wc);
            v2[0] += fabs(rn);
            v2[1] = fma(wc, rn, v2[1]);
          }
        }
      } else {
        // LF_REVERSE: phase 2 sweeps the trips backwards, so it starts on the
        // cells phase 1 wrote last (q still in L2) and ends on the ones the
        // next phase 1 reads first (w, r still in L2)
        for (int i0 = 0; i0 <= nFull; i0 += U) {
          int cs[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int ii = LF_REVERSE ? nFull - (i0 + u) : i0 + u;
            cs[u] = (ii >= 0 && ii < nFull) ? cstart + ii * cstep : (ii == nFull ? tailC : -1);
          }
          if constexpr (lpf && LF_LPF2 > 0 && LF_REVERSE) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int ii = nFull - (i0 + u + U * LF_LPF2);
              if (ii >= 0 && lane < 9 && pfn > 0) {
                const long cb = (long)wbase + (long)ii * cstep;
                l2_pf_line(pfTab[48 + lane].p + (cb << pfTab[48 + lane].sh));
              }
            }
          }
          p2cells(cs);
        }
      }
#else
      for (int c0 = cstart; c0 < cend; c0 += cstep * U) {
        int cs[U];
#pragma unroll
        for (int u = 0; u < U; ++u) cs[u] = c0 + u * cstep < cend ? c0 + u * cstep : -1;
        p2cells(cs);
      }
#endif
    }
    LF_TSTAMP(3);
    // idleF: psi += alpha_k p_k for this thread's cells (p_k written by this
    // thread in phase 1) while the block waits for beta — fills the barrier
    // latency and takes the psi stream out of phase 1, at the price of
    // re-reading p (8n).  OpenFOAM's order is kept (the update follows the
    // singularity check of the same iteration).
    psiSum = 0.0;
    auto flush = [&]() {
      if constexpr (LF_IDLE_PF > 0 && !IDLE && LF_TAIL && KE > 0 && !E16) {
        // the next phase 1's first trips: w, p (next p_old), diag, psi and the ELL slices
        constexpr int NA = 4 + 3 * KE;
        const int j = threadIdx.x;
        if (j < NA * LF_IDLE_PF) {
          const int i = j / NA, f = j % NA;
          if (i < nFull) {
            const long c0 = (long)blockIdx.x * BS + (long)i * cstep;
            const long ld = m.ldE;
            const void *pa;
            unsigned bytes = BS * sizeof(double);
            if (f == 0) pa = ws.w + c0;
            else if (f == 1) pa = pnew + c0;
            else if (f == 2) pa = a.diag + c0;
            else if (f == 3) pa = psi + c0;
            else if (f < 4 + KE) pa = a.upperE + (f - 4) * ld + c0;
            else if (f < 4 + 2 * KE) { pa = m.loE + (f - 4 - KE) * ld + c0; bytes = BS * sizeof(int); }
            else { pa = m.nbrE + (f - 4 - 2 * KE) * ld + c0; bytes = BS * sizeof(int); }
            l2_prefetch(pa, bytes);
          }
        }
      }
      if (!idleF) return;
#if LF_TAIL
      for (int i = 0; i <= nFull; ++i) {
        const int c = i < nFull ? cstart + i * cstep : tailC;
        if (c < 0) break;
#else
      for (int c = cstart; c < cend; c += cstep) {
#endif
        const double ps = fma(alpha2, pnew[c], psi[c]);
        psi[c] = ps;
        psiSum += ps;
      }
    };
    grid_reduce_sync<2, HALO>(v2, ws.partials, bar, ws.gsum->p2, ws.p2p LF_DBG_ARG(2 * k + 1), flush);
    LF_TSTAMP(4);
    if (threadIdx.x == 0) ++st.k;
  }
  const int k = st.k;
  if (psi2 && st.singular && (k & 1)) {
    // singular break after a phase 1 that deferred alpha_{k-1} p_{k-1}: apply
    // it (OpenFOAM's psi at the break) and re-form sum(psi) for the next setup
    const double *__restrict__ pold = ws.p[0];  // odd k: p_{k-1} in p[0]
    const double alpha = st.alpha;
    double vs[2] = {0.0, 0.0};
#if LF_TAIL
    for (int i = 0; i <= nFull; ++i) {
      const int c = i < nFull ? cstart + i * cstep : tailC;
      if (c < 0) break;
#else
    for (int c = cstart; c < cend; c += cstep) {
#endif
      const double ps = fma(alpha, pold[c], psi[c]);
      psi[c] = ps;
      vs[1] += ps;
    }
    grid_reduce_sync<2, HALO>(vs, ws.partials, bar, ws.gsum->p1, ws.p2p LF_DBG_ARG(LF_DBG_N - 1));
  }
#if LF_TIMING
  if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x / 2) && k > 0)
    printf("LF_TIMING block %d iters %d: phase1 %.2f us, bar1 %.2f us, phase2 %.2f us, bar2 %.2f us\n",
           blockIdx.x, k, tacc[0] / 1e3 / k, tacc[1] / 1e3 / k, tacc[2] / 1e3 / k, tacc[3] / 1e3 / k);
  if (threadIdx.x == 0 && blockIdx.x == 0 && k > 4) {
    const int G = min((int)gridDim.x, LF_DBG_G), NB = min(LF_DBG_N, 2 * k - 2);
    double acc[2][5] = {{0, 0, 0, 0, 0}, {0, 0, 0, 0, 0}};
    int cnt[2] = {0, 0};
    for (int i = 2; i < NB; ++i) {
      unsigned long long amin = ~0ull, amax = 0, wmax = 0, wsum = 0, asum = 0;
      for (int b = 0; b < G; ++b) { const unsigned long long a = __ldcg(&g_dbg_arr[i][b]); amin = a < amin ? a : amin; }
      int nw = 0;
      const int last = __ldcg(&g_dbg_last[i]);
      for (int b = 0; b < G; ++b) {
        const unsigned long long a = __ldcg(&g_dbg_arr[i][b]);
        amin = a < amin ? a : amin;
        amax = a > amax ? a : amax;
        asum += a - amin;
        if (b != last) {
          const unsigned long long w = __ldcg(&g_dbg_wake[i][b]);
          wmax = w > wmax ? w : wmax;
          wsum += w;
          ++nw;
        }
      }
      const unsigned long long rel = __ldcg(&g_dbg_rel[i]);
      const int j = i & 1;
      acc[j][0] += (double)(amax - amin);
      acc[j][1] += (double)(rel - amax);
      acc[j][2] += (double)(wmax - rel);
      acc[j][3] += nw ? (double)(wsum / nw - rel) : 0.0;
      acc[j][4] += (double)(rel - amin) - (double)asum / G;
      if (i == 20 || i == 21 || i == 40) {
        if (i == 20) {
          printf("LF_SMID:");
          for (int b = 0; b < G; ++b) printf(" %d", __ldcg(&g_dbg_smid[b]));
          printf("\n");
        }
        printf("LF_ARRIVALS %d:", i);
        for (int b = 0; b < G; ++b) printf(" %.1f", (double)(__ldcg(&g_dbg_arr[i][b]) - amin) / 1e3);
        printf("\n");
      }
      ++cnt[j];
    }
    for (int j = 0; j < 2; ++j)
      if (cnt[j])
        printf("LF_BARRIER %d: arrival spread %.2f us, last-arrival->release %.2f us, "
               "release->last wake %.2f us (mean wake %.2f us), mean arrival->release %.2f us\n", j + 1,
               acc[j][0] / 1e3 / cnt[j], acc[j][1] / 1e3 / cnt[j], acc[j][2] / 1e3 / cnt[j],
               acc[j][3] / 1e3 / cnt[j], acc[j][4] / 1e3 / cnt[j]);
  }
#endif
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctl->it = k;
    ctl->stop = 1;
    ctl->singular = st.singular;
    ctl->converged = conv(st.finRes, st.initRes, ctl) ? 1 : 0;
    ctl->normFactor = st.nf;
    ctl->initRes = st.initRes;
    ctl->finRes = st.finRes;
    ctl->wArA = st.wArA;
    ctl->alpha = st.alpha;
  }
}

// co-resident grid for every persistent variant that may be launched on a
// mesh (any row layout: the full-row rows are chosen after this call)
template <int KE, bool E16 = false>
static void persistent_occupancy(int &best) {
  int nb = 0;
  for (const void *fn : {(const void *)k_pcg_persistent<KE, false, false, E16>,
                         (const void *)k_pcg_persistent<KE, true, false, E16>}) {
    if (LF_CPASYNC)
      LF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CPA_BYTES));
    LF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, BS, LF_CPASYNC ? CPA_BYTES : 0));
    best = std::min(best, nb);
  }
  // the L2-resident variants with the shared-memory stash
  for (const void *fi : {(const void *)k_pcg_persistent<KE, false, true, E16>,
                         (const void *)k_pcg_persistent<KE, true, true, E16>}) {
    LF_CUDA(cudaFuncSetAttribute(fi, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)stash_bytes()));
    LF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fi, BS, stash_bytes()));
    best = std::min(best, nb);
  }
}

int persistent_grid(int device, int K) {
  int sms = 0;
  LF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  int best = 1 << 30;
  if (K == 4) {
    persistent_occupancy<4>(best);
    persistent_occupancy<4, true>(best);
  } else if (K > 0) {
    persistent_occupancy<3>(best);
    persistent_occupancy<3, true>(best);
  }
  else {
    persistent_occupancy<0>(best);
    persistent_occupancy<-6>(best);
    persistent_occupancy<-8>(best);
  }
  return sms * (best < 1 ? 1 : best);
}

template <bool HALO, bool IDLE = false>
static const void *persistent_fn(const MeshDev &m) {
  const bool e16 = m.codeE != nullptr;
  return (!LF_NO_ELL && m.K == 4) ? (e16 ? (const void *)k_pcg_persistent<4, HALO, IDLE, true>
                                         : (const void *)k_pcg_persistent<4, HALO, IDLE>)
         : (!LF_NO_ELL && m.K > 0) ? (e16 ? (const void *)k_pcg_persistent<3, HALO, IDLE, true>
                                          : (const void *)k_pcg_persistent<3, HALO, IDLE>)
         : m.KS == 6               ? (const void *)k_pcg_persistent<-6, HALO, IDLE>
         : m.KS == 8               ? (const void *)k_pcg_persistent<-8, HALO, IDLE>
                                   : (const void *)k_pcg_persistent<0, HALO, IDLE>;
}

void launch_pcg_persistent(cudaStream_t s, int grid, const MeshDev &m, const LduDev &a,
                           const Workspace &ws, unsigned *bar) {
  const bool halo = m.hasProc || ws.p2p.P > 0;
  void *args[] = {(void *)&m, (void *)&a, (void *)&ws, (void *)&bar};
  // L2-resident variant (stash + psi update in the barrier wait) on either path
  const bool idle = LF_IDLE_FLUSH && ws.idleFlush;
  const void *fn = halo ? (idle ? persistent_fn<true, true>(m) : persistent_fn<true>(m))
                        : (idle ? persistent_fn<false, true>(m) : persistent_fn<false>(m));
  LF_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(BS), args,
                                      idle ? stash_fit(m.n, grid, sizeof(double2)) : (LF_CPASYNC ? CPA_BYTES : 0), s));
}

// ------------------------------------------------------------------ Amul
template <int KE>
__global__ void __launch_bounds__(BS, LF_MINB_G)
    k_amul(MeshDev m, LduDev a, const double *__restrict__ halo, const double *__restrict__ x,
           double *__restrict__ y) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < m.n; c += gridDim.x * blockDim.x) {
    double acc = a.diag[c] * x[c];
    acc = row_offdiag<KE>(m, a, c, acc, [&](int j) { return x[j]; });
    y[c] = acc - row_proc(m, a.bBnd, halo, c);
  }
}

void launch_amul(cudaStream_t s, const Launch &L, const MeshDev &m, const LduDev &a,
                 const double *halo, const double *x, double *y) {
  LF_DISPATCH_KE(m, k_amul, <<<L.grid, BS, 0, s>>>(m, a, halo, x, y));
}

// ------------------------------------------------------ solver controls
__global__ void k_set_ctl(PcgCtl *ctl, PcgCtl v) { *ctl = v; }

void launch_set_ctl(cudaStream_t s, PcgCtl *ctl, const PcgCtl &value) { k_set_ctl<<<1, 1, 0, s>>>(ctl, value); }

// ------------------------------------------------------------ halo packs
__global__ void k_pack_x(int32_t ns, const int32_t *__restrict__ cells, const double *__restrict__ x,
                         double *__restrict__ buf) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += gridDim.x * blockDim.x)
    buf[i] = x[cells[i]];
}

void launch_pack_x(cudaStream_t s, int32_t ns, const int32_t *cells, const double *x, double *buf) {
  if (ns <= 0) return;
  k_pack_x<<<(ns + BS - 1) / BS, BS, 0, s>>>(ns, cells, x, buf);
}


// ------------------------------------------------------------ utilities
static int grid_for(int64_t n) {
  int64_t g = (n + BS - 1) / BS;
  if (g < 1) g = 1;
  if (g > 65535L * 8) g = 65535L * 8;
  return (int)g;
}

__global__ void k_permute(int32_t n, const int32_t *__restrict__ idx, const double *__restrict__ in,
                          double *__restrict__ out, bool scatter) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (scatter)
      out[idx[i]] = in[i];
    else
      out[i] = in[idx[i]];
  }
}

void launch_permute(cudaStream_t s, int32_t n, const int32_t *idx, const double *in, double *out,
                    bool scatter) {
  if (n <= 0) return;
  k_permute<<<grid_for(n), BS, 0, s>>>(n, idx, in, out, scatter);
}

__global__ void k_gather_f64(int64_t n, const int32_t *__restrict__ idx, const double *__restrict__ in,
                             double *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[idx[i]];
}

void launch_gather_f64(cudaStream_t s, int64_t n, const int32_t *idx, const double *in, double *out) {
  if (n <= 0) return;
  k_gather_f64<<<grid_for(n), BS, 0, s>>>(n, idx, in, out);
}

__global__ void k_gather_i32(int64_t n, const int32_t *__restrict__ idx, const int32_t *__restrict__ in,
                             int32_t *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[idx[i]];
}

void launch_gather_i32(cudaStream_t s, int64_t n, const int32_t *idx, const int32_t *in, int32_t *out) {
  if (n <= 0) return;
  k_gather_i32<<<grid_for(n), BS, 0, s>>>(n, idx, in, out);
}

__global__ void k_iota(int32_t *a, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = (int32_t)i;
}

void launch_iota(cudaStream_t s, int32_t *a, int64_t n) {
  if (n <= 0) return;
  k_iota<<<grid_for(n), BS, 0, s>>>(a, n);
}

// starts[g] = first position of key >= g in a sorted key list (n+1 entries,
// total appended — reading A14).  Every starts[] entry is written by exactly
// one thread: thread f covers groups (sorted[f-1], sorted[f]].  This is the
// exclusive scan of the per-group counts of P:419-427 without the sentinel
// sort (any equivalent primitive, A17).
__global__ void k_starts(const int32_t *__restrict__ sorted, int64_t m, int32_t n, int32_t *starts) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f <= m; f += (int64_t)gridDim.x * blockDim.x) {
    const int32_t prev = f > 0 ? sorted[f - 1] : -1;
    const int32_t cur = f < m ? sorted[f] : n;
    for (int32_t g = prev + 1; g <= cur; ++g) starts[g] = (int32_t)f;
  }
}

void launch_starts_from_sorted(cudaStream_t s, const int32_t *sorted, int64_t m, int32_t n,
                               int32_t *starts) {
  k_starts<<<grid_for(m + 1), BS, 0, s>>>(sorted, m, n, starts);
}

__global__ void k_make_keys(const int32_t *__restrict__ a, const int32_t *__restrict__ b, int64_t m,
                            uint64_t *keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t x = (uint32_t)a[i], y = (uint32_t)b[i];
    const uint32_t lo = x < y ? x : y, hi = x < y ? y : x;
    keys[i] = ((uint64_t)lo << 32) | hi;
  }
}

void launch_make_keys(cudaStream_t s, const int32_t *a, const int32_t *b, int64_t m, uint64_t *keys) {
  if (m <= 0) return;
  k_make_keys<<<grid_for(m), BS, 0, s>>>(a, b, m, keys);
}

__global__ void k_split_keys(const uint64_t *__restrict__ keys, int64_t m, int32_t *lo, int32_t *hi) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    lo[i] = (int32_t)(keys[i] >> 32);
    hi[i] = (int32_t)(keys[i] & 0xffffffffu);
  }
}

void launch_split_keys(cudaStream_t s, const uint64_t *keys, int64_t m, int32_t *lo, int32_t *hi) {
  if (m <= 0) return;
  k_split_keys<<<grid_for(m), BS, 0, s>>>(keys, m, lo, hi);
}

// ELL slices from the CSR lists (see the header comment).  Padding: -1.
__global__ void k_build_ell(MeshDev m, const int32_t *__restrict__ owner, int32_t K, int32_t *nbrE,
                            int32_t *loE) {
  const int n = m.n, ld = m.ldE;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    const int o0 = m.ownerStart[c], o1 = m.ownerStart[c + 1];
    const int l0 = m.losortStart[c], l1 = m.losortStart[c + 1];
    for (int k = 0; k < K; ++k) {
      nbrE[k * ld + c] = o0 + k < o1 ? m.nbr[o0 + k] : -1;
      int packed = -1;
      if (l0 + k < l1) {
        const int f = m.losort[l0 + k];
        const int oc = owner[f];
        packed = ((f - m.ownerStart[oc]) << ELL_SHIFT) | oc;
      }
      loE[k * ld + c] = packed;
    }
  }
}

void launch_build_ell(cudaStream_t s, const MeshDev &m, const int32_t *owner, int32_t K, int32_t *nbrE,
                      int32_t *loE) {
  k_build_ell<<<grid_for(m.n), BS, 0, s>>>(m, owner, K, nbrE, loE);
}

// upper (face order) from the ELL copy: face ownerStart[c] + k is slot k of c
__global__ void k_upper_from_ell(MeshDev m, LduDev a) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < m.n; c += gridDim.x * blockDim.x) {
    const int o0 = m.ownerStart[c], o1 = m.ownerStart[c + 1];
    for (int i = o0; i < o1; ++i) a.upper[i] = a.upperE[(i - o0) * m.ldE + c];
  }
}

void launch_upper_from_ell(cudaStream_t s, const MeshDev &m, const LduDev &a) {
  k_upper_from_ell<<<grid_for(m.n), BS, 0, s>>>(m, a);
}

// ------------------------------------------ uniform 32-cell label groups
// One warp per (slot, group): if every cell of the group has the slot with
// the same offset nbr - c (owner side: the same owner slot kk and c - owner)
// the group's labels are implied by {offset}; all empty -> 0; else -1.
__global__ void k_build_uni(MeshDev m, int2 *__restrict__ uniE) {
  const int lane = threadIdx.x & 31, ld = m.ldE;
  const long nw = (long)m.K * m.ngE;
  for (long wi = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; wi < nw;
       wi += ((long)gridDim.x * blockDim.x) >> 5) {
    const int k = (int)(wi / m.ngE), g = (int)(wi % m.ngE), c = g * 32 + lane;
    const bool in = c < m.n;
    const int nb = in ? m.nbrE[k * ld + c] : 0, lo = in ? m.loE[k * ld + c] : 0;
    const unsigned inMask = __ballot_sync(FULL, in);
    // neighbour side
    const int vn = nb >= 0 ? nb - c : -1;
    const unsigned anyN = __ballot_sync(FULL, in && nb >= 0), allN = __ballot_sync(FULL, !in || nb >= 0);
    const int v0n = __shfl_sync(FULL, vn, 0);
    const bool sameN = __all_sync(FULL, !in || vn == v0n);
    int x = -1;
    if (anyN == 0) x = 0;
    else if (allN == FULL && sameN && v0n > 0) x = v0n;
    // owner side (packed kk << 29 | owner)
    const int vl = lo >= 0 ? ((lo & ~ELL_MASK) | (c - (lo & ELL_MASK))) : -1;
    const unsigned anyL = __ballot_sync(FULL, in && lo >= 0), allL = __ballot_sync(FULL, !in || lo >= 0);
    const int v0l = __shfl_sync(FULL, vl, 0);
    const bool sameL = __all_sync(FULL, !in || vl == v0l);
    int y = -1;
    if (anyL == 0) y = 0;
    else if (allL == FULL && sameL && (v0l & ELL_MASK) > 0) y = v0l;
    (void)inMask;
    if (lane == 0) uniE[(long)k * m.ngE + g] = make_int2(x, y);
  }
}

void launch_build_uni(cudaStream_t s, const MeshDev &m, int2 *uniE) {
  k_build_uni<<<grid_for((int64_t)m.K * m.ngE * 32), BS, 0, s>>>(m, uniE);
}

// ------------------------------------------------ compressed ELL labels
// The solve is HBM-bound and the two int32 labels of an ELL slot are a third
// of its face bytes.  Within 32 consecutive cells (one warp of a grid-stride
// trip) the label offsets nbr - c and c - owner of a slot take few distinct
// values on any locally numbered mesh (+1, +N, +N^2 on a block mesh), so each
// slot stores them as 16-bit codes relative to the group's most frequent
// offset (one u32 per slot and cell: low half owner side, high half
// neighbour side = 2 bits of owner-slot kk + 14-bit offset):
//   nb:  0xFFFF none, 0xFFFE escape (label in nbrE), else c + off.x + d - 0x8000
//   lo:  0xFFFF none, 0xFFFE escape (packed in loE),
//        else kk = d >> 14, owner = c - off.y - (d & 0x3FFF) + 0x2000
// 12 B per face slot instead of 16 B; the escape arrays are touched only by
// the (rare) lanes that need them.  Decoded labels are bitwise the int32 ones.
__device__ __forceinline__ int warp_mode(int v, bool valid) {
  // most frequent valid value among the 32 lanes (ties: lowest lane); 0 if none
  const unsigned same = __match_any_sync(FULL, valid ? v : INT_MIN);
  const int lane = threadIdx.x & 31;
  int key = valid ? (__popc(same) << 5) | (31 - lane) : -1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) key = max(key, __shfl_xor_sync(FULL, key, o));
  const int src = key < 0 ? 0 : 31 - (key & 31);
  const int mv = __shfl_sync(FULL, v, src);
  return key < 0 ? 0 : mv;
}

__global__ void k_build_ell16(MeshDev m, uint32_t *__restrict__ codeE, int2 *__restrict__ offE,
                              int32_t *nEsc) {
  const int lane = threadIdx.x & 31, ld = m.ldE;
  const long nw = (long)m.K * m.ngE;
  int esc = 0;
  for (long wi = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; wi < nw;
       wi += ((long)gridDim.x * blockDim.x) >> 5) {
    const int k = (int)(wi / m.ngE), g = (int)(wi % m.ngE), c = g * 32 + lane;
    const bool in = c < m.n;
    const int nb = in ? m.nbrE[k * ld + c] : -1, lo = in ? m.loE[k * ld + c] : -1;
    const int vn = nb - c, vl = c - (lo & ELL_MASK);
    const int on = warp_mode(vn, nb >= 0), ol = warp_mode(vl, lo >= 0);
    unsigned cn = 0xFFFFu, cl = 0xFFFFu;
    if (nb >= 0) {
      const long d = (long)vn - on + 0x8000;
      cn = (d >= 0 && d <= 0xFFFD) ? (unsigned)d : 0xFFFEu;
    }
    if (lo >= 0) {
      const long d = (long)vl - ol + 0x2000;
      const unsigned kk = (unsigned)lo >> ELL_SHIFT;
      const unsigned code = (unsigned)(kk << 14) | (unsigned)d;
      cl = (d >= 0 && d <= 0x3FFF && code < 0xFFFEu) ? code : 0xFFFEu;
    }
    esc += (cn == 0xFFFEu) + (cl == 0xFFFEu);
    if (in) codeE[k * ld + c] = cn | (cl << 16);
    if (lane == 0) offE[(long)k * m.ngE + g] = make_int2(on, ol);
  }
  if (esc) atomicAdd(nEsc, esc);  // integer statistic only
}

void launch_build_ell16(cudaStream_t s, const MeshDev &m, uint32_t *codeE, int2 *offE, int32_t *nEsc) {
  LF_CUDA(cudaMemsetAsync(nEsc, 0, sizeof(int32_t), s));
  const long threads = (long)m.K * m.ngE * 32;
  k_build_ell16<<<grid_for(threads), BS, 0, s>>>(m, codeE, offE, nEsc);
}

// ------------------------------------------------------------- CUB sorts
// Stable LSD radix sort (the paper's "std::sort" of P:409, made stable per
// reading A13).  In-place interface over a scratch double buffer.
template <class Key>
static void sort_pairs(cudaStream_t s, Key *keys, int32_t *vals, int64_t m, int end_bit) {
  if (m <= 1) return;
  Key *k2 = nullptr;
  int32_t *v2 = nullptr;
  void *tmp = nullptr;
  size_t tb = 0;
  LF_CUDA(cudaMallocAsync(&k2, sizeof(Key) * m, s));
  LF_CUDA(cudaMallocAsync(&v2, sizeof(int32_t) * m, s));
  cub::DoubleBuffer<Key> kb(keys, k2);
  cub::DoubleBuffer<int32_t> vb(vals, v2);
  LF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kb, vb, m, 0, end_bit, s));
  LF_CUDA(cudaMallocAsync(&tmp, tb, s));
  LF_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, kb, vb, m, 0, end_bit, s));
  if (kb.Current() != keys) LF_CUDA(cudaMemcpyAsync(keys, kb.Current(), sizeof(Key) * m, cudaMemcpyDeviceToDevice, s));
  if (vb.Current() != vals) LF_CUDA(cudaMemcpyAsync(vals, vb.Current(), sizeof(int32_t) * m, cudaMemcpyDeviceToDevice, s));
  LF_CUDA(cudaFreeAsync(tmp, s));
  LF_CUDA(cudaFreeAsync(k2, s));
  LF_CUDA(cudaFreeAsync(v2, s));
}

void sort_pairs_u64(cudaStream_t s, uint64_t *keys, int32_t *vals, int64_t m, int end_bit) {
  sort_pairs<uint64_t>(s, keys, vals, m, end_bit);
}
void sort_pairs_i32(cudaStream_t s, int32_t *keys, int32_t *vals, int64_t m, int end_bit) {
  sort_pairs<int32_t>(s, keys, vals, m, end_bit);
}

// ------------------------------------- lane-distributed L2 prefetch sets
// A list of (array, point) entries — first / last byte of an int array's
// 32-cell run, first / middle / last byte of a double array's — so that one
// warp covers every line of its run with one or two prefetch instructions
// per lane (the L2 prefetch of k_pcg_persistent, for the other solves).
struct PfSet {
  PfEnt e[48];
  int n;
  __device__ void clear() { n = 0; }
  __device__ void addI(const int32_t *b) {
    e[n++] = {(const char *)b, 2};
    e[n++] = {(const char *)b + 124, 2};
  }
  __device__ void addD(const double *b) {
    e[n++] = {(const char *)b, 3};
    e[n++] = {(const char *)b + 128, 3};
    e[n++] = {(const char *)b + 248, 3};
  }
};
// prefetch the warp's run of 32 cells starting at cb (every lane passes the
// same cb)
__device__ __forceinline__ void pf_run(const PfSet &s, long cb) {
  const int lane = threadIdx.x & 31, n = s.n;
  if (lane < n) l2_pf_line(s.e[lane].p + (cb << s.e[lane].sh));
  if (lane + 32 < n) l2_pf_line(s.e[lane + 32].p + (cb << s.e[lane + 32].sh));
}

// ----------------------------------------------------- DIC preconditioner
#include "dic.cuh"

// ---------------------------------------------------- GAMG preconditioner
#include "gamg.cuh"

// ------------------------------------------------------------- occupancy
int occupancy_grid(int kernel_id, int device) {
  int sms = 0, nb = 0;
  LF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  const void *fn = nullptr;
  switch (kernel_id) {
    case 0: fn = (const void *)k_assemble<true>; break;
    case 1: fn = (const void *)k_phase1<3>; break;
    case 2: fn = (const void *)k_phase2; break;
    case 3: fn = (const void *)k_amul<3>; break;
    case 4: fn = (const void *)k_pcg_setup<3>; break;
    case 5: fn = (const void *)k_sum; break;
    default: fn = (const void *)k_assemble<false>; break;
  }
  LF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, BS, 0));
  if (nb < 1) nb = 1;
  return sms * nb;
}

}  // namespace lf
