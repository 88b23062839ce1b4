// Peer-memory transport (SURVEY.md §8(e) "Halo, option A: P2P").
//
// Every rank exports ONE cudaMalloc block per mesh with cudaIpcGetMemHandle:
//   [mailbox flags | mailbox values | recvT[2] | recvW | recvX[3]]
// and maps every other rank's block with cudaIpcOpenMemHandle (over NVLink
// between GPUs; the same physical memory for ranks sharing a GPU).  The
// kernels then
//   * store w (PCG) / T (assembly) of their processor-face cells straight
//     into the neighbour's recvW / recvT (fused into phase 2 / the sum kernel),
//   * exchange the PCG sums through the mailboxes in the last block of every
//     reduction (system-scope release/acquire, rank-ordered sum),
// so an iteration has no host-side communication step and the whole solve
// can run as one persistent launch per rank.
#include <algorithm>

#include "host.h"

namespace lf {

namespace {
constexpr int32_t kMagic = 0x4c463250;  // "LF2P"
constexpr int kMaxSeg = 32;
struct Handle {
  cudaIpcMemHandle_t ipc;  // 64 bytes
  int32_t magic, rank, nranks, n_cells, nproc, nseg;
  int64_t offFlags, offVals, offRecvT, offRecvW, offRecvX;
  struct Seg {
    int32_t peer, offset, count, pad;
  } seg[kMaxSeg];
};
static_assert(sizeof(Handle) <= LF_P2P_HANDLE_BYTES, "handle too large");
}  // namespace

void p2p_init(lf_context *ctx, int nranks, int rank) {
  LF_REQUIRE(nranks >= 1 && nranks <= LF_MAXP, "nranks must be in [1, 16]");
  LF_REQUIRE(rank >= 0 && rank < nranks, "rank out of range");
  LF_REQUIRE(ctx->comm == nullptr, "context already uses NCCL");
  ctx->p2p = true;
  ctx->nranks = nranks;
  ctx->rank = rank;
}

void p2p_export(lf_mesh *M, void *out) {
  LF_REQUIRE(M->ctx->p2p, "lf_p2p_init the context before mesh_create");
  LF_REQUIRE((int)M->segs.size() <= kMaxSeg, "too many processor patches for the P2P handle");
  Handle h;
  std::memset(&h, 0, sizeof(h));
  LF_CUDA(cudaSetDevice(M->ctx->device));
  LF_CUDA(cudaIpcGetMemHandle(&h.ipc, M->p2pBlock));
  h.magic = kMagic;
  h.rank = M->ctx->rank;
  h.nranks = M->ctx->nranks;
  h.n_cells = M->n;
  h.nproc = M->nproc;
  h.nseg = (int32_t)M->segs.size();
  h.offFlags = (int64_t)M->offFlags;
  h.offVals = (int64_t)M->offVals;
  h.offRecvT = (int64_t)M->offRecvT;
  h.offRecvW = (int64_t)M->offRecvW;
  h.offRecvX = (int64_t)M->offRecvX;
  for (int g = 0; g < h.nseg; ++g) h.seg[g] = {M->segs[g].peer, M->segs[g].offset, M->segs[g].count, 0};
  std::memset(out, 0, LF_P2P_HANDLE_BYTES);
  std::memcpy(out, &h, sizeof(h));
}

void p2p_connect(lf_mesh *M, int nranks, int rank, const void *handles) {
  lf_context *ctx = M->ctx;
  LF_REQUIRE(ctx->p2p && nranks == ctx->nranks && rank == ctx->rank,
             "lf_p2p_connect: nranks/rank differ from lf_p2p_init");
  LF_REQUIRE(!M->p2pConnected, "mesh already connected");
  std::vector<Handle> H(nranks);
  for (int q = 0; q < nranks; ++q) {
    std::memcpy(&H[q], static_cast<const char *>(handles) + (size_t)q * LF_P2P_HANDLE_BYTES, sizeof(Handle));
    LF_REQUIRE(H[q].magic == kMagic && H[q].rank == q && H[q].nranks == nranks,
               "lf_p2p_connect: handle " + std::to_string(q) + " is not rank " + std::to_string(q) + "'s export");
  }
  cudaStream_t s = ctx->stream;
  LF_CUDA(cudaSetDevice(ctx->device));
  std::vector<char *> base(nranks, nullptr);
  for (int q = 0; q < nranks; ++q) {
    if (q == rank) {
      base[q] = M->p2pBlock;
    } else {
      void *p = nullptr;
      LF_CUDA(cudaIpcOpenMemHandle(&p, H[q].ipc, cudaIpcMemLazyEnablePeerAccess));
      M->ipcOpened.push_back(p);
      base[q] = static_cast<char *>(p);
    }
  }
  P2PDev &P = M->ws.p2p;
  std::memset(&P, 0, sizeof(P));
  for (int q = 0; q < nranks; ++q) {
    P.flags[q] = reinterpret_cast<unsigned *>(base[q] + H[q].offFlags);
    P.vals[q] = reinterpret_cast<double *>(base[q] + H[q].offVals);
  }
  // destination of every segment: the matching segment of the neighbour's
  // halo towards us (i-th patch to s <-> s's i-th patch to us), or the
  // partner segment of a self pair — one base pointer per segment (and per
  // parity of the double-buffered recvT); a slot adds its offset in the segment
  LF_REQUIRE((int)M->segs.size() <= LF_MAXSEG,
             "more than " + std::to_string(LF_MAXSEG) + " processor patches on one rank");
  std::vector<int> used(nranks, 0);
  P.nseg = (int32_t)M->segs.size();
  P.tPar = 0;
  for (size_t g = 0; g < M->segs.size(); ++g) {
    const HaloSeg &sg = M->segs[g];
    LF_REQUIRE(g == 0 ? sg.offset == 0 : sg.offset == M->segs[g - 1].offset + M->segs[g - 1].count,
               "processor segments must tile the send slots in order");
    int32_t off, rn;
    char *b;
    int64_t oT, oW, oX;
    if (sg.peer == rank) {
      LF_REQUIRE(sg.partner >= 0, "unpaired self processor patch");
      off = M->segs[sg.partner].offset;
      b = base[rank];
      oT = (int64_t)M->offRecvT;
      oW = (int64_t)M->offRecvW;
      oX = (int64_t)M->offRecvX;
      rn = M->nproc;
    } else {
      const Handle &hs = H[sg.peer];
      int found = -1, k = 0;
      for (int j = 0; j < hs.nseg; ++j)
        if (hs.seg[j].peer == rank && k++ == used[sg.peer]) {
          found = j;
          break;
        }
      LF_REQUIRE(found >= 0, "rank " + std::to_string(sg.peer) + " has no processor patch towards rank " +
                                 std::to_string(rank));
      LF_REQUIRE(hs.seg[found].count == sg.count, "processor patch sizes differ between ranks " +
                                                      std::to_string(rank) + " and " + std::to_string(sg.peer));
      ++used[sg.peer];
      off = hs.seg[found].offset;
      b = base[sg.peer];
      oT = hs.offRecvT;
      oW = hs.offRecvW;
      oX = hs.offRecvX;
      rn = hs.nproc;
    }
    P.segBeg[g] = sg.offset;
    P.dstW[g] = reinterpret_cast<double *>(b + oW) + off;
    P.dstT[0][g] = reinterpret_cast<double *>(b + oT) + off;
    P.dstT[1][g] = reinterpret_cast<double *>(b + oT) + rn + off;  // parity-1 half of its recvT
    P.dstX[g] = reinterpret_cast<double *>(b + oX) + off;             // component k at + k * rn
    P.xStr[g] = rn;
  }
  P.segBeg[P.nseg] = M->nproc;
  P.seq = M->arena.alloc<unsigned>(1);
  LF_CUDA(cudaMemsetAsync(P.seq, 0, sizeof(unsigned), s));
  P.P = nranks;
  P.rank = rank;
  double total = 0.0;  // gAverage denominator: rank-ordered sum of the cell counts
  for (int q = 0; q < nranks; ++q) total += (double)H[q].n_cells;
  M->nTotal = total;
  LF_CUDA(cudaStreamSynchronize(s));
  M->p2pConnected = true;
  M->sumPsiValid = false;
  for (auto &gexe : M->chunkGraph)  // graphs captured with the old transport
    if (gexe) {
      cudaGraphExecDestroy(gexe);
      gexe = nullptr;
    }
  M->kernelsPerIteration = 0;
}

}  // namespace lf
