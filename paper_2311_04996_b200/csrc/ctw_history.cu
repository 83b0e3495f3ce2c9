// ctw_history.cu -- partial-history garbage collection for long-running
// streams.
//
// The reference keeps every frame's records for the life of a channel
// (DecodeState.frames, decoder.py:160, :319-331), so a stream's memory grows
// linearly with its audio. Only records reachable from the active tokens can
// ever be on a best path or a partial hypothesis (best_path walks prev
// pointers from an active token, decoder.py:377-415), so a lane can drop the
// rest: mark the prev-chains of the active tokens (chains of different tokens
// merge within a few frames, so marking stops at the first record already
// marked), renumber the kept records with a prefix sum, copy them into fresh
// history pages with remapped prev pointers, and remap the frame starts and
// the sources' backpointers. Kept records keep their frame order, so
// best_path and the per-chunk partial hypotheses are unchanged.
#include <cuda_runtime.h>
#include <cub/block/block_scan.cuh>
#include <stdint.h>

#include "ctw_common.h"

#define HG_BS 1024

namespace {

__device__ __forceinline__ int2 hg_link(CtwRecPage* const* pages, long long r) {
  return pages[r >> CTW_PAGE_LOG2]->link[r & (CTW_PAGE - 1)];
}

// One CTA per lane: mark every record reachable from the lane's sources.
__global__ void __launch_bounds__(HG_BS) k_hist_mark(const CtwLane* lanes, const int* lane_ids,
                                                     uint32_t* const* marks) {
  const CtwLane& L = lanes[lane_ids[blockIdx.x]];
  uint32_t* m = marks[blockIdx.x];
  const CtwSrc* src = L.src[L.src_buf];
  for (int i = threadIdx.x; i < L.n_src; i += HG_BS) {
    long long r = src[i].bp;
    while (r >= 0) {
      const uint32_t bit = 1u << (r & 31);
      if (atomicOr(&m[r >> 5], bit) & bit) break;  // merged into an already marked chain
      r = hg_link(L.pages, r).x;
    }
  }
}

// One CTA per lane: new index of every kept record (exclusive prefix of the
// marks, written over the mark words' companion array), then the copy into
// the new pages with remapped prev pointers, the new frame starts and the
// sources' backpointers.
__global__ void __launch_bounds__(HG_BS) k_hist_compact(CtwLane* lanes, const int* lane_ids,
                                                        uint32_t* const* marks, int32_t* const* newidx,
                                                        CtwRecPage* const* const* new_pages, long long* kept) {
  typedef cub::BlockScan<int, HG_BS> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry;
  CtwLane& L = lanes[lane_ids[blockIdx.x]];
  const uint32_t* m = marks[blockIdx.x];
  int32_t* ni = newidx[blockIdx.x];
  CtwRecPage* const* np = new_pages[blockIdx.x];
  const long long R = L.n_rec;
  const int tid = threadIdx.x;
  if (tid == 0) carry = 0;
  __syncthreads();
  // prefix over 32-record words: thread t handles word w0 + t
  const long long W = (R + 31) >> 5;
  for (long long w0 = 0; w0 < W; w0 += HG_BS) {
    const long long w = w0 + tid;
    const uint32_t bits = w < W ? m[w] : 0u;
    int ex, tot;
    Scan(tmp).ExclusiveSum(__popc(bits), ex, tot);
    const int base = carry + ex;
    if (w < W) {
      int k = base;  // ni[r] = kept records before r (the new index when r is kept)
      for (int b = 0; b < 32; ++b) {
        const long long r = (w << 5) + b;
        if (r >= R) break;
        ni[r] = k;
        k += (bits >> b) & 1u;
      }
    }
    __syncthreads();
    if (tid == 0) carry += tot;
    __syncthreads();
  }
  const int nk = carry;
  if (tid == 0) ni[R] = nk;
  __syncthreads();
  // copy kept records into the new pages, prev pointers remapped (the chain
  // of a kept record is kept, so prev always maps)
  for (long long r = tid; r < R; r += HG_BS) {
    if (!((m[r >> 5] >> (r & 31)) & 1u)) continue;
    const int k = ni[r];
    const CtwRecPage* op = L.pages[r >> CTW_PAGE_LOG2];
    const int oo = (int)(r & (CTW_PAGE - 1));
    int2 lk = op->link[oo];
    if (lk.x >= 0) lk.x = ni[lk.x];
    const int pl = op->plab[oo];  // (an ancestor of a kept record: kept)
    CtwRecPage* pg = np[k >> CTW_PAGE_LOG2];
    const int o = k & (CTW_PAGE - 1);
    pg->link[o] = lk;
    pg->plab[o] = pl >= 0 ? ni[pl] : pl;
    pg->state[o] = op->state[oo];
    pg->cost[o] = op->cost[oo];
  }
  // frame starts: kept records before the old start
  for (int f = tid; f < L.frame_count; f += HG_BS) L.frame_base[f] = ni[L.frame_base[f]];
  CtwSrc* src = L.src[L.src_buf];
  for (int i = tid; i < L.n_src; i += HG_BS) {
    if (src[i].bp >= 0) src[i].bp = ni[src[i].bp];
    if (src[i].anc >= 0) src[i].anc = ni[src[i].anc];
  }
  if (tid == 0) kept[blockIdx.x] = nk;
}

// Seed tokens of the lanes of a reset, one CTA per lane (a batch reset
// would otherwise issue two copies per lane).
__global__ void k_copy_seeds(const CtwSeedCopy* jobs) {
  const CtwSeedCopy j = jobs[blockIdx.x];
  for (int i = threadIdx.x; i < j.n; i += blockDim.x) {
    j.dst_src[i] = j.src_src[i];
    j.dst_pend[i] = j.src_pend[i];
  }
}

}  // namespace

extern "C" int ctw_launch_copy_seeds(const CtwSeedCopy* d_jobs, int n, cudaStream_t stream) {
  (void)cudaGetLastError();
  if (n > 0) k_copy_seeds<<<n, 256, 0, stream>>>(d_jobs);
  return (int)cudaGetLastError();
}

extern "C" int ctw_launch_hist_mark(const CtwLane* d_lanes, const int* d_ids, uint32_t* const* d_marks, int n,
                                    cudaStream_t stream) {
  (void)cudaGetLastError();
  k_hist_mark<<<n, HG_BS, 0, stream>>>(d_lanes, d_ids, d_marks);
  return (int)cudaGetLastError();
}

extern "C" int ctw_launch_hist_compact(CtwLane* d_lanes, const int* d_ids, uint32_t* const* d_marks,
                                       int32_t* const* d_newidx, CtwRecPage* const* const* d_new_pages,
                                       long long* d_kept, int n, cudaStream_t stream) {
  (void)cudaGetLastError();
  k_hist_compact<<<n, HG_BS, 0, stream>>>(d_lanes, d_ids, d_marks, d_newidx, d_new_pages, d_kept);
  return (int)cudaGetLastError();
}
