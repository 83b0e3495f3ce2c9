// ctw_api.cu -- host side of libctcwfst_b200.so: the C-ABI declared in
// include/ctcwfst_b200.h. Owns HBM allocations (graph, lanes), staging of
// log-likelihood chunks, the grow-and-rerun protocol of chunk-atomic lanes,
// and the export of histories in the reference layout.
//
// Reference call sites this layer stands behind (pkg/src/ctcwfst/):
//   FlatGraph / flatten                      decoder.py:70-138
//   DecodeState seeding / set_boost          decoder.py:173-238
//   DecodeState.advance_frames               decoder.py:264-341
//   best_path                                decoder.py:377-415
//   history_records / active_tokens          decoder.py:240-260
//   kernel plug-in contract                  _pykernel.py:28-248
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <unordered_map>
#include <unordered_set>
#include <string>
#include <atomic>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/ctcwfst_b200.h"
#include "ctw_common.h"

extern "C" int ctw_launch_decode(CtwLane*, const CtwStateRange*, const CtwArc*, const int32_t*,
                                 const double*, const void*, int, int, const long long*, const int*,
                                 const int*, int, const CtwDecodeCfg*, CtwLaneOut*, int, int, int, int,
                                 cudaStream_t);
extern "C" int ctw_launch_seed(CtwLane*, const CtwStateRange*, const CtwArc*, const int32_t*,
                               const double*, const int*, int, int, const CtwDecodeCfg*, CtwLaneOut*,
                               cudaStream_t);
extern "C" int ctw_launch_best(const CtwLane*, const CtwStateRange*, const CtwArc*, const int32_t*,
                               const double*, const int*, int, int32_t*, const long long*, const int*,
                               int*, double*, int*, CtwBpCache, cudaStream_t);
extern "C" int ctw_launch_clear(CtwTok*, uint32_t, cudaStream_t);
extern "C" int ctw_launch_copy_seeds(const CtwSeedCopy*, int, cudaStream_t);
extern "C" int ctw_launch_hist_mark(const CtwLane*, const int*, uint32_t* const*, int, cudaStream_t);
extern "C" int ctw_launch_hist_compact(CtwLane*, const int*, uint32_t* const*, int32_t* const*,
                                       CtwRecPage* const* const*, long long*, int, cudaStream_t);
extern "C" int ctw_launch_lattice(CtwLane*, const CtwStateRange*, const CtwArc*, const int32_t*, const double*,
                                  const uint32_t*, const CtwClo*, CtwLatEntry*, int, const void*, int, int, double,
                                  double, int, int, cudaStream_t);
extern "C" int ctw_build_closure_index(const CtwStateRange*, const CtwArc*, long long, uint32_t**, CtwClo**,
                                       long long*, cudaStream_t);

namespace {

thread_local std::string g_err;

// NVTX range around a C-ABI operation (nsys / ncu --nvtx timelines; free
// when no tool is attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                       \
  do {                                                                                       \
    cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      return fail(-100 - (int)e_, std::string(#expr) + ": " + cudaGetErrorString(e_));       \
  } while (0)

template <class T>
cudaError_t dalloc(T** p, size_t n) {
  *p = nullptr;
  if (n == 0) n = 1;
  return cudaMalloc((void**)p, n * sizeof(T));
}

template <class T>
void dfree(T*& p) {
  if (p) cudaFree((void*)p);
  p = nullptr;
}

// Lane buffers come from the stream-ordered pool allocator: growing a lane
// (table, history, pool) is an async alloc + copy + free on the lane stream,
// with no device-wide synchronisation.
template <class T>
cudaError_t salloc(T** p, size_t n, cudaStream_t st) {
  *p = nullptr;
  if (n == 0) n = 1;
  return cudaMallocAsync((void**)p, n * sizeof(T), st);
}

template <class T>
void sfree(T*& p, cudaStream_t st) {
  if (p) cudaFreeAsync((void*)p, st);
  p = nullptr;
}

uint32_t ceil_log2(uint64_t x) {
  uint32_t r = 0;
  while ((1ull << r) < x) ++r;
  return r;
}

}  // namespace

// ------------------------------------------------------------------ graph --

struct ctw_graph {
  int refs = 1;  // the creator + one per lane set (lanes keep their graph alive)
  int device = 0;
  bool eps_nonneg = true;  // every epsilon arc weight >= 0
  double w_min_emit = 0.0;  // min(0, smallest emitting arc weight): lattice source bound
  bool eps_olabel = false; // some epsilon arc carries an output label (boost applies)
  int64_t S = 0, A = 0, start = 0, max_il = 0, max_ol = 0;
  // fast search mode (ctw_kernels.cu): winner words hold an emitting-arc
  // offset in `ebits` bits and an epsilon-arc offset above the table index
  int64_t max_emit_deg = 0, max_eps_deg = 0;
  uint32_t ebits = 0;
  CtwStateRange* ranges = nullptr;
  CtwArc* arcs = nullptr;
  int32_t* olabel = nullptr;
  double* final_w = nullptr;
  std::vector<double> h_final;
  // epsilon-closure index of the lattice kernel (ctw_lattice.cu), built on
  // the first lattice request when no epsilon arc carries an output label
  std::mutex clo_mu;
  int clo_state = 0;  // 0 not built, 1 built, -1 not available
  uint32_t* clo_off = nullptr;
  CtwClo* clo_ent = nullptr;
  long long clo_n = 0;
};

// ------------------------------------------------------------------ lanes --

struct ctw_lanes {
  ctw_graph* g = nullptr;
  ctw_config cfg{};
  CtwDecodeCfg dcfg{};
  int n = 0, cap = 0;
  CtwLane* h = nullptr;  // pinned host mirror
  CtwLane* d = nullptr;  // device copy
  std::vector<double*> boost_buf;
  std::vector<int64_t> boost_cap;
  std::vector<char> seeded;
  std::vector<double> surv_ema;  // survivors per frame estimate, for history sizing
  // paged history: per-lane page lists (host) mirrored in device page tables;
  // pages beyond a lane's first return to a free list when it is reset
  std::vector<std::vector<CtwRecPage*>> hpages;
  std::vector<int64_t> ptab_cap;
  std::vector<CtwRecPage*> free_pages;
  std::vector<CtwRecPage*> slabs;  // page allocations (CTW_SLAB pages each)
  // seed tokens of each lane's current utterance (the lattice's first layer)
  std::vector<CtwSrc*> seed_src;
  std::vector<int32_t*> seed_pend;
  std::vector<int32_t> seed_n, seed_cap;
  std::vector<int32_t> seed_pool;  // label-pool prefix written by the seeding (seed label codes)
  char* lat_pin = nullptr;         // pinned staging of lattice results (grow-only)
  size_t lat_pin_cap = 0;
  CtwSeedCopy* seedjob_h = nullptr;  // batched seed copies of a reset (pinned / device, grow-only)
  CtwSeedCopy* seedjob_d = nullptr;
  int seedjob_cap = 0;
  // phrase automata (ctw_lane_set_fsa), device copies per lane
  std::vector<uint16_t*> fsa_next;
  std::vector<double*> fsa_cost;
  std::vector<int64_t> fsa_cap;
  std::vector<double> fsa_min;  // most negative entry cost (early-pruning exactness)
  std::vector<char> compacted;  // history garbage-collected since the last reset (no lattice)
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // scratch
  int* d_ids = nullptr;
  int* d_nframes = nullptr;
  long long* d_lloff = nullptr;
  CtwLaneOut* d_out = nullptr;
  int scratch_cap = 0;
  int* h_ids = nullptr;
  int* h_nframes = nullptr;
  long long* h_lloff = nullptr;
  CtwLaneOut* h_out = nullptr;
  char* d_stage = nullptr;
  size_t stage_bytes = 0;
  // best-path scratch
  int32_t* d_words = nullptr;
  size_t words_cap = 0;
  int32_t* h_words = nullptr;  // pinned staging of the whole word window (one D2H)
  size_t h_words_cap = 0;
  long long* d_woff = nullptr;
  int* d_wcap = nullptr;
  int* d_nwords = nullptr;
  double* d_tcost = nullptr;
  int* d_bstatus = nullptr;
  long long* h_woff = nullptr;
  int* h_wcap = nullptr;
  int* h_nwords = nullptr;
  double* h_tcost = nullptr;
  int* h_bstatus = nullptr;
  int best_cap = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // stats
  int64_t launches = 0, decode_launches = 0, arcs = 0, srcs = 0, frames = 0, max_slots = 0;
  double decode_ms = 0.0;
  // host-side breakdown of ctw_advance (seconds): staging H2D, capacity
  // pre-sizing, launch-to-completion, post-processing; grow re-runs
  double h_stage = 0, h_presize = 0, h_wait = 0, h_post = 0;
  int64_t h_reruns = 0, h_calls = 0;
  int64_t h_grow[4] = {0, 0, 0, 0};  // lanes re-run for: table, history, pool, sources
  int64_t prof[CTW_NPROF] = {0};
  int32_t search = 0;         // 0 exact (reference histories), 1 fast (words-exact)
  int64_t fast_launches = 0;  // decode launches that ran the fast mode
  uint32_t tlog2_hint = 0;  // largest token-table size any lane of this set grew to
  // CUDA graphs of a streaming step (ctw_advance_best's first round: the
  // parameter uploads, the frame kernel, the partial best paths and the
  // result copies as one graph launch), keyed by launch shape and buffers
  struct StepGraph {
    uintptr_t key[13];
    cudaGraphExec_t exec;
  };
  std::vector<StepGraph> step_graphs;
  // best-path caches of the streaming path (allocated on first use, for
  // bpc_lanes lanes; see CtwBpCache)
  CtwBpCache bpc{nullptr, nullptr, nullptr, nullptr, 0};
  int bpc_lanes = 0;
  bool graphs_off = false;
  int64_t graph_launches = 0, graph_builds = 0;
  std::mutex mu;
};

namespace {

std::mutex g_graph_mu;

int sync_lane(ctw_lanes* l, int i) {
  CUDA_TRY(cudaMemcpyAsync(&l->d[i], &l->h[i], sizeof(CtwLane), cudaMemcpyHostToDevice, l->stream));
  return 0;
}

void free_lane(CtwLane& L, cudaStream_t st) {
  sfree(L.table, st);
  sfree(L.slots, st);
  sfree(L.front, st);
  for (auto& s : L.src) sfree(s, st);
  sfree(L.pend, st);
  sfree(L.pages, st);
  sfree(L.frame_base, st);
  sfree(L.pool, st);
}

// (Re)allocate the table-sized buffers of lane i at capacity 1 << tlog2,
// preserving the committed sources (and their pending chains). Sources hold
// at most max_active survivors, or the seed closure (want_src).
int alloc_table(ctw_lanes* l, int i, uint32_t tlog2, int64_t want_src = 0) {
  CtwLane& L = l->h[i];
  if (tlog2 > 24) return fail(-3, "token table would exceed 2^24 entries per lane");
  const uint64_t tcap = 1ull << tlog2;
  const int64_t want = std::max<int64_t>({want_src, (int64_t)L.scap, std::min<int64_t>(l->cfg.max_active, 1 << 30),
                                          (int64_t)L.n_src, 256});
  const uint64_t scap = (uint64_t)std::min<int64_t>(want, (int64_t)CTW_LOAD(tcap)) + 1;
  CtwTok* table;
  uint2 *slots, *front;
  CtwSrc* src[3];
  int32_t* pend;
  cudaStream_t st = l->stream;
  CUDA_TRY(salloc(&table, tcap, st));
  CUDA_TRY(salloc(&slots, CTW_SLOTS_LEN(tcap), st));
  CUDA_TRY(salloc(&front, CTW_FRONT_LEN(tcap), st));
  for (int b = 0; b < 3; ++b) CUDA_TRY(salloc(&src[b], scap, st));
  CUDA_TRY(salloc(&pend, scap, st));
  if (ctw_launch_clear(table, (uint32_t)tcap, l->stream)) return fail(-1, "clear kernel launch failed");
  if (L.table) {
    if (L.n_src > 0) {
      CUDA_TRY(cudaMemcpyAsync(src[L.src_buf], L.src[L.src_buf], (size_t)L.n_src * sizeof(CtwSrc),
                               cudaMemcpyDeviceToDevice, l->stream));
      CUDA_TRY(cudaMemcpyAsync(pend, L.pend, (size_t)L.n_src * sizeof(int32_t), cudaMemcpyDeviceToDevice,
                               l->stream));
    }
    sfree(L.table, st);
    sfree(L.slots, st);
    sfree(L.front, st);
    for (auto& s : L.src) sfree(s, st);
    sfree(L.pend, st);
  }
  L.table = table;
  L.slots = slots;
  L.front = front;
  for (int b = 0; b < 3; ++b) L.src[b] = src[b];
  L.pend = pend;
  L.tlog2 = tlog2;
  L.scap = (int32_t)(scap - 1);
  l->tlog2_hint = std::max(l->tlog2_hint, tlog2);
  return sync_lane(l, i);
}

template <class T>
int grow_keep(cudaStream_t st, T*& p, int64_t keep, int64_t ncap) {
  T* np;
  CUDA_TRY(salloc(&np, (size_t)ncap, st));
  if (p && keep > 0) CUDA_TRY(cudaMemcpyAsync(np, p, (size_t)keep * sizeof(T), cudaMemcpyDeviceToDevice, st));
  sfree(p, st);
  p = np;
  return 0;
}

#define CTW_SLAB 16

// History capacity: append pages (recycled ones first) until `need` records
// fit; only the lane's page table is uploaded -- records are never copied.
int grow_hist(ctw_lanes* l, int i, int64_t need) {
  CtwLane& L = l->h[i];
  if (need <= L.rcap) return 0;
  // record indices are int32 on the device (prev pointers, source
  // backpointers): a channel's history is capped at 2^31 - 1 records
  if (need > (int64_t)INT32_MAX)
    return fail(-1, "channel history would exceed 2^31 records: compact it (DecodeState.compact_history, "
                    "StreamPool(gc_every=...)) or start a new channel");
  auto& pg = l->hpages[i];
  // two pages of headroom beyond the request: a channel that grows by a
  // chunk at a time (streaming) re-uploads its page table every few chunks
  // instead of on every one
  const int64_t want = std::min<int64_t>(need + 2 * (int64_t)CTW_PAGE, (int64_t)INT32_MAX);
  while ((int64_t)pg.size() * CTW_PAGE < want) {
    CtwRecPage* p = nullptr;
    if (l->free_pages.empty()) {
      // pages come in slabs: one allocation per CTW_SLAB pages
      CtwRecPage* slab = nullptr;
      CUDA_TRY(salloc(&slab, CTW_SLAB, l->stream));
      l->slabs.push_back(slab);
      for (int k = CTW_SLAB - 1; k >= 0; --k) l->free_pages.push_back(slab + k);
    }
    p = l->free_pages.back();
    l->free_pages.pop_back();
    pg.push_back(p);
  }
  if ((int64_t)pg.size() > l->ptab_cap[i]) {
    const int64_t nc = std::max<int64_t>((int64_t)pg.size(), 2 * l->ptab_cap[i]);
    sfree(L.pages, l->stream);
    CUDA_TRY(salloc(&L.pages, (size_t)nc, l->stream));
    l->ptab_cap[i] = nc;
  }
  CUDA_TRY(cudaMemcpyAsync(L.pages, pg.data(), pg.size() * sizeof(CtwRecPage*), cudaMemcpyHostToDevice, l->stream));
  L.rcap = (int64_t)pg.size() * CTW_PAGE;
  return sync_lane(l, i);
}

// A lane starts a new utterance: keep one history page, recycle the rest.
void trim_hist(ctw_lanes* l, int i) {
  auto& pg = l->hpages[i];
  while (pg.size() > 1) {
    l->free_pages.push_back(pg.back());
    pg.pop_back();
  }
  l->h[i].rcap = (int64_t)pg.size() * CTW_PAGE;
}

int grow_frames(ctw_lanes* l, int i, int64_t need) {
  CtwLane& L = l->h[i];
  if (need <= L.fcap) return 0;
  int64_t ncap = std::max<int64_t>(need, 2 * (int64_t)L.fcap);
  if (ncap > INT32_MAX) return fail(-1, "frame count exceeds 2^31");
  if (int r = grow_keep(l->stream, L.frame_base, L.frame_count, ncap)) return r;
  L.fcap = (int32_t)ncap;
  return sync_lane(l, i);
}

int grow_pool(ctw_lanes* l, int i, int64_t need) {
  CtwLane& L = l->h[i];
  if (need <= L.pcap) return 0;
  int64_t ncap = std::max<int64_t>(need, 2 * (int64_t)L.pcap);
  if (ncap > INT32_MAX) return fail(-1, "olabel pool exceeds 2^31");
  if (int r = grow_keep(l->stream, L.pool, L.pool_used, ncap)) return r;
  L.pcap = (int32_t)ncap;
  return sync_lane(l, i);
}

int init_lane(ctw_lanes* l, int i) {
  CtwLane& L = l->h[i];
  std::memset(&L, 0, sizeof(L));
  const uint64_t S = (uint64_t)std::max<int64_t>(l->g->S, 1);
  // new lanes start at the largest table any lane of this set needed
  const uint32_t tlog2 = std::max(std::min<uint32_t>(std::max<uint32_t>(6, ceil_log2(2 * S + 2)), 16),
                                  std::min<uint32_t>(l->tlog2_hint, ceil_log2(2 * S + 2)));
  if (int r = alloc_table(l, i, tlog2)) return r;
  L.smask = 0xFFFFFFFFu;
  L.rcap = 0;
  L.fcap = 256;
  L.pcap = 1 << 10;
  cudaStream_t st = l->stream;
  l->hpages[i].clear();
  l->ptab_cap[i] = 0;
  CUDA_TRY(salloc(&L.frame_base, (size_t)L.fcap, st));
  CUDA_TRY(salloc(&L.pool, (size_t)L.pcap, st));
  return grow_hist(l, i, 1);
}

int ensure_scratch(ctw_lanes* l, int n) {
  if (n <= l->scratch_cap) return 0;
  int c = std::max(n, 2 * l->scratch_cap);
  dfree(l->d_ids);
  dfree(l->d_nframes);
  dfree(l->d_lloff);
  dfree(l->d_out);
  if (l->h_ids) cudaFreeHost(l->h_ids);
  if (l->h_nframes) cudaFreeHost(l->h_nframes);
  if (l->h_lloff) cudaFreeHost(l->h_lloff);
  if (l->h_out) cudaFreeHost(l->h_out);
  CUDA_TRY(dalloc(&l->d_ids, c));
  CUDA_TRY(dalloc(&l->d_nframes, c));
  CUDA_TRY(dalloc(&l->d_lloff, c));
  CUDA_TRY(dalloc(&l->d_out, c));
  CUDA_TRY(cudaMallocHost((void**)&l->h_ids, c * sizeof(int)));
  CUDA_TRY(cudaMallocHost((void**)&l->h_nframes, c * sizeof(int)));
  CUDA_TRY(cudaMallocHost((void**)&l->h_lloff, c * sizeof(long long)));
  CUDA_TRY(cudaMallocHost((void**)&l->h_out, c * sizeof(CtwLaneOut)));
  l->scratch_cap = c;
  return 0;
}

// Best-path caches for every lane of the set (streaming path): allocated on
// first use, re-allocated (all empty) when the set grew.
int bpc_ensure(ctw_lanes* l) {
  if (l->bpc_lanes >= l->n) return 0;
  dfree(l->bpc.n);
  dfree(l->bpc.rec);
  dfree(l->bpc.cum);
  dfree(l->bpc.words);
  l->bpc_lanes = 0;
  l->bpc.lanes = 0;
  const size_t c = (size_t)l->cap;
  CUDA_TRY(dalloc(&l->bpc.n, c));
  CUDA_TRY(dalloc(&l->bpc.rec, c * CTW_BPC_REC));
  CUDA_TRY(dalloc(&l->bpc.cum, c * CTW_BPC_REC));
  CUDA_TRY(dalloc(&l->bpc.words, c * CTW_BPC_WORDS));
  CUDA_TRY(cudaMemsetAsync(l->bpc.n, 0, c * sizeof(int32_t), l->stream));
  l->bpc_lanes = l->cap;
  l->bpc.lanes = l->cap;
  return 0;
}

// Empty a lane's best-path cache (its history was reset or renumbered).
int bpc_clear(ctw_lanes* l, int lane) {
  if (l->bpc.n && lane < l->bpc_lanes)
    CUDA_TRY(cudaMemsetAsync(l->bpc.n + lane, 0, sizeof(int32_t), l->stream));
  return 0;
}

int reserve_lanes(ctw_lanes* l, int n) {
  if (n <= l->n) return 0;
  if (n > l->cap) {
    int c = std::max(n, 2 * l->cap);
    CtwLane* nh;
    CtwLane* nd;
    CUDA_TRY(cudaMallocHost((void**)&nh, c * sizeof(CtwLane)));
    CUDA_TRY(dalloc(&nd, c));
    if (l->h) {
      std::memcpy(nh, l->h, l->n * sizeof(CtwLane));
      cudaFreeHost(l->h);
    }
    if (l->d) {
      CUDA_TRY(cudaMemcpyAsync(nd, l->d, l->n * sizeof(CtwLane), cudaMemcpyDeviceToDevice, l->stream));
      CUDA_TRY(cudaStreamSynchronize(l->stream));
      dfree(l->d);
    }
    l->h = nh;
    l->d = nd;
    l->cap = c;
  }
  l->hpages.resize(n);
  l->ptab_cap.resize(n, 0);
  l->seed_src.resize(n, nullptr);
  l->seed_pend.resize(n, nullptr);
  l->seed_n.resize(n, 0);
  l->seed_cap.resize(n, 0);
  l->seed_pool.resize(n, 0);
  l->fsa_next.resize(n, nullptr);
  l->fsa_cost.resize(n, nullptr);
  l->fsa_cap.resize(n, 0);
  l->fsa_min.resize(n, 0.0);
  l->compacted.resize(n, 0);
  for (int i = l->n; i < n; ++i) {
    if (int r = init_lane(l, i)) return r;
  }
  l->boost_buf.resize(n, nullptr);
  l->boost_cap.resize(n, 0);
  l->seeded.resize(n, 0);
  l->surv_ema.resize(n, -1.0);
  l->n = n;
  CUDA_TRY(cudaStreamSynchronize(l->stream));
  return 0;
}

// Early beam pruning is exact when epsilon increments cannot be negative
// (see CtwLane::prune_ok) and the cap on Gauss-Seidel passes cannot bind: with
// non-negative epsilon weights a closure over K distinct token keys converges
// in at most K passes (Bellman-Ford: shortest epsilon paths have < K arcs) plus
// one quiet pass, so max_ne_iters >= K + 1 never triggers ERR_EPS_ITERS -- the
// default cap 2 x num_states (decoder.py:164-168) always qualifies. Below that
// (a tight user cap) the pass accounting must include out-of-beam slots.
// `keys` = token-key space (states, x automaton states with a phrase FSA).
int64_t prune_cap_needed(const ctw_lanes* l, int64_t keys) {
  return std::min<int64_t>((int64_t)1 << 16, keys + 1);
}

int32_t prune_flag(const ctw_lanes* l, const double* boost, int64_t len, int64_t keys) {
  const ctw_graph* g = l->g;
  if (!g->eps_nonneg || l->cfg.max_ne_iters < prune_cap_needed(l, keys)) return 0;
  if (boost && g->eps_olabel)
    for (int64_t i = 0; i < len; ++i)
      if (!(boost[i] >= 0.0)) return 0;
  return 1;
}

int64_t key_space(const ctw_lanes* l, const CtwLane& L) {
  return L.fsa_next ? l->g->S * (int64_t)std::max(1, L.fsa_states) : l->g->S;
}

// Fast search mode for a launch over `ids`: requested, and every lane fits its
// preconditions -- early pruning exact (prune_ok), winner words wide enough
// for the source capacity and the epsilon out-degree at the lane's table size.
bool fast_launch(const ctw_lanes* l, const int* ids, int n) {
  const ctw_graph* g = l->g;
  if (l->search != 1 || g->ebits > 24) return false;
  for (int k = 0; k < n; ++k) {
    const CtwLane& L = l->h[ids[k]];
    if (!L.prune_ok) return false;
    if ((uint64_t)L.scap >= (1ull << (31 - g->ebits))) return false;
    if ((uint64_t)g->max_eps_deg > (1ull << (31 - L.tlog2))) return false;
  }
  return true;
}

void update_from_out(CtwLane& L, const CtwLaneOut& o) {
  L.n_src = o.n_src;
  L.src_buf = o.src_buf;
  L.frame_count = o.frame_count;
  L.pool_used = o.pool_used;
  L.n_rec = o.n_rec;
  L.pend_valid = o.pend_valid;
}

int check_ids(ctw_lanes* l, const int32_t* ids, int n) {
  std::vector<char> seen(l->n, 0);
  for (int i = 0; i < n; ++i) {
    if (ids[i] < 0 || ids[i] >= l->n) return fail(-1, "lane id out of range");
    if (seen[ids[i]]) return fail(-1, "duplicate lane id in one batch");
    seen[ids[i]] = 1;
  }
  return 0;
}

// Device view of log-likelihood rows: device buffers pass through; host rows
// are staged into HBM with one copy covering every lane's span.
int stage_rows(ctw_lanes* l, const void* loglik, int32_t location, size_t esz, const int64_t* ll_offsets,
               const int32_t* frames, int n, int32_t width, const char** dev_ll) {
  *dev_ll = (const char*)loglik;
  if (location != 0) return 0;
  int64_t lo = INT64_MAX, hi = 0;
  for (int i = 0; i < n; ++i) {
    if (frames[i] == 0) continue;
    lo = std::min<int64_t>(lo, ll_offsets[i]);
    hi = std::max<int64_t>(hi, ll_offsets[i] + (int64_t)frames[i] * width);
  }
  if (lo == INT64_MAX) lo = hi = 0;
  const size_t bytes = (size_t)(hi - lo) * esz;
  if (bytes > l->stage_bytes) {
    dfree(l->d_stage);
    CUDA_TRY(dalloc(&l->d_stage, bytes + bytes / 4));
    l->stage_bytes = bytes + bytes / 4;
  }
  if (bytes)
    CUDA_TRY(cudaMemcpyAsync(l->d_stage, (const char*)loglik + lo * esz, bytes, cudaMemcpyHostToDevice, l->stream));
  *dev_ll = l->d_stage - lo * (int64_t)esz;
  return 0;
}

// Run the seed kernel on `ids`, growing tables / pools and re-running lanes
// that ask for it. st[i] gets the per-lane CTW status.
int run_seed(ctw_lanes* l, std::vector<int> ids, std::vector<int>& st) {
  ctw_graph* g = l->g;
  std::vector<int> pos(l->n, -1);
  for (size_t i = 0; i < ids.size(); ++i) pos[ids[i]] = (int)i;
  st.assign(ids.size(), CTW_OK);
  std::vector<int> todo = ids;
  for (int round = 0; !todo.empty(); ++round) {
    if (round > 40) return fail(-1, "seed: grow loop did not converge");
    const int n = (int)todo.size();
    if (int r = ensure_scratch(l, n)) return r;
    for (int i = 0; i < n; ++i) l->h_ids[i] = todo[i];
    CUDA_TRY(cudaMemcpyAsync(l->d_ids, l->h_ids, n * sizeof(int), cudaMemcpyHostToDevice, l->stream));
    if (ctw_launch_seed(l->d, g->ranges, g->arcs, g->olabel, g->final_w, l->d_ids, n, (int)g->start,
                        &l->dcfg, l->d_out, l->stream))
      return fail(-1, std::string("seed launch: ") + cudaGetErrorString(cudaGetLastError()));
    l->launches++;
    CUDA_TRY(cudaMemcpyAsync(l->h_out, l->d_out, n * sizeof(CtwLaneOut), cudaMemcpyDeviceToHost, l->stream));
    CUDA_TRY(cudaStreamSynchronize(l->stream));
    std::vector<int> again;
    for (int i = 0; i < n; ++i) {
      const int lane = todo[i];
      const CtwLaneOut& o = l->h_out[i];
      CtwLane& L = l->h[lane];
      if (o.status == CTW_GROW_TABLE) {
        if (int r = alloc_table(l, lane, L.tlog2 + 1)) return r;
        again.push_back(lane);
      } else if (o.status == CTW_GROW_SRC) {
        if (int r = alloc_table(l, lane, L.tlog2, 2 * (int64_t)L.scap + 1)) return r;
        again.push_back(lane);
      } else if (o.status == CTW_GROW_POOL) {
        if (int r = grow_pool(l, lane, 2 * (int64_t)L.pcap)) return r;
        again.push_back(lane);
      } else {
        update_from_out(L, o);
        st[pos[lane]] = o.status;
      }
    }
    todo.swap(again);
  }
  return 0;
}

}  // namespace

extern "C" {

int ctw_abi_version(void) { return CTW_ABI_VERSION; }

const char* ctw_last_error(void) { return g_err.c_str(); }

int ctw_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int ctw_graph_create(const int64_t* off, const int64_t* eps_end, const int32_t* ilabel,
                     const int32_t* olabel, const double* weight, const int32_t* nextstate,
                     const double* final_w, int64_t num_states, int64_t num_arcs, int64_t start,
                     int32_t device, ctw_graph** out) {
  NvtxRange nvtx_("ctw_graph_create");
  *out = nullptr;
  if (num_states <= 0) return fail(-1, "empty graph");
  if (num_arcs < 0 || num_arcs >= 0x7FFFFFFFLL) return fail(-1, "arc count must be < 2^31");
  if (num_states >= 0x7FFFFFFFLL) return fail(-1, "state count must be < 2^31");
  if (start < 0 || start >= num_states) return fail(-1, "start state out of range");
  if (off[0] != 0 || off[num_states] != num_arcs) return fail(-1, "off[] does not span the arcs");
  std::vector<CtwStateRange> r((size_t)num_states);
  int64_t max_il = 0, max_ol = 0, max_emit_deg = 0, max_eps_deg = 0;
  for (int64_t s = 0; s < num_states; ++s) {
    if (off[s + 1] < off[s] || eps_end[s] < off[s] || eps_end[s] > off[s + 1])
      return fail(-1, "inconsistent CSR offsets");
    max_eps_deg = std::max<int64_t>(max_eps_deg, eps_end[s] - off[s]);
    max_emit_deg = std::max<int64_t>(max_emit_deg, off[s + 1] - eps_end[s]);
    r[s] = CtwStateRange{(uint32_t)off[s], (uint32_t)eps_end[s], (uint32_t)off[s + 1], 0u};
  }
  std::vector<CtwArc> arcs((size_t)std::max<int64_t>(num_arcs, 1));
  bool eps_nonneg = true, eps_olabel = false;
  double w_min_emit = 0.0;
  for (int64_t s = 0; s < num_states; ++s) {
    for (int64_t a = off[s]; a < off[s + 1]; ++a) {
      const bool eps = a < eps_end[s];
      if ((ilabel[a] == 0) != eps) return fail(-1, "arcs are not ilabel-sorted with epsilons first");
      if (nextstate[a] < 0 || nextstate[a] >= num_states) return fail(-1, "nextstate out of range");
      if (olabel[a] < 0 || ilabel[a] < 0) return fail(-1, "negative label");
      arcs[a] = CtwArc{weight[a], nextstate[a], ilabel[a]};
      if (eps) {
        if (!(weight[a] >= 0.0)) eps_nonneg = false;
        if (olabel[a] != 0) eps_olabel = true;
      } else if (weight[a] < w_min_emit) {
        w_min_emit = weight[a];
      }
      max_il = std::max<int64_t>(max_il, ilabel[a]);
      max_ol = std::max<int64_t>(max_ol, olabel[a]);
    }
  }
  ctw_graph* g = new ctw_graph();
  g->device = device;
  g->S = num_states;
  g->A = num_arcs;
  g->start = start;
  g->max_il = max_il;
  g->max_ol = max_ol;
  g->h_final.assign(final_w, final_w + num_states);
  g->eps_nonneg = eps_nonneg;
  g->eps_olabel = eps_olabel;
  g->w_min_emit = w_min_emit;
  g->max_emit_deg = max_emit_deg;
  g->max_eps_deg = max_eps_deg;
  g->ebits = ceil_log2((uint64_t)max_emit_deg + 1);
  auto bail = [&](int code) {
    ctw_graph_destroy(g);
    return code;
  };
  if (cudaSetDevice(device) != cudaSuccess) return bail(fail(-2, "cudaSetDevice failed"));
  if (dalloc(&g->ranges, (size_t)num_states) || dalloc(&g->arcs, arcs.size()) ||
      dalloc(&g->olabel, (size_t)std::max<int64_t>(num_arcs, 1)) || dalloc(&g->final_w, (size_t)num_states))
    return bail(fail(-3, "graph allocation failed"));
  if (cudaMemcpy(g->ranges, r.data(), r.size() * sizeof(CtwStateRange), cudaMemcpyHostToDevice) ||
      cudaMemcpy(g->arcs, arcs.data(), (size_t)num_arcs * sizeof(CtwArc), cudaMemcpyHostToDevice) ||
      cudaMemcpy(g->olabel, olabel, (size_t)num_arcs * sizeof(int32_t), cudaMemcpyHostToDevice) ||
      cudaMemcpy(g->final_w, final_w, (size_t)num_states * sizeof(double), cudaMemcpyHostToDevice))
    return bail(fail(-3, "graph upload failed"));
  *out = g;
  return 0;
}

int ctw_graph_load(const char* path, int32_t device, ctw_graph** out) {
  *out = nullptr;
  const int fd = open(path, O_RDONLY);
  if (fd < 0) return fail(-1, std::string("cannot open graph file ") + path);
  struct stat st;
  if (fstat(fd, &st) != 0 || st.st_size < 64) {
    close(fd);
    return fail(-1, "graph file too small");
  }
  const size_t size = (size_t)st.st_size;
  void* base = mmap(nullptr, size, PROT_READ, MAP_PRIVATE, fd, 0);
  close(fd);
  if (base == MAP_FAILED) return fail(-1, "mmap of the graph file failed");
  const char* b = (const char*)base;
  int rc = 0;
  do {
    if (std::memcmp(b, "CTWGRAPH", 8) != 0) {
      rc = fail(-1, "not a CTWGRAPH file");
      break;
    }
    uint32_t ver;
    std::memcpy(&ver, b + 8, 4);
    if (ver != 1) {
      rc = fail(-1, "unsupported CTWGRAPH version");
      break;
    }
    int64_t h[5];
    std::memcpy(h, b + 16, sizeof(h));
    const int64_t S = h[0], A = h[1], start = h[2];
    if (S <= 0 || A < 0 || start < 0 || start >= S) {
      rc = fail(-1, "bad CTWGRAPH header");
      break;
    }
    // graphio.py layout: arrays in order, each 8-byte aligned
    size_t pos = 64;
    auto take = [&](size_t bytes) {
      const size_t at = pos;
      pos = (pos + bytes + 7) & ~(size_t)7;
      return at;
    };
    const size_t o_off = take((size_t)(S + 1) * 8), o_eps = take((size_t)S * 8), o_il = take((size_t)A * 4),
                 o_ol = take((size_t)A * 4), o_w = take((size_t)A * 8), o_ns = take((size_t)A * 4),
                 o_fin = take((size_t)S * 8);
    if (pos > size) {
      rc = fail(-1, "truncated CTWGRAPH file");
      break;
    }
    rc = ctw_graph_create((const int64_t*)(b + o_off), (const int64_t*)(b + o_eps), (const int32_t*)(b + o_il),
                          (const int32_t*)(b + o_ol), (const double*)(b + o_w), (const int32_t*)(b + o_ns),
                          (const double*)(b + o_fin), S, A, start, device, out);
  } while (false);
  munmap(base, size);
  return rc;
}

void ctw_graph_destroy(ctw_graph* g) {
  if (!g) return;
  {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    if (--g->refs > 0) return;
  }
  cudaSetDevice(g->device);
  dfree(g->ranges);
  dfree(g->arcs);
  dfree(g->olabel);
  dfree(g->final_w);
  dfree(g->clo_off);
  dfree(g->clo_ent);
  delete g;
}

int ctw_graph_info(const ctw_graph* g, int64_t* num_states, int64_t* num_arcs, int64_t* max_ilabel,
                   int64_t* max_olabel, int64_t* bytes) {
  if (num_states) *num_states = g->S;
  if (num_arcs) *num_arcs = g->A;
  if (max_ilabel) *max_ilabel = g->max_il;
  if (max_olabel) *max_olabel = g->max_ol;
  if (bytes) *bytes = g->S * (int64_t)(sizeof(CtwStateRange) + sizeof(double)) + g->A * (int64_t)(sizeof(CtwArc) + 4);
  if (bytes && g->clo_state == 1) *bytes += (g->S + 1) * 4 + g->clo_n * (int64_t)sizeof(CtwClo);
  return 0;
}

int ctw_lanes_create(ctw_graph* g, int32_t n_lanes, const ctw_config* cfg, void* stream, ctw_lanes** out) {
  *out = nullptr;
  if (!g) return fail(-1, "null graph");
  if (n_lanes < 0) return fail(-1, "negative lane count");
  if (!(cfg->beam > 0) || cfg->max_active < 1 || !(cfg->acoustic_scale > 0))
    return fail(-1, "invalid decoder config");
  CUDA_TRY(cudaSetDevice(g->device));
  {
    // keep freed lane memory in the pool (no release at synchronisation points)
    cudaMemPool_t mp;
    if (cudaDeviceGetDefaultMemPool(&mp, g->device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  ctw_lanes* l = new ctw_lanes();
  l->g = g;
  {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    g->refs++;
  }
  l->cfg = *cfg;
  l->dcfg = CtwDecodeCfg{cfg->beam, cfg->acoustic_scale, cfg->relax_eps, (long long)cfg->max_active,
                         (long long)cfg->max_ne_iters};
  if (stream) {
    l->stream = (cudaStream_t)stream;
  } else {
    if (cudaStreamCreateWithFlags(&l->stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete l;
      return fail(-2, "stream creation failed");
    }
    l->own_stream = true;
  }
  cudaEventCreate(&l->ev0);
  cudaEventCreate(&l->ev1);
  {
    // lane buffers come from the stream-ordered pool; keep freed memory
    // mapped in the pool (regrown tables / history pages reuse it instead of
    // remapping at every synchronisation)
    cudaMemPool_t mp;
    if (cudaDeviceGetDefaultMemPool(&mp, g->device) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  if (int r = reserve_lanes(l, n_lanes)) {
    ctw_lanes_destroy(l);
    return r;
  }
  *out = l;
  return 0;
}

void ctw_lanes_destroy(ctw_lanes* l) {
  if (!l) return;
  cudaSetDevice(l->g->device);
  cudaStreamSynchronize(l->stream);
  for (int i = 0; i < l->n; ++i) {
    free_lane(l->h[i], l->stream);
    dfree(l->boost_buf[i]);
    sfree(l->seed_src[i], l->stream);
    sfree(l->seed_pend[i], l->stream);
    dfree(l->fsa_next[i]);
    dfree(l->fsa_cost[i]);
  }
  for (CtwRecPage* p : l->slabs) sfree(p, l->stream);
  cudaStreamSynchronize(l->stream);
  if (l->h) cudaFreeHost(l->h);
  if (l->lat_pin) cudaFreeHost(l->lat_pin);
  if (l->seedjob_h) cudaFreeHost(l->seedjob_h);
  dfree(l->seedjob_d);
  dfree(l->d);
  dfree(l->d_ids);
  dfree(l->d_nframes);
  dfree(l->d_lloff);
  dfree(l->d_out);
  dfree(l->d_stage);
  dfree(l->d_words);
  dfree(l->d_woff);
  dfree(l->d_wcap);
  dfree(l->d_nwords);
  dfree(l->d_tcost);
  dfree(l->d_bstatus);
  for (void* p : {(void*)l->h_ids, (void*)l->h_nframes, (void*)l->h_lloff, (void*)l->h_out, (void*)l->h_woff,
                  (void*)l->h_wcap, (void*)l->h_nwords, (void*)l->h_tcost, (void*)l->h_bstatus, (void*)l->h_words})
    if (p) cudaFreeHost(p);
  dfree(l->bpc.n);
  dfree(l->bpc.rec);
  dfree(l->bpc.cum);
  dfree(l->bpc.words);
  for (auto& sg : l->step_graphs) cudaGraphExecDestroy(sg.exec);
  l->step_graphs.clear();
  if (l->ev0) cudaEventDestroy(l->ev0);
  if (l->ev1) cudaEventDestroy(l->ev1);
  if (l->own_stream) cudaStreamDestroy(l->stream);
  ctw_graph* g = l->g;
  delete l;
  ctw_graph_destroy(g);  // drop the lane set's reference
}

int ctw_lanes_reserve(ctw_lanes* l, int32_t n) {
  std::lock_guard<std::mutex> lk(l->mu);
  CUDA_TRY(cudaSetDevice(l->g->device));
  if (int r = reserve_lanes(l, n)) return r;
  return l->n;
}

int ctw_lane_reset(ctw_lanes* l, const int32_t* lane_ids, int32_t n, const double* const* boosts,
                   const int64_t* boost_lens, int32_t* status) {
  NvtxRange nvtx_("ctw_lane_reset");
  std::lock_guard<std::mutex> lk(l->mu);
  CUDA_TRY(cudaSetDevice(l->g->device));
  if (int r = check_ids(l, lane_ids, n)) return r;
  std::vector<int> ids(lane_ids, lane_ids + n);
  for (int i = 0; i < n; ++i) {
    const int lane = ids[i];
    CtwLane& L = l->h[lane];
    const double* b = boosts ? boosts[i] : nullptr;
    if (b) {
      const int64_t len = boost_lens[i];
      if (len < l->g->max_ol + 1) return fail(-1, "boost vector shorter than max_olabel + 1");
      if (l->boost_cap[lane] < len) {
        dfree(l->boost_buf[lane]);
        CUDA_TRY(dalloc(&l->boost_buf[lane], (size_t)len));
        l->boost_cap[lane] = len;
      }
      CUDA_TRY(cudaMemcpyAsync(l->boost_buf[lane], b, (size_t)len * sizeof(double), cudaMemcpyHostToDevice,
                               l->stream));
      L.boost = l->boost_buf[lane];
      L.boost_len = (int32_t)len;
    } else {
      L.boost = nullptr;
      L.boost_len = 0;
    }
    L.prune_ok = prune_flag(l, b, b ? boost_lens[i] : 0, key_space(l, L)) &&
                 !(L.fsa_next && l->g->eps_olabel && l->fsa_min[lane] < 0);
    L.n_src = 0;
    L.src_buf = 0;
    L.frame_count = 0;
    L.pool_used = 0;
    L.n_rec = 0;
    L.pend_valid = 0;
    l->compacted[lane] = 0;
    trim_hist(l, lane);
  }
  // descriptor uploads and cache clears per run of consecutive lane ids
  {
    std::vector<int> sorted(ids);
    std::sort(sorted.begin(), sorted.end());
    sorted.erase(std::unique(sorted.begin(), sorted.end()), sorted.end());
    for (size_t a = 0; a < sorted.size();) {
      size_t b = a + 1;
      while (b < sorted.size() && sorted[b] == sorted[b - 1] + 1) ++b;
      const int lo = sorted[a], cnt = (int)(b - a);
      CUDA_TRY(cudaMemcpyAsync(&l->d[lo], &l->h[lo], cnt * sizeof(CtwLane), cudaMemcpyHostToDevice, l->stream));
      if (l->bpc.n && lo + cnt <= l->bpc_lanes)
        CUDA_TRY(cudaMemsetAsync(l->bpc.n + lo, 0, cnt * sizeof(int32_t), l->stream));
      else
        for (int k = lo; k < lo + cnt; ++k)
          if (int r = bpc_clear(l, k)) return r;
      a = b;
    }
  }
  std::vector<int> st;
  if (int r = run_seed(l, ids, st)) return r;
  // keep the seed tokens (device copies, stream-ordered) for lattices: one
  // batched copy kernel (run_seed synchronised, so the pinned job list is free)
  if (n > l->seedjob_cap) {
    const int c = std::max(n, 2 * l->seedjob_cap);
    if (l->seedjob_h) cudaFreeHost(l->seedjob_h);
    dfree(l->seedjob_d);
    l->seedjob_h = nullptr;
    l->seedjob_cap = 0;
    CUDA_TRY(cudaMallocHost((void**)&l->seedjob_h, c * sizeof(CtwSeedCopy)));
    CUDA_TRY(dalloc(&l->seedjob_d, (size_t)c));
    l->seedjob_cap = c;
  }
  int njobs = 0;
  for (int i = 0; i < n; ++i) {
    status[i] = st[i];
    l->seeded[ids[i]] = st[i] == CTW_OK;
    if (st[i] != CTW_OK) continue;
    const int lane = ids[i];
    const CtwLane& L = l->h[lane];
    if (L.n_src > l->seed_cap[lane]) {
      sfree(l->seed_src[lane], l->stream);
      sfree(l->seed_pend[lane], l->stream);
      const int32_t c = std::max<int32_t>(L.n_src, 64);
      CUDA_TRY(salloc(&l->seed_src[lane], (size_t)c, l->stream));
      CUDA_TRY(salloc(&l->seed_pend[lane], (size_t)c, l->stream));
      l->seed_cap[lane] = c;
    }
    l->seed_n[lane] = L.n_src;
    l->seed_pool[lane] = L.pool_used;
    if (L.n_src)
      l->seedjob_h[njobs++] = CtwSeedCopy{l->seed_src[lane], L.src[L.src_buf], l->seed_pend[lane], L.pend,
                                          L.n_src, 0};
  }
  if (njobs) {
    CUDA_TRY(cudaMemcpyAsync(l->seedjob_d, l->seedjob_h, njobs * sizeof(CtwSeedCopy), cudaMemcpyHostToDevice,
                             l->stream));
    if (ctw_launch_copy_seeds(l->seedjob_d, njobs, l->stream))
      return fail(-1, std::string("seed copy launch: ") + cudaGetErrorString(cudaGetLastError()));
    // (the job list is pinned host memory read by the copy: the next reset
    // must not overwrite it before the copy ran)
    CUDA_TRY(cudaStreamSynchronize(l->stream));
  }
  return 0;
}

int ctw_lane_set_boost(ctw_lanes* l, int32_t lane, const double* boost, int64_t boost_len) {
  std::lock_guard<std::mutex> lk(l->mu);
  CUDA_TRY(cudaSetDevice(l->g->device));
  if (lane < 0 || lane >= l->n) return fail(-1, "lane id out of range");
  CtwLane& L = l->h[lane];
  if (boost) {
    if (boost_len < l->g->max_ol + 1) return fail(-1, "boost vector shorter than max_olabel + 1");
    if (l->boost_cap[lane] < boost_len) {
      CUDA_TRY(cudaStreamSynchronize(l->stream));
      dfree(l->boost_buf[lane]);
      CUDA_TRY(dalloc(&l->boost_buf[lane], (size_t)boost_len));
      l->boost_cap[lane] = boost_len;
    }
    CUDA_TRY(cudaMemcpyAsync(l->boost_buf[lane], boost, (size_t)boost_len * sizeof(double),
                             cudaMemcpyHostToDevice, l->stream));
    L.boost = l->boost_buf[lane];
    L.boost_len = (int32_t)boost_len;
  } else {
    L.boost = nullptr;
    L.boost_len = 0;
  }
  L.prune_ok = prune_flag(l, boost, boost_len, key_space(l, L)) &&
               !(L.fsa_next && l->g->eps_olabel && l->fsa_min[lane] < 0);
  if (int r = sync_lane(l, lane)) return r;
  CUDA_TRY(cudaStreamSynchronize(l->stream));
  return 0;
}

int ctw_lane_set_fsa(ctw_lanes* l, int32_t lane, int32_t n_states, const uint16_t* next, const double* cost) {
  std::lock_guard<std::mutex> lk(l->mu);
  CUDA_TRY(cudaSetDevice(l->g->device));
  if (lane < 0 || lane >= l->n) return fail(-1, "lane id out of range");
  CtwLane& L = l->h[lane];
  if (n_states <= 0) {
    L.fsa_next = nullptr;
    L.fsa_cost = nullptr;
    L.fsa_states = L.fsa_width = 0;
    L.sbits = 0;
    L.smask = 0xFFFFFFFFu;
    l->fsa_min[lane] = 0.0;
    return sync_lane(l, lane);
  }
  const uint32_t sbits = std::max<uint32_t>(1, ceil_log2((uint64_t)l->g->S));
  if (sbits >= 32 || (uint64_t)n_states > ((1ull << (32 - sbits)) - 1))
    return fail(-1, "phrase automaton has too many states for this graph's token keys");
  const int64_t width = l->g->max_ol + 1;
  const int64_t cells = (int64_t)n_states * width;
  for (int64_t k = 0; k < cells; ++k)
    if (next[k] >= n_states) return fail(-1, "phrase automaton transition out of range");
  if (l->fsa_cap[lane] < cells) {
    CUDA_TRY(cudaStreamSynchronize(l->stream));
    dfree(l->fsa_next[lane]);
    dfree(l->fsa_cost[lane]);
    CUDA_TRY(dalloc(&l->fsa_next[lane], (size_t)cells));
    CUDA_TRY(dalloc(&l->fsa_cost[lane], (size_t)std::max<int64_t>(cells / width, n_states)));
    l->fsa_cap[lane] = cells;
  }
  CUDA_TRY(cudaMemcpyAsync(l->fsa_next[lane], next, (size_t)cells * 2, cudaMemcpyHostToDevice, l->stream));
  CUDA_TRY(cudaMemcpyAsync(l->fsa_cost[lane], cost, (size_t)n_states * 8, cudaMemcpyHostToDevice, l->stream));
  double mn = 0.0;
  for (int32_t b = 0; b < n_states; ++b) mn = std::min(mn, cost[b]);
  l->fsa_min[lane] = mn;
  L.fsa_next = l->fsa_next[lane];
  L.fsa_cost = l->fsa_cost[lane];
  L.fsa_states = n_states;
  L.fsa_width = (int32_t)width;
  L.sbits = sbits;
  L.smask = (1u << sbits) - 1u;
  if (int r = sync_lane(l, lane)) return r;
  CUDA_TRY(cudaStreamSynchronize(l->stream));  // host arrays may go away
  return 0;
}

}  // extern "C"

namespace {

// Best-path scratch for n lanes (device arrays + pinned mirrors).
int best_prepare(ctw_lanes* l, int n) {
  if (n <= l->best_cap) return 0;
  const int c = std::max(n, 2 * l->best_cap);
  dfree(l->d_woff);
  dfree(l->d_wcap);
  dfree(l->d_nwords);
  dfree(l->d_tcost);
  dfree(l->d_bstatus);
  for (void* p : {(void*)l->h_woff, (void*)l->h_wcap, (void*)l->h_nwords, (void*)l->h_tcost, (void*)l->h_bstatus})
    if (p) cudaFreeHost(p);
  CUDA_TRY(dalloc(&l->d_woff, c));
  CUDA_TRY(dalloc(&l->d_wcap, c));
  CUDA_TRY(dalloc(&l->d_nwords, c));
  CUDA_TRY(dalloc(&l->d_tcost, c));
  CUDA_TRY(dalloc(&l->d_bstatus, c));
  CUDA_TRY(cudaMallocHost((void**)&l->h_woff, c * sizeof(long long)));
  CUDA_TRY(cudaMallocHost((void**)&l->h_wcap, c * sizeof(int)));
  CUDA_TRY(cudaMallocHost((void**)&l->h_nwords, c * sizeof(int)));
  CUDA_TRY(cudaMallocHost((void**)&l->h_tcost, c * sizeof(double)));
  CUDA_TRY(cudaMallocHost((void**)&l->h_bstatus, c * sizeof(int)));
  l->best_cap = c;
  return 0;
}

// Enqueue k_best_path over the n lanes whose ids are in l->d_ids (uploaded
// from l->h_ids when `upload_ids`) with word windows caps[], and the copies
// of its results into the pinned mirrors. No synchronisation.
// host half of best_enqueue: buffers sized, word windows in the pinned
// mirrors; *tot_out = total window
int best_host(ctw_lanes* l, int n, const std::vector<int>& caps, long long* tot_out) {
  if (int r = best_prepare(l, n)) return r;
  long long tot = 0;
  for (int i = 0; i < n; ++i) {
    l->h_woff[i] = tot;
    l->h_wcap[i] = caps[i];
    tot += caps[i];
  }
  if ((size_t)tot > l->words_cap) {
    dfree(l->d_words);
    CUDA_TRY(dalloc(&l->d_words, (size_t)tot + tot / 2));
    l->words_cap = (size_t)tot + tot / 2;
  }
  if ((size_t)tot > l->h_words_cap) {
    CUDA_TRY(cudaStreamSynchronize(l->stream));  // (the old pinned window may still be a copy target)
    if (l->h_words) cudaFreeHost(l->h_words);
    CUDA_TRY(cudaMallocHost((void**)&l->h_words, ((size_t)tot + tot / 2) * sizeof(int32_t)));
    l->h_words_cap = (size_t)tot + tot / 2;
  }
  *tot_out = tot;
  return 0;
}

// device half: window uploads, k_best_path, the per-lane result copies
// (graph-capturable: fixed sizes for a given n)
int best_device(ctw_lanes* l, int n, bool upload_ids) {
  ctw_graph* g = l->g;
  if (upload_ids) CUDA_TRY(cudaMemcpyAsync(l->d_ids, l->h_ids, n * sizeof(int), cudaMemcpyHostToDevice, l->stream));
  CUDA_TRY(cudaMemcpyAsync(l->d_woff, l->h_woff, n * sizeof(long long), cudaMemcpyHostToDevice, l->stream));
  CUDA_TRY(cudaMemcpyAsync(l->d_wcap, l->h_wcap, n * sizeof(int), cudaMemcpyHostToDevice, l->stream));
  if (ctw_launch_best(l->d, g->ranges, g->arcs, g->olabel, g->final_w, l->d_ids, n, l->d_words, l->d_woff,
                      l->d_wcap, l->d_nwords, l->d_tcost, l->d_bstatus, l->bpc, l->stream))
    return fail(-1, std::string("best-path launch: ") + cudaGetErrorString(cudaGetLastError()));
  CUDA_TRY(cudaMemcpyAsync(l->h_nwords, l->d_nwords, n * sizeof(int), cudaMemcpyDeviceToHost, l->stream));
  CUDA_TRY(cudaMemcpyAsync(l->h_tcost, l->d_tcost, n * sizeof(double), cudaMemcpyDeviceToHost, l->stream));
  CUDA_TRY(cudaMemcpyAsync(l->h_bstatus, l->d_bstatus, n * sizeof(int), cudaMemcpyDeviceToHost, l->stream));
  return 0;
}

int best_words(ctw_lanes* l, long long tot) {
  if (tot) CUDA_TRY(cudaMemcpyAsync(l->h_words, l->d_words, (size_t)tot * sizeof(int32_t), cudaMemcpyDeviceToHost,
                                    l->stream));
  return 0;
}

int best_enqueue(ctw_lanes* l, int n, const std::vector<int>& caps, bool upload_ids) {
  long long tot = 0;
  if (int r = best_host(l, n, caps, &tot)) return r;
  if (int r = best_device(l, n, upload_ids)) return r;
  l->launches++;
  return best_words(l, tot);
}

// Results of a completed best_enqueue in the reference layout (status 2 = no
// frames decoded yet; words oldest first, word_off[n] = total).
int best_finish(ctw_lanes* l, const int32_t* lane_ids, int n, int32_t* words, int64_t words_cap, int64_t* word_off,
                double* total_cost, int64_t* frame_count, int32_t* status) {
  int64_t need = 0;
  for (int i = 0; i < n; ++i) {
    const CtwLane& L = l->h[lane_ids[i]];
    word_off[i] = need;
    frame_count[i] = L.frame_count;
    if (L.frame_count == 0) {
      status[i] = 2;
      total_cost[i] = INFINITY;
      continue;
    }
    status[i] = l->h_bstatus[i];
    total_cost[i] = l->h_tcost[i];
    if (status[i] == 0) need += l->h_nwords[i];
  }
  word_off[n] = need;
  if (need > words_cap) return -2;
  for (int i = 0; i < n; ++i) {
    if (status[i] != 0 || l->h_nwords[i] == 0) continue;
    std::memcpy(words + word_off[i], l->h_words + l->h_woff[i], l->h_nwords[i] * sizeof(int32_t));
  }
  return 0;
}

int best_path_impl(ctw_lanes* l, const int32_t* lane_ids, int32_t n, int32_t* words, int64_t words_cap,
                   int64_t* word_off, double* total_cost, int64_t* frame_count, int32_t* status) {
  NvtxRange nvtx_("ctw_best_path");
  ctw_graph* g = l->g;
  CUDA_TRY(cudaSetDevice(g->device));
  if (n <= 0) {
    word_off[0] = 0;
    return 0;
  }
  for (int i = 0; i < n; ++i)
    if (lane_ids[i] < 0 || lane_ids[i] >= l->n) return fail(-1, "lane id out of range");
  if (int r = ensure_scratch(l, n)) return r;
  // capacity guess: one word per frame is generous for word-level graphs
  std::vector<int> caps(n);
  for (int i = 0; i < n; ++i) caps[i] = l->h[lane_ids[i]].frame_count + 8;
  for (int i = 0; i < n; ++i) l->h_ids[i] = lane_ids[i];
  for (int round = 0; round < 2; ++round) {
    if (int r = best_enqueue(l, n, caps, true)) return r;
    CUDA_TRY(cudaStreamSynchronize(l->stream));
    bool redo = false;
    for (int i = 0; i < n; ++i)
      if (l->h_nwords[i] > caps[i]) {
        caps[i] = l->h_nwords[i];
        redo = true;
      }
    if (!redo) break;
  }
  return best_finish(l, lane_ids, n, words, words_cap, word_off, total_cost, frame_count, status);
}

// The frame kernel over lanes `lane_ids` (grow-and-rerun protocol). With
// `bp`, the partial best path of every lane is enqueued right behind the
// first decode launch (the common case needs no re-run) and comes back with
// the same synchronisation; *bp_valid says whether it can be used (false
// after a re-run or a too-small word window: the caller runs it again).
int advance_impl(ctw_lanes* l, const int32_t* lane_ids, int32_t n, const void* loglik, int32_t dtype,
                 int32_t location, const int64_t* ll_offsets, const int32_t* frames, int32_t width,
                 int32_t* status, int32_t* err_frame, std::vector<int>* bp, bool* bp_valid) {
  NvtxRange nvtx_("ctw_advance");
  ctw_graph* g = l->g;
  if (bp_valid) *bp_valid = false;
  CUDA_TRY(cudaSetDevice(g->device));
  if (n <= 0) return 0;
  using clk = std::chrono::steady_clock;
  auto secs = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); };
  const clk::time_point t0 = clk::now();
  l->h_calls++;
  if (int r = check_ids(l, lane_ids, n)) return r;
  if (dtype != 0 && dtype != 1) return fail(-1, "dtype must be 0 (f32) or 1 (f64)");
  if (width < g->max_il) return fail(-1, "frame width smaller than the graph's max input label");
  const size_t esz = dtype ? 8 : 4;
  for (int i = 0; i < n; ++i) {
    if (!l->seeded[lane_ids[i]]) return fail(-1, "lane not seeded (call ctw_lane_reset first)");
    if (frames[i] < 0) return fail(-1, "negative frame count");
  }
  // stage host rows into HBM (one copy when the chunks are contiguous)
  const char* dev_ll = nullptr;
  if (int r = ensure_scratch(l, n)) return r;
  if (int r = stage_rows(l, loglik, location, esz, ll_offsets, frames, n, width, &dev_ll)) return r;
  const clk::time_point t1 = clk::now();
  l->h_stage += secs(t0, t1);
  // pre-size per-lane frame / history capacity
  for (int i = 0; i < n; ++i) {
    const int lane = lane_ids[i];
    CtwLane& L = l->h[lane];
    if (int r = grow_frames(l, lane, (int64_t)L.frame_count + frames[i])) return r;
    // history is paged (growing never copies a record), so reserve for the
    // worst case: max_active survivors per frame (or twice the observed
    // rate when max_active is effectively unbounded)
    const double ema = l->surv_ema[lane];
    const double est = std::min<double>((double)l->cfg.max_active, std::max(ema < 0 ? 65536.0 : 2.0 * ema, 4096.0));
    // (a presize estimate never asks for more than the int32 record range;
    // the kernel's exact request is checked when it is made)
    const int64_t need = std::min<int64_t>(L.n_rec + (int64_t)std::ceil(est * frames[i]) + 64, INT32_MAX);
    if (need > L.rcap)
      if (int r = grow_hist(l, lane, need)) return r;
  }
  std::vector<int> pos(l->n, -1);
  for (int i = 0; i < n; ++i) pos[lane_ids[i]] = i;
  std::vector<int> todo(lane_ids, lane_ids + n);
  l->h_presize += secs(t1, clk::now());
  for (int round = 0; !todo.empty(); ++round) {
    if (round > 60) return fail(-1, "advance: grow loop did not converge");
    if (round) l->h_reruns++;
    const clk::time_point tl = clk::now();
    const int m = (int)todo.size();
    for (int k = 0; k < m; ++k) {
      const int i = pos[todo[k]];
      l->h_ids[k] = todo[k];
      l->h_nframes[k] = frames[i];
      l->h_lloff[k] = (long long)ll_offsets[i];
    }
    int any_fsa = 0;
    for (int k = 0; k < m; ++k) any_fsa |= l->h[todo[k]].fsa_next != nullptr;
    const bool fast = fast_launch(l, l->h_ids, m);
    l->fast_launches += fast;
    // the device work of this round (capturable: fixed sizes for a given m)
    // (under stream capture the timing events must be external event nodes:
    // a plain record only orders the capture)
    auto device_round = [&](bool with_best, bool capture) -> int {
      const unsigned evf = capture ? cudaEventRecordExternal : cudaEventRecordDefault;
      CUDA_TRY(cudaMemcpyAsync(l->d_ids, l->h_ids, m * sizeof(int), cudaMemcpyHostToDevice, l->stream));
      CUDA_TRY(cudaMemcpyAsync(l->d_nframes, l->h_nframes, m * sizeof(int), cudaMemcpyHostToDevice, l->stream));
      CUDA_TRY(cudaMemcpyAsync(l->d_lloff, l->h_lloff, m * sizeof(long long), cudaMemcpyHostToDevice, l->stream));
      CUDA_TRY(cudaEventRecordWithFlags(l->ev0, l->stream, evf));
      if (ctw_launch_decode(l->d, g->ranges, g->arcs, g->olabel, g->final_w, dev_ll, dtype, width, l->d_lloff,
                            l->d_nframes, l->d_ids, m, &l->dcfg, l->d_out, any_fsa, fast ? 1 : 0, (int)g->ebits,
                            g->eps_olabel ? 1 : 0, l->stream))
        return fail(-1, std::string("decode launch: ") + cudaGetErrorString(cudaGetLastError()));
      CUDA_TRY(cudaEventRecordWithFlags(l->ev1, l->stream, evf));
      // partial best paths behind the decode (lane ids already on the device)
      if (with_best)
        if (int r = best_device(l, m, false)) return r;
      CUDA_TRY(cudaMemcpyAsync(l->h_out, l->d_out, m * sizeof(CtwLaneOut), cudaMemcpyDeviceToHost, l->stream));
      return 0;
    };
    const bool with_best = bp && round == 0;
    long long btot = 0;
    if (with_best) {
      if (int r = bpc_ensure(l)) return r;
      bp->resize(m);
      for (int k = 0; k < m; ++k) (*bp)[k] = l->h[todo[k]].frame_count + l->h_nframes[k] + 8;
      if (int r = best_host(l, m, *bp, &btot)) return r;
    }
    // a streaming step (the first round of ctw_advance_best) runs as one CUDA
    // graph launch: the graph of this launch shape is captured once and
    // replayed (parameters live in the pinned mirrors it copies from)
    cudaGraphExec_t exec = nullptr;
    if (with_best && !l->graphs_off && m <= 64 && getenv("CTW_NO_GRAPH") == nullptr) {
      {
        const uintptr_t key[13] = {(uintptr_t)m, (uintptr_t)(fast ? 1 : 0) | (uintptr_t)any_fsa << 1,
                                   (uintptr_t)dtype, (uintptr_t)width, (uintptr_t)dev_ll, (uintptr_t)l->d,
                                   (uintptr_t)l->d_ids, (uintptr_t)l->h_ids, (uintptr_t)l->d_woff,
                                   (uintptr_t)l->h_woff, (uintptr_t)l->d_words, (uintptr_t)l->h_out,
                                   (uintptr_t)l->bpc.n};
        for (auto& sg : l->step_graphs)
          if (std::equal(key, key + 13, sg.key)) exec = sg.exec;
        if (!exec) {
          cudaGraph_t graph = nullptr;
          int rc = (int)cudaStreamBeginCapture(l->stream, cudaStreamCaptureModeThreadLocal);
          if (rc == 0) {
            rc = device_round(true, true);
            cudaGraph_t gr = nullptr;
            const cudaError_t ec = cudaStreamEndCapture(l->stream, &gr);
            graph = gr;
            if (rc == 0 && ec != cudaSuccess) rc = (int)ec;
          }
          if (rc == 0 && graph && cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
            exec = nullptr;
            rc = -1;
          }
          if (graph) cudaGraphDestroy(graph);
          (void)cudaGetLastError();
          if (rc != 0 || !exec) {
            l->graphs_off = true;  // capture not possible here: plain stream launches from now on
            exec = nullptr;
          } else {
            if (l->step_graphs.size() >= 32) {
              cudaGraphExecDestroy(l->step_graphs.front().exec);
              l->step_graphs.erase(l->step_graphs.begin());
            }
            ctw_lanes::StepGraph sg;
            std::copy(key, key + 13, sg.key);
            sg.exec = exec;
            l->step_graphs.push_back(sg);
            l->graph_builds++;
          }
        }
      }
    }
    if (exec) {
      CUDA_TRY(cudaGraphLaunch(exec, l->stream));
      l->graph_launches++;
    } else {
      if (int r = device_round(with_best, false)) return r;
    }
    if (with_best)
      if (int r = best_words(l, btot)) return r;
    l->launches += with_best ? 2 : 1;
    l->decode_launches++;
    CUDA_TRY(cudaStreamSynchronize(l->stream));
    const clk::time_point tw = clk::now();
    l->h_wait += secs(tl, tw);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, l->ev0, l->ev1);
    l->decode_ms += ms;
    std::vector<int> again;
    for (int k = 0; k < m; ++k) {
      const int lane = todo[k];
      const int i = pos[lane];
      const CtwLaneOut& o = l->h_out[k];
      CtwLane& L = l->h[lane];
      l->max_slots = std::max<int64_t>(l->max_slots, o.n_slots_max);
      if (o.status >= CTW_GROW_TABLE && o.status <= CTW_GROW_SRC) l->h_grow[o.status - CTW_GROW_TABLE]++;
      // a grow that cannot be satisfied (device memory, or the int32
      // record range) fails this lane alone with CTW_ERR_OOM -- its chunk is
      // not committed and the lane keeps its state -- while the other lanes
      // of the launch go on (the reference's per-channel MemoryError)
      int gr = 0;
      if (o.status == CTW_GROW_TABLE) {
        gr = alloc_table(l, lane, L.tlog2 + 1);
      } else if (o.status == CTW_GROW_SRC) {
        gr = alloc_table(l, lane, L.tlog2, std::max<int64_t>(o.rec_need, 2 * (int64_t)L.scap));
      } else if (o.status == CTW_GROW_HIST) {
        const int64_t per = (o.rec_need - L.n_rec) / std::max(1, o.err_frame + 1) + 1;
        const int64_t want = L.n_rec + (int64_t)(per * 1.5 * frames[i]) + 64;
        gr = grow_hist(l, lane, o.rec_need > INT32_MAX ? o.rec_need : std::min<int64_t>(want, INT32_MAX));
      } else if (o.status == CTW_GROW_POOL) {
        gr = grow_pool(l, lane, 2 * (int64_t)L.pcap);
      }
      if (o.status >= CTW_GROW_TABLE && o.status <= CTW_GROW_SRC) {
        if (gr == 0) {
          again.push_back(lane);
        } else if (gr == -100 - (int)cudaErrorMemoryAllocation || gr == -1 || gr == -3) {
          (void)cudaGetLastError();
          status[i] = CTW_ERR_OOM;
          err_frame[i] = 0;
        } else {
          return gr;
        }
        continue;
      } else {
        const int64_t before = L.n_rec;
        update_from_out(L, o);
        status[i] = o.status;
        err_frame[i] = o.err_frame;
        if (o.status == CTW_OK) {
          for (int k = 0; k < CTW_NPROF; ++k) l->prof[k] += o.prof[k];
          l->arcs += o.arcs_expanded;
          l->srcs += o.src_total;
          l->frames += frames[i];
          if (frames[i] > 0) {
            const double per = (double)(L.n_rec - before) / frames[i];
            l->surv_ema[lane] = l->surv_ema[lane] < 0 ? per : 0.5 * (l->surv_ema[lane] + per);
          }
        }
      }
    }
    if (bp && round == 0 && again.empty()) {
      *bp_valid = true;
      for (int k = 0; k < m; ++k)
        if (l->h_nwords[k] > (*bp)[k]) *bp_valid = false;  // a word window was too small
    }
    todo.swap(again);
    l->h_post += secs(tw, clk::now());
  }
  return 0;
}

}  // namespace

extern "C" {

int ctw_advance(ctw_lanes* l, const int32_t* lane_ids, int32_t n, const void* loglik, int32_t dtype,
                int32_t location, const int64_t* ll_offsets, const int32_t* frames, int32_t width,
                int32_t* status, int32_t* err_frame) {
  std::lock_guard<std::mutex> lk(l->mu);
  return advance_impl(l, lane_ids, n, loglik, dtype, location, ll_offsets, frames, width, status, err_frame,
                      nullptr, nullptr);
}

int ctw_advance_best(ctw_lanes* l, const int32_t* lane_ids, int32_t n, const void* loglik, int32_t dtype,
                     int32_t location, const int64_t* ll_offsets, const int32_t* frames, int32_t width,
                     int32_t* status, int32_t* err_frame, int32_t* words, int64_t words_cap, int64_t* word_off,
                     double* total_cost, int64_t* frame_count, int32_t* bstatus) {
  std::lock_guard<std::mutex> lk(l->mu);
  if (n <= 0) {
    word_off[0] = 0;
    return 0;
  }
  std::vector<int> caps;
  bool ok = false;
  if (int r = advance_impl(l, lane_ids, n, loglik, dtype, location, ll_offsets, frames, width, status, err_frame,
                           &caps, &ok))
    return r;
  if (!ok) return best_path_impl(l, lane_ids, n, words, words_cap, word_off, total_cost, frame_count, bstatus);
  return best_finish(l, lane_ids, n, words, words_cap, word_off, total_cost, frame_count, bstatus);
}

int ctw_lanes_set_search(ctw_lanes* l, int32_t mode) {
  if (mode != 0 && mode != 1) return fail(-1, "search mode must be 0 (exact) or 1 (fast)");
  std::lock_guard<std::mutex> lk(l->mu);
  l->search = mode;
  return 0;
}

int ctw_lanes_search_info(ctw_lanes* l, int64_t* out3) {
  std::lock_guard<std::mutex> lk(l->mu);
  out3[0] = l->search;
  out3[1] = l->fast_launches;
  out3[2] = l->decode_launches;
  return 0;
}

int ctw_lanes_graph_info(ctw_lanes* l, int64_t* out3) {
  std::lock_guard<std::mutex> lk(l->mu);
  out3[0] = l->graph_launches;
  out3[1] = l->graph_builds;
  out3[2] = l->graphs_off ? 1 : 0;
  return 0;
}

int ctw_lanes_host_timing(ctw_lanes* l, double* out) {
  std::lock_guard<std::mutex> lk(l->mu);
  out[0] = l->h_stage;
  out[1] = l->h_presize;
  out[2] = l->h_wait;
  out[3] = l->h_post;
  out[4] = (double)l->h_reruns;
  out[5] = (double)l->h_calls;
  for (int k = 0; k < 4; ++k) out[6 + k] = (double)l->h_grow[k];
  return 0;
}

int ctw_best_path(ctw_lanes* l, const int32_t* lane_ids, int32_t n, int32_t* words, int64_t words_cap,
                  int64_t* word_off, double* total_cost, int64_t* frame_count, int32_t* status) {
  std::lock_guard<std::mutex> lk(l->mu);
  return best_path_impl(l, lane_ids, n, words, words_cap, word_off, total_cost, frame_count, status);
}

int ctw_lane_compact(ctw_lanes* l, const int32_t* lane_ids, int32_t n, int64_t* kept) {
  NvtxRange nvtx_("ctw_lane_compact");
  std::lock_guard<std::mutex> lk(l->mu);
  CUDA_TRY(cudaSetDevice(l->g->device));
  if (n <= 0) return 0;
  if (int r = check_ids(l, lane_ids, n)) return r;
  cudaStream_t st = l->stream;
  std::vector<uint32_t*> marks(n, nullptr);
  std::vector<int32_t*> newidx(n, nullptr);
  std::vector<CtwRecPage**> nptab(n, nullptr);
  std::vector<std::vector<CtwRecPage*>> npages(n);
  auto take_page = [&]() -> CtwRecPage* {
    if (l->free_pages.empty()) {
      CtwRecPage* slab = nullptr;
      if (salloc(&slab, CTW_SLAB, st) != cudaSuccess) return nullptr;
      l->slabs.push_back(slab);
      for (int k = CTW_SLAB - 1; k >= 0; --k) l->free_pages.push_back(slab + k);
    }
    CtwRecPage* p = l->free_pages.back();
    l->free_pages.pop_back();
    return p;
  };
  for (int i = 0; i < n; ++i) {
    const CtwLane& L = l->h[lane_ids[i]];
    const int64_t R = L.n_rec;
    const int64_t W = (R + 31) / 32 + 1;
    CUDA_TRY(salloc(&marks[i], (size_t)W, st));
    CUDA_TRY(cudaMemsetAsync(marks[i], 0, (size_t)W * 4, st));
    CUDA_TRY(salloc(&newidx[i], (size_t)R + 1, st));
    const int64_t np = std::max<int64_t>(1, (R + CTW_PAGE - 1) / CTW_PAGE);  // worst case: all kept
    for (int64_t k = 0; k < np; ++k) {
      CtwRecPage* p = take_page();
      if (!p) return fail(-3, "out of memory for history pages");
      npages[i].push_back(p);
    }
    CUDA_TRY(salloc(&nptab[i], (size_t)np, st));
    CUDA_TRY(cudaMemcpyAsync(nptab[i], npages[i].data(), np * sizeof(CtwRecPage*), cudaMemcpyHostToDevice, st));
  }
  if (int r = ensure_scratch(l, n)) return r;
  for (int i = 0; i < n; ++i) l->h_ids[i] = lane_ids[i];
  uint32_t** d_marks = nullptr;
  int32_t** d_newidx = nullptr;
  CtwRecPage*** d_nptab = nullptr;
  long long* d_kept = nullptr;
  CUDA_TRY(salloc(&d_marks, (size_t)n, st));
  CUDA_TRY(salloc(&d_newidx, (size_t)n, st));
  CUDA_TRY(salloc(&d_nptab, (size_t)n, st));
  CUDA_TRY(salloc(&d_kept, (size_t)n, st));
  CUDA_TRY(cudaMemcpyAsync(l->d_ids, l->h_ids, n * sizeof(int), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d_marks, marks.data(), n * sizeof(uint32_t*), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d_newidx, newidx.data(), n * sizeof(int32_t*), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d_nptab, nptab.data(), n * sizeof(CtwRecPage**), cudaMemcpyHostToDevice, st));
  if (ctw_launch_hist_mark(l->d, l->d_ids, d_marks, n, st) ||
      ctw_launch_hist_compact(l->d, l->d_ids, d_marks, d_newidx, d_nptab, d_kept, n, st))
    return fail(-1, std::string("history compaction launch: ") + cudaGetErrorString(cudaGetLastError()));
  std::vector<long long> kv(n);
  CUDA_TRY(cudaMemcpyAsync(kv.data(), d_kept, n * sizeof(long long), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  for (int i = 0; i < n; ++i) {
    const int lane = lane_ids[i];
    CtwLane& L = l->h[lane];
    // the lane adopts the first pages of the new set; the rest and the old
    // pages go back to the free list
    const int64_t keep_pages = std::max<int64_t>(1, (kv[i] + CTW_PAGE - 1) / CTW_PAGE);
    for (CtwRecPage* p : l->hpages[lane]) l->free_pages.push_back(p);
    l->hpages[lane].assign(npages[i].begin(), npages[i].begin() + keep_pages);
    for (size_t k = (size_t)keep_pages; k < npages[i].size(); ++k) l->free_pages.push_back(npages[i][k]);
    if ((int64_t)l->hpages[lane].size() > l->ptab_cap[lane]) {
      sfree(L.pages, st);
      CUDA_TRY(salloc(&L.pages, l->hpages[lane].size(), st));
      l->ptab_cap[lane] = (int64_t)l->hpages[lane].size();
    }
    CUDA_TRY(cudaMemcpyAsync(L.pages, l->hpages[lane].data(), l->hpages[lane].size() * sizeof(CtwRecPage*),
                             cudaMemcpyHostToDevice, st));
    L.rcap = (int64_t)l->hpages[lane].size() * CTW_PAGE;
    L.n_rec = kv[i];
    l->compacted[lane] = 1;
    if (int r = bpc_clear(l, lane)) return r;
    if (kept) kept[i] = kv[i];
    if (int r = sync_lane(l, lane)) return r;
    sfree(marks[i], st);
    sfree(newidx[i], st);
    sfree(nptab[i], st);
  }
  sfree(d_marks, st);
  sfree(d_newidx, st);
  sfree(d_nptab, st);
  sfree(d_kept, st);
  CUDA_TRY(cudaStreamSynchronize(st));
  return 0;
}

int ctw_lanes_presize(ctw_lanes* l, const int32_t* lane_ids, int32_t n) {
  std::lock_guard<std::mutex> lk(l->mu);
  CUDA_TRY(cudaSetDevice(l->g->device));
  if (int r = check_ids(l, lane_ids, n)) return r;
  for (int i = 0; i < n; ++i) {
    CtwLane& L = l->h[lane_ids[i]];
    if (L.tlog2 < l->tlog2_hint)
      if (int r = alloc_table(l, lane_ids[i], l->tlog2_hint)) return r;
  }
  return 0;
}

int ctw_lane_info(ctw_lanes* l, int32_t lane, int64_t* frame_count, int64_t* n_tokens, int64_t* n_records) {
  std::lock_guard<std::mutex> lk(l->mu);
  if (lane < 0 || lane >= l->n) return fail(-1, "lane id out of range");
  const CtwLane& L = l->h[lane];
  if (frame_count) *frame_count = L.frame_count;
  if (n_tokens) *n_tokens = L.n_src;
  if (n_records) *n_records = L.n_rec;
  return 0;
}

int ctw_lane_capacity(ctw_lanes* l, int32_t lane, int64_t* out6) {
  std::lock_guard<std::mutex> lk(l->mu);
  if (lane < 0 || lane >= l->n) return fail(-1, "lane id out of range");
  if (!out6) return fail(-1, "null output");
  const CtwLane& L = l->h[lane];
  const uint64_t tcap = 1ull << L.tlog2;
  const int64_t scap = (int64_t)L.scap + 1;
  const int64_t bytes = (int64_t)(tcap * sizeof(CtwTok) + CTW_SLOTS_LEN(tcap) * sizeof(uint2) +
                                  CTW_FRONT_LEN(tcap) * sizeof(uint2)) +
                        scap * (int64_t)(3 * sizeof(CtwSrc) + sizeof(int32_t)) +
                        (int64_t)l->hpages[lane].size() * (int64_t)sizeof(CtwRecPage) +
                        (int64_t)L.fcap * (int64_t)sizeof(int64_t) + (int64_t)L.pcap * (int64_t)sizeof(int32_t);
  out6[0] = L.tlog2;
  out6[1] = L.scap;
  out6[2] = L.rcap;
  out6[3] = L.fcap;
  out6[4] = L.pcap;
  out6[5] = bytes;
  return 0;
}

void ctw_export_free(ctw_export* e) {
  if (!e) return;
  free(e->counts);
  free(e->rec_prev);
  free(e->rec_state);
  free(e->rec_cost);
  free(e->rec_olab_off);
  free(e->rec_olab_pool);
  free(e->tok_state);
  free(e->tok_cost);
  free(e->tok_bp);
  free(e->tok_chain_off);
  free(e->tok_chain_pool);
  std::memset(e, 0, sizeof(*e));
}

}  // extern "C"

namespace {
template <class T>
T* cmalloc(size_t n) {
  return (T*)malloc(std::max<size_t>(n, 1) * sizeof(T));
}

void expand_code(const int32_t* pool, int32_t code, std::vector<int32_t>& out) {
  if (code > 0) out.push_back(code);
  else if (code < 0) {
    const int64_t off = -(int64_t)code - 1;
    const int32_t m = pool[off];
    for (int32_t j = 0; j < m; ++j) out.push_back(pool[off + 1 + j]);
  }
}
}  // namespace

extern "C" {

int ctw_lane_export(ctw_lanes* l, int32_t lane, int64_t frame_from, int64_t base, const int64_t* ext_bp,
                    int64_t n_ext, ctw_export* out) {
  std::lock_guard<std::mutex> lk(l->mu);
  std::memset(out, 0, sizeof(*out));
  CUDA_TRY(cudaSetDevice(l->g->device));
  if (lane < 0 || lane >= l->n) return fail(-1, "lane id out of range");
  const CtwLane& L = l->h[lane];
  const int64_t F = L.frame_count, R = L.n_rec;
  if (frame_from < 0 || frame_from > F) return fail(-1, "frame_from out of range");
  std::vector<int64_t> fb((size_t)F);
  std::vector<int2> link((size_t)R);
  std::vector<int32_t> st((size_t)R), pool((size_t)L.pool_used);
  std::vector<double> cost((size_t)R);
  const auto& pages = l->hpages[lane];
  std::vector<CtwSrc> src((size_t)L.n_src);
  std::vector<int32_t> pend((size_t)(L.pend_valid ? L.n_src : 0));
  if (F) CUDA_TRY(cudaMemcpyAsync(fb.data(), L.frame_base, F * 8, cudaMemcpyDeviceToHost, l->stream));
  for (int64_t r0 = 0; r0 < R; r0 += CTW_PAGE) {
    const CtwRecPage* p = pages[(size_t)(r0 >> CTW_PAGE_LOG2)];
    const size_t m = (size_t)std::min<int64_t>(CTW_PAGE, R - r0);
    CUDA_TRY(cudaMemcpyAsync(link.data() + r0, p->link, m * sizeof(int2), cudaMemcpyDeviceToHost, l->stream));
    CUDA_TRY(cudaMemcpyAsync(st.data() + r0, p->state, m * 4, cudaMemcpyDeviceToHost, l->stream));
    CUDA_TRY(cudaMemcpyAsync(cost.data() + r0, p->cost, m * 8, cudaMemcpyDeviceToHost, l->stream));
  }
  if (L.pool_used)
    CUDA_TRY(cudaMemcpyAsync(pool.data(), L.pool, L.pool_used * 4, cudaMemcpyDeviceToHost, l->stream));
  if (L.n_src)
    CUDA_TRY(cudaMemcpyAsync(src.data(), L.src[L.src_buf], L.n_src * sizeof(CtwSrc), cudaMemcpyDeviceToHost,
                             l->stream));
  if (!pend.empty())
    CUDA_TRY(cudaMemcpyAsync(pend.data(), L.pend, pend.size() * 4, cudaMemcpyDeviceToHost, l->stream));
  CUDA_TRY(cudaStreamSynchronize(l->stream));
  // per frame: order by state; global index = base + rank
  std::vector<int64_t> gidx((size_t)R);
  std::vector<int64_t> order;
  order.reserve((size_t)R);
  for (int64_t f = 0; f < F; ++f) {
    const int64_t b = fb[f], e = (f + 1 < F) ? fb[f + 1] : R;
    const size_t o0 = order.size();
    for (int64_t r = b; r < e; ++r) order.push_back(r);
    std::sort(order.begin() + o0, order.end(), [&](int64_t x, int64_t y) { return st[x] < st[y]; });
    for (size_t k = o0; k < order.size(); ++k) gidx[order[k]] = base + (int64_t)k;
  }
  auto map_prev = [&](int32_t p) -> int64_t {
    if (p >= 0) return gidx[p];
    if (p == -1) return -1;
    const int64_t x = -2 - (int64_t)p;
    return (ext_bp && x < n_ext) ? ext_bp[x] : -1;
  };
  const int64_t r0 = frame_from < F ? fb[frame_from] : R;
  const int64_t nr = R - r0;
  out->n_frames = F - frame_from;
  out->n_records = nr;
  out->counts = cmalloc<int64_t>(out->n_frames);
  for (int64_t f = frame_from; f < F; ++f) out->counts[f - frame_from] = ((f + 1 < F) ? fb[f + 1] : R) - fb[f];
  out->rec_prev = cmalloc<int64_t>(nr);
  out->rec_state = cmalloc<int32_t>(nr);
  out->rec_cost = cmalloc<double>(nr);
  out->rec_olab_off = cmalloc<int64_t>(nr + 1);
  std::vector<int32_t> labs;
  out->rec_olab_off[0] = 0;
  for (int64_t k = 0; k < nr; ++k) {
    const int64_t r = order[(size_t)(r0 + k)];
    out->rec_prev[k] = map_prev(link[r].x);
    out->rec_state[k] = st[r];
    out->rec_cost[k] = cost[r];
    expand_code(pool.data(), link[r].y, labs);
    out->rec_olab_off[k + 1] = (int64_t)labs.size();
  }
  out->n_olab = (int64_t)labs.size();
  out->rec_olab_pool = cmalloc<int32_t>(labs.size());
  std::copy(labs.begin(), labs.end(), out->rec_olab_pool);
  // active tokens, state-ascending
  std::vector<int64_t> to((size_t)L.n_src);
  std::iota(to.begin(), to.end(), 0);
  std::sort(to.begin(), to.end(), [&](int64_t x, int64_t y) { return src[x].state < src[y].state; });
  out->n_tok = L.n_src;
  out->tok_state = cmalloc<int32_t>(L.n_src);
  out->tok_cost = cmalloc<double>(L.n_src);
  out->tok_bp = cmalloc<int64_t>(L.n_src);
  out->tok_chain_off = cmalloc<int64_t>(L.n_src + 1);
  std::vector<int32_t> ch;
  out->tok_chain_off[0] = 0;
  for (int64_t k = 0; k < L.n_src; ++k) {
    const CtwSrc& t = src[to[k]];
    out->tok_state[k] = t.state;
    out->tok_cost[k] = t.cost;
    out->tok_bp[k] = map_prev(t.bp);
    if (!pend.empty()) expand_code(pool.data(), pend[to[k]], ch);
    out->tok_chain_off[k + 1] = (int64_t)ch.size();
  }
  out->n_chain = (int64_t)ch.size();
  out->tok_chain_pool = cmalloc<int32_t>(ch.size());
  std::copy(ch.begin(), ch.end(), out->tok_chain_pool);
  return 0;
}

int ctw_lanes_stats(ctw_lanes* l, int64_t* launches, int64_t* decode_launches, double* decode_ms, int64_t* arcs,
                    int64_t* src_tokens, int64_t* frames, int64_t* max_slots) {
  std::lock_guard<std::mutex> lk(l->mu);
  if (launches) *launches = l->launches;
  if (decode_launches) *decode_launches = l->decode_launches;
  if (decode_ms) *decode_ms = l->decode_ms;
  if (arcs) *arcs = l->arcs;
  if (src_tokens) *src_tokens = l->srcs;
  if (frames) *frames = l->frames;
  if (max_slots) *max_slots = l->max_slots;
  return 0;
}

int ctw_lanes_reset_stats(ctw_lanes* l) {
  std::lock_guard<std::mutex> lk(l->mu);
  l->launches = l->decode_launches = l->arcs = l->srcs = l->frames = l->max_slots = 0;
  l->fast_launches = 0;
  l->h_stage = l->h_presize = l->h_wait = l->h_post = 0;
  l->h_reruns = l->h_calls = 0;
  for (auto& x : l->h_grow) x = 0;
  for (int k = 0; k < CTW_NPROF; ++k) l->prof[k] = 0;
  l->decode_ms = 0.0;
  return 0;
}

void* ctw_lanes_stream(ctw_lanes* l) { return (void*)l->stream; }

int ctw_lanes_profile(ctw_lanes* l, int64_t* out) {
  std::lock_guard<std::mutex> lk(l->mu);
  for (int k = 0; k < CTW_NPROF; ++k) out[k] = l->prof[k];
  return 0;
}

// ------------------------------------------------------------- compat ----
}  // extern "C"

namespace {
struct CompatCache {
  uint64_t hash = 0;
  int64_t S = -1, A = -1;
  int device = -1;
  ctw_graph* g = nullptr;
  ctw_lanes* l = nullptr;
};
std::mutex g_compat_mu;
CompatCache g_compat;

uint64_t fnv(uint64_t h, const void* p, size_t n) {
  const unsigned char* c = (const unsigned char*)p;
  for (size_t i = 0; i < n; ++i) h = (h ^ c[i]) * 1099511628211ull;
  return h;
}
}  // namespace

extern "C" {

int ctw_advance_chunk_compat(const int64_t* off, const int64_t* eps_end, const int32_t* ilabel,
                             const int32_t* olabel, const double* weight, const int32_t* nextstate,
                             int64_t num_states, int64_t num_arcs, const int32_t* act_state,
                             const double* act_cost, const int64_t* act_bp, const int64_t* act_chain_off,
                             const int32_t* act_chain_pool, int64_t n_src, const double* loglik,
                             int64_t num_frames, int64_t width, double acoustic_scale, double beam,
                             int64_t max_active, double relax_eps, int64_t max_ne_iters, const double* boost,
                             int64_t boost_len, int64_t base, int32_t device, int64_t* err_frame,
                             ctw_export* out) {
  std::lock_guard<std::mutex> lk(g_compat_mu);
  std::memset(out, 0, sizeof(*out));
  *err_frame = -1;
  // the reference kernel derives finals nowhere; use +inf (best path is not part of the contract)
  uint64_t h = 1469598103934665603ull;
  h = fnv(h, off, (size_t)(num_states + 1) * 8);
  h = fnv(h, eps_end, (size_t)num_states * 8);
  h = fnv(h, ilabel, (size_t)num_arcs * 4);
  h = fnv(h, olabel, (size_t)num_arcs * 4);
  h = fnv(h, weight, (size_t)num_arcs * 8);
  h = fnv(h, nextstate, (size_t)num_arcs * 4);
  CompatCache& c = g_compat;
  if (!(c.g && c.hash == h && c.S == num_states && c.A == num_arcs && c.device == device)) {
    if (c.l) ctw_lanes_destroy(c.l);
    if (c.g) ctw_graph_destroy(c.g);
    c = CompatCache();
    std::vector<double> fin((size_t)num_states, INFINITY);
    if (int r = ctw_graph_create(off, eps_end, ilabel, olabel, weight, nextstate, fin.data(), num_states, num_arcs,
                                 0, device, &c.g))
      return r;
    ctw_config cfg{beam, max_active, acoustic_scale, relax_eps, max_ne_iters};
    if (int r = ctw_lanes_create(c.g, 1, &cfg, nullptr, &c.l)) return r;
    c.hash = h;
    c.S = num_states;
    c.A = num_arcs;
    c.device = device;
  }
  ctw_lanes* l = c.l;
  if (!(beam > 0) || max_active < 1 || !(acoustic_scale > 0)) return fail(-1, "invalid decoder config");
  l->cfg = ctw_config{beam, max_active, acoustic_scale, relax_eps, max_ne_iters};
  l->dcfg = CtwDecodeCfg{beam, acoustic_scale, relax_eps, (long long)max_active, (long long)max_ne_iters};
  CUDA_TRY(cudaSetDevice(device));
  CtwLane& L = l->h[0];
  // table must hold the external sources
  while ((int64_t)CTW_LOAD(1ull << L.tlog2) < n_src)
    if (int r = alloc_table(l, 0, L.tlog2 + 1)) return r;
  if (L.scap < n_src)
    if (int r = alloc_table(l, 0, L.tlog2, n_src)) return r;
  if (boost && boost_len < c.g->max_ol + 1) return fail(-1, "boost vector shorter than max_olabel + 1");
  // load sources (bp = -2 - i refers back to act_bp[i]) and their pending chains
  std::vector<CtwSrc> srcs((size_t)n_src);
  std::vector<int32_t> pend((size_t)n_src, 0), pool;
  bool any_pend = false;
  for (int64_t i = 0; i < n_src; ++i) {
    if (act_state[i] < 0 || act_state[i] >= num_states) return fail(-1, "active state out of range");
    const int32_t st = act_state[i];
    srcs[i] = CtwSrc{st, (int32_t)(-2 - i), act_cost[i], (uint32_t)eps_end[st], (uint32_t)off[st + 1], -1, 0};
    const int64_t a0 = act_chain_off[i], a1 = act_chain_off[i + 1];
    if (a1 - a0 == 1) pend[i] = act_chain_pool[a0];
    else if (a1 - a0 > 1) {
      pend[i] = -(int32_t)pool.size() - 1;
      pool.push_back((int32_t)(a1 - a0));
      for (int64_t k = a0; k < a1; ++k) pool.push_back(act_chain_pool[k]);
    }
    any_pend |= a1 > a0;
  }
  if (int r = grow_pool(l, 0, (int64_t)pool.size() + 1)) return r;
  if (n_src) {
    CUDA_TRY(cudaMemcpyAsync(L.src[0], srcs.data(), n_src * sizeof(CtwSrc), cudaMemcpyHostToDevice, l->stream));
    CUDA_TRY(cudaMemcpyAsync(L.pend, pend.data(), n_src * 4, cudaMemcpyHostToDevice, l->stream));
  }
  if (!pool.empty())
    CUDA_TRY(cudaMemcpyAsync(L.pool, pool.data(), pool.size() * 4, cudaMemcpyHostToDevice, l->stream));
  double* dboost = nullptr;
  if (boost) {
    if (l->boost_cap[0] < boost_len) {
      dfree(l->boost_buf[0]);
      CUDA_TRY(dalloc(&l->boost_buf[0], (size_t)boost_len));
      l->boost_cap[0] = boost_len;
    }
    CUDA_TRY(cudaMemcpyAsync(l->boost_buf[0], boost, boost_len * 8, cudaMemcpyHostToDevice, l->stream));
    dboost = l->boost_buf[0];
  }
  auto load_state = [&]() -> int {
    L.n_src = (int32_t)n_src;
    L.src_buf = 0;
    L.frame_count = 0;
    L.pool_used = (int32_t)pool.size();
    L.n_rec = 0;
    L.pend_valid = any_pend ? 1 : 0;
    L.boost = dboost;
    L.boost_len = (int32_t)boost_len;
    L.prune_ok = prune_flag(l, boost, boost_len, key_space(l, L));
    l->seeded[0] = 1;
    return sync_lane(l, 0);
  };
  if (int r = load_state()) return r;
  int32_t lane = 0, st = 0, ef = -1;
  const int64_t zero = 0;
  int32_t nf = (int32_t)num_frames;
  if (num_frames > 0) {
    if (int r = ctw_advance(l, &lane, 1, loglik, 1, 0, &zero, &nf, (int32_t)width, &st, &ef)) return r;
    if (st != CTW_OK && ef > 0) {
      // the contract returns the frames completed before the failure: redo them
      if (int r = load_state()) return r;
      int32_t st2 = 0, ef2 = -1, nf2 = ef;
      if (int r = ctw_advance(l, &lane, 1, loglik, 1, 0, &zero, &nf2, (int32_t)width, &st2, &ef2)) return r;
      if (st2 != CTW_OK) return fail(-1, "compat: replay of completed frames failed");
    }
  }
  *err_frame = (st == CTW_OK) ? -1 : ef;
  if (st == CTW_OK || ef > 0) {
    if (int r = ctw_lane_export(l, 0, 0, base, act_bp, n_src, out)) return r;
  } else {
    out->counts = cmalloc<int64_t>(0);
    out->rec_prev = cmalloc<int64_t>(0);
    out->rec_state = cmalloc<int32_t>(0);
    out->rec_cost = cmalloc<double>(0);
    out->rec_olab_off = cmalloc<int64_t>(1);
    out->rec_olab_off[0] = 0;
    out->rec_olab_pool = cmalloc<int32_t>(0);
  }
  // leave the cached lane empty of history
  L.n_rec = 0;
  L.frame_count = 0;
  return st;
}


// ---------------------------------------------------------------- lattice --

void ctw_lattice_free(ctw_lattice* lat) {
  if (!lat) return;
  for (void* p : {(void*)lat->seed_state, (void*)lat->seed_cost, (void*)lat->seed_lab_off, (void*)lat->seed_lab,
                  (void*)lat->arc_src, (void*)lat->arc_dst, (void*)lat->arc_frame, (void*)lat->arc_dst_state,
                  (void*)lat->arc_src_state,
                  (void*)lat->arc_w, (void*)lat->arc_dst_final, (void*)lat->arc_lab_off, (void*)lat->arc_lab})
    free(p);
  std::memset(lat, 0, sizeof(*lat));
}

int ctw_lane_lattice(ctw_lanes* l, const int32_t* lane_ids, int32_t n, const void* loglik, int32_t dtype,
                int32_t location, const int64_t* ll_offsets, int32_t width, double lattice_beam,
                ctw_lattice* out) {
  NvtxRange nvtx_("ctw_lane_lattice");
  std::lock_guard<std::mutex> lk(l->mu);
  ctw_graph* g = l->g;
  CUDA_TRY(cudaSetDevice(g->device));
  if (n <= 0) return 0;
  if (int r = check_ids(l, lane_ids, n)) return r;
  if (dtype != 0 && dtype != 1) return fail(-1, "dtype must be 0 (f32) or 1 (f64)");
  if (!(lattice_beam >= 0)) return fail(-1, "lattice_beam must be >= 0");
  for (int i = 0; i < n; ++i) {
    std::memset(&out[i], 0, sizeof(out[i]));
    if (!l->seeded[lane_ids[i]]) return fail(-1, "lane not seeded (call ctw_lane_reset first)");
    if (l->compacted[lane_ids[i]]) return fail(-1, "lane history was garbage-collected: no lattice");
  }
  const size_t esz = dtype ? 8 : 4;
  using clk = std::chrono::steady_clock;
  const bool tm = getenv("CTW_LAT_TIMING") != nullptr;  // diagnostics: phase times on stderr
  clk::time_point tp = clk::now();
  auto lap = [&](const char* what) {
    if (!tm) return;
    const clk::time_point t = clk::now();
    fprintf(stderr, "lattice %s %.3f ms\n", what, std::chrono::duration<double>(t - tp).count() * 1e3);
    tp = t;
  };
  std::vector<int32_t> frames(n);
  for (int i = 0; i < n; ++i) frames[i] = l->h[lane_ids[i]].frame_count;
  const char* dev_ll = nullptr;
  if (int r = stage_rows(l, loglik, location, esz, ll_offsets, frames.data(), n, width, &dev_ll)) return r;
  // per-entry buffers; arc / label capacities grow and the lane re-runs on overflow
  std::vector<CtwLatEntry> ent(n);
  std::vector<int32_t> arc_cap(n), lab_cap(n);
  std::vector<char> big(n, 0);  // re-run with the large closure capacities
  for (int i = 0; i < n; ++i) {
    arc_cap[i] = 4096 + 256 * frames[i];  // ~40 kept arcs per frame at lattice beam 6 on C2
    lab_cap[i] = 4 * arc_cap[i];
  }
  // closure index (once per graph; CTW_LAT_NOPRE=1 runs the general kernel)
  const bool pre_env = getenv("CTW_LAT_NOPRE") == nullptr;
  if (pre_env && !g->eps_olabel) {
    std::lock_guard<std::mutex> gl(g->clo_mu);
    if (g->clo_state == 0) {
      const int rc = ctw_build_closure_index(g->ranges, g->arcs, g->S, &g->clo_off, &g->clo_ent, &g->clo_n,
                                             l->stream);
      if (rc == (int)cudaErrorMemoryAllocation) (void)cudaGetLastError();  // no room for the index: general kernel
      else if (rc > 0) return fail(-100 - rc, std::string("closure index: ") + cudaGetErrorString((cudaError_t)rc));
      g->clo_state = rc == 0 ? 1 : -1;
    }
  }
  const bool pre = pre_env && g->clo_state == 1;
  CtwLatEntry* d_ent = nullptr;
  CUDA_TRY(salloc(&d_ent, (size_t)n, l->stream));
  std::vector<int> todo(n);
  std::iota(todo.begin(), todo.end(), 0);
  std::vector<CtwLatArc*> d_arcs(n, nullptr);
  std::vector<int32_t*> d_lab(n, nullptr);
  std::vector<unsigned long long*> d_beta(n, nullptr);
  auto release = [&]() {
    for (int i = 0; i < n; ++i) {
      sfree(d_arcs[i], l->stream);
      sfree(d_lab[i], l->stream);
      sfree(d_beta[i], l->stream);
    }
    sfree(d_ent, l->stream);
  };
  for (int round = 0; !todo.empty(); ++round) {
    if (round > 6) {
      release();
      return fail(-1, "lattice: buffer growth did not converge");
    }
    const int m = (int)todo.size();
    for (int k = 0; k < m; ++k) {
      const int i = todo[k];
      const int lane = lane_ids[i];
      const CtwLane& L = l->h[lane];
      sfree(d_arcs[i], l->stream);
      sfree(d_lab[i], l->stream);
      if (!d_beta[i]) CUDA_TRY(salloc(&d_beta[i], (size_t)(l->seed_n[lane] + L.n_rec + 1), l->stream));
      CUDA_TRY(salloc(&d_arcs[i], (size_t)arc_cap[i], l->stream));
      CUDA_TRY(salloc(&d_lab[i], (size_t)lab_cap[i], l->stream));
      CtwLatEntry e{};
      e.lane = lane;
      e.n_seeds = l->seed_n[lane];
      e.seeds = l->seed_src[lane];
      e.ll_off = (long long)ll_offsets[i];
      e.arcs = d_arcs[i];
      e.arc_cap = arc_cap[i];
      e.lpool = d_lab[i];
      e.lpool_cap = lab_cap[i];
      e.beta = d_beta[i];
      // lower bound of any emitting step's graph part: min arc weight plus the
      // most negative boost (source-level pruning in the kernel)
      double bmin = 0.0;
      if (L.boost) {
        std::vector<double> hb((size_t)L.boost_len);
        CUDA_TRY(cudaMemcpy(hb.data(), L.boost, hb.size() * 8, cudaMemcpyDeviceToHost));
        for (double x : hb) bmin = std::min(bmin, x);
      }
      if (L.fsa_next) bmin = std::min(bmin, l->fsa_min[lane]);
      e.emit_lb = g->w_min_emit + bmin;
      ent[k] = e;
    }
    CUDA_TRY(cudaMemcpyAsync(d_ent, ent.data(), m * sizeof(CtwLatEntry), cudaMemcpyHostToDevice, l->stream));
    lap("setup");
    // CTAs per lane: up to 8 while the batch leaves SMs idle, bounded so a
    // rank's share of a layer fits its slice of the lane's frontier scratch;
    // a re-run after a closure overflow takes the large-capacity kernel on
    // one CTA per lane
    bool any_big = false;
    int ranks = 8;
    {
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      while (ranks > 1 && (int64_t)m * ranks > 4LL * sms) ranks >>= 1;
      for (int k = 0; k < m; ++k) {
        any_big |= big[todo[k]] != 0;
        const int64_t seg = (int64_t)CTW_LOAD(1ull << l->h[lane_ids[todo[k]]].tlog2);
        while (ranks > 1 && 512LL * ranks > 3 * seg) ranks >>= 1;
      }
      if (any_big) ranks = 1;
      if (const char* e = getenv("CTW_LAT_RANKS")) ranks = std::max(1, std::min(8, atoi(e)));  // diagnostics
    }
    if (ctw_launch_lattice(l->d, g->ranges, g->arcs, g->olabel, g->final_w, pre ? g->clo_off : nullptr,
                           pre ? g->clo_ent : nullptr, d_ent, m, dev_ll, dtype, width, l->cfg.acoustic_scale,
                           lattice_beam, ranks, any_big ? 1 : 0, l->stream)) {
      release();
      return fail(-1, std::string("lattice launch: ") + cudaGetErrorString(cudaGetLastError()));
    }
    l->launches++;
    CUDA_TRY(cudaMemcpyAsync(ent.data(), d_ent, m * sizeof(CtwLatEntry), cudaMemcpyDeviceToHost, l->stream));
    CUDA_TRY(cudaStreamSynchronize(l->stream));
    lap("kernel");
    std::vector<int> again;
    // stage every finished lane's device results first, into one pinned
    // buffer (one synchronisation): kept arcs, their label segments, the
    // seeds and the label-pool prefix their codes point into
    struct Host {
      const CtwLatArc* arcs = nullptr;
      const int32_t *lab = nullptr, *spend = nullptr, *pool = nullptr;
      const CtwSrc* seeds = nullptr;
    };
    std::vector<Host> hb((size_t)m);
    std::vector<size_t> hoff((size_t)m * 5, 0);
    auto al16 = [](size_t x) { return (x + 15) & ~(size_t)15; };
    size_t pin_need = 0;
    for (int k = 0; k < m; ++k) {
      const int i = todo[k];
      const CtwLatEntry& e = ent[k];
      if (e.status == 1 || e.status == 2 || (e.status == 3 && !big[i])) continue;
      const int lane = lane_ids[i];
      const size_t ns = (size_t)l->seed_n[lane];
      const size_t sz[5] = {(size_t)e.n_arcs * sizeof(CtwLatArc), (size_t)e.lpool_used * 4, ns * sizeof(CtwSrc),
                            ns * 4, (size_t)l->seed_pool[lane] * 4};
      for (int q = 0; q < 5; ++q) {
        hoff[(size_t)k * 5 + q] = pin_need;
        pin_need += al16(sz[q]);
      }
    }
    if (pin_need > l->lat_pin_cap) {
      if (l->lat_pin) cudaFreeHost(l->lat_pin);
      l->lat_pin = nullptr;
      l->lat_pin_cap = 0;
      const size_t c = std::max(pin_need + pin_need / 2, (size_t)1 << 20);
      if (cudaMallocHost((void**)&l->lat_pin, c) != cudaSuccess) {
        release();
        return fail(CTW_ERR_OOM, "lattice: pinned staging allocation failed");
      }
      l->lat_pin_cap = c;
    }
    for (int k = 0; k < m; ++k) {
      const int i = todo[k];
      const CtwLatEntry& e = ent[k];
      if (e.status == 1 || e.status == 2 || (e.status == 3 && !big[i])) continue;
      const int lane = lane_ids[i];
      const CtwLane& L = l->h[lane];
      Host& h = hb[k];
      char* b = l->lat_pin;
      const size_t* o = &hoff[(size_t)k * 5];
      h.arcs = reinterpret_cast<const CtwLatArc*>(b + o[0]);
      h.lab = reinterpret_cast<const int32_t*>(b + o[1]);
      h.seeds = reinterpret_cast<const CtwSrc*>(b + o[2]);
      h.spend = reinterpret_cast<const int32_t*>(b + o[3]);
      h.pool = reinterpret_cast<const int32_t*>(b + o[4]);
      const int ns = l->seed_n[lane];
      if (e.n_arcs)
        CUDA_TRY(cudaMemcpyAsync(b + o[0], d_arcs[i], (size_t)e.n_arcs * sizeof(CtwLatArc), cudaMemcpyDeviceToHost,
                                 l->stream));
      if (e.lpool_used)
        CUDA_TRY(cudaMemcpyAsync(b + o[1], d_lab[i], (size_t)e.lpool_used * 4, cudaMemcpyDeviceToHost, l->stream));
      if (ns) {
        CUDA_TRY(cudaMemcpyAsync(b + o[2], l->seed_src[lane], ns * sizeof(CtwSrc), cudaMemcpyDeviceToHost,
                                 l->stream));
        CUDA_TRY(cudaMemcpyAsync(b + o[3], l->seed_pend[lane], ns * 4, cudaMemcpyDeviceToHost, l->stream));
      }
      if (l->seed_pool[lane])
        CUDA_TRY(cudaMemcpyAsync(b + o[4], L.pool, (size_t)l->seed_pool[lane] * 4, cudaMemcpyDeviceToHost,
                                 l->stream));
    }
    CUDA_TRY(cudaStreamSynchronize(l->stream));
    lap("d2h");
    std::vector<int> done;
    for (int k = 0; k < m; ++k) {
      const int i = todo[k];
      const CtwLatEntry& e = ent[k];
      if (e.status == 1 || e.status == 2) {
        arc_cap[i] = std::max<int32_t>(4 * arc_cap[i], e.n_arcs + 1024);
        lab_cap[i] = std::max<int32_t>(4 * lab_cap[i], e.lpool_used + 4096);
        again.push_back(i);
        continue;
      }
      if (e.status == 3 && !big[i]) {  // a local closure overflowed: re-run with the large capacities
        big[i] = 1;
        again.push_back(i);
        continue;
      }
      done.push_back(k);
    }
    // ---- host copy of the kept lattices (canonical arc order, labels
    // expanded): independent per lane, spread over host threads
    auto post = [&](int k) {
      const int i = todo[k];
      const CtwLatEntry& e = ent[k];
      const int lane = lane_ids[i];
      const CtwLane& L = l->h[lane];
      ctw_lattice& o = out[i];
      o.status = e.status;
      o.final_mode = e.final_mode;
      o.frame_count = L.frame_count;
      o.best = e.best;
      o.lattice_beam = lattice_beam;
      o.closure_items = e.closure_items;
      o.closure_pruned = e.closure_pruned;
      const Host& hh = hb[k];
      const CtwLatArc* arcs = hh.arcs;
      const int32_t* lab = hh.lab;
      const CtwSrc* seeds = hh.seeds;
      const int32_t* spend = hh.spend;
      const int32_t* pool = hh.pool;
      const int ns = l->seed_n[lane];
      o.n_seeds = ns;
      o.seed_state = cmalloc<int32_t>(ns);
      o.seed_cost = cmalloc<double>(ns);
      o.seed_lab_off = cmalloc<int64_t>(ns + 1);
      std::vector<int32_t> sl;
      o.seed_lab_off[0] = 0;
      for (int k2 = 0; k2 < ns; ++k2) {
        o.seed_state[k2] = seeds[k2].state;
        o.seed_cost[k2] = seeds[k2].cost;
        expand_code(pool, spend[k2], sl);
        o.seed_lab_off[k2 + 1] = (int64_t)sl.size();
      }
      o.seed_lab = cmalloc<int32_t>(sl.size());
      std::copy(sl.begin(), sl.end(), o.seed_lab);
      const int64_t na = e.n_arcs;
      o.n_arcs = na;
      o.arc_src = cmalloc<int32_t>(na);
      o.arc_dst = cmalloc<int32_t>(na);
      o.arc_frame = cmalloc<int32_t>(na);
      o.arc_dst_state = cmalloc<int32_t>(na);
      o.arc_src_state = cmalloc<int32_t>(na);
      o.arc_w = cmalloc<double>(na);
      o.arc_dst_final = cmalloc<double>(na);
      o.arc_lab_off = cmalloc<int64_t>(na + 1);
      // canonical order: by (frame, src, dst, w) so results do not depend on
      // the kernel's append order
      std::vector<int64_t> ord((size_t)na);
      std::iota(ord.begin(), ord.end(), 0);
      std::sort(ord.begin(), ord.end(), [&](int64_t x, int64_t y) {
        const CtwLatArc &a = arcs[x], &b = arcs[y];
        if (a.frame != b.frame) return a.frame < b.frame;
        if (a.src != b.src) return a.src < b.src;
        if (a.dst != b.dst) return a.dst < b.dst;
        return a.w < b.w;
      });
      std::vector<int32_t> al;
      o.arc_lab_off[0] = 0;
      const double INF = HUGE_VAL;
      const int T = L.frame_count;
      for (int64_t k2 = 0; k2 < na; ++k2) {
        const CtwLatArc& a = arcs[ord[k2]];
        o.arc_src[k2] = a.src;
        o.arc_dst[k2] = a.dst;
        o.arc_frame[k2] = a.frame;
        o.arc_dst_state[k2] = a.dst_state;
        o.arc_src_state[k2] = a.src_state;
        o.arc_w[k2] = a.w;
        double fw = INF;
        if (a.frame == T - 1) fw = e.final_mode ? g->h_final[(uint32_t)a.dst_state & L.smask] : 0.0;
        o.arc_dst_final[k2] = fw;
        if (a.code > 0) al.push_back(a.code);
        else if (a.code < 0) {
          const int64_t off = -(int64_t)a.code - 1;
          for (int32_t j = 0; j < lab[off]; ++j) al.push_back(lab[off + 1 + j]);
        }
        o.arc_lab_off[k2 + 1] = (int64_t)al.size();
      }
      o.arc_lab = cmalloc<int32_t>(al.size());
      std::copy(al.begin(), al.end(), o.arc_lab);
    };
    const int nt = (int)std::min<size_t>(done.size(), std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
    if (nt <= 1) {
      for (int k : done) post(k);
    } else {
      std::atomic<size_t> next{0};
      std::vector<std::thread> th;
      for (int t = 0; t < nt; ++t)
        th.emplace_back([&]() {
          for (size_t j; (j = next.fetch_add(1)) < done.size();) post(done[j]);
        });
      for (auto& t : th) t.join();
    }
    lap("post");
    todo.swap(again);
  }
  release();
  lap("release");
  return 0;
}

namespace {

// Deterministic phrase automaton (Aho-Corasick over word ids): per state a
// sorted goto list, a failure link and the cost of the phrases completed on
// entering the state (negative = boost).
struct PhraseFsa {
  int32_t n;
  const int32_t* goto_off;
  const int32_t* goto_word;
  const int32_t* goto_next;
  const int32_t* fail;
  const double* out_cost;
};

inline int32_t fsa_step(const PhraseFsa* F, int32_t b, int32_t w, double* cost) {
  if (!F) return 0;
  for (;;) {
    const int32_t* lo = F->goto_word + F->goto_off[b];
    const int32_t* hi = F->goto_word + F->goto_off[b + 1];
    const int32_t* it = std::lower_bound(lo, hi, w);
    if (it != hi && *it == w) {
      const int32_t nb = F->goto_next[it - F->goto_word];
      *cost += F->out_cost[nb];
      return nb;
    }
    if (b == 0) {
      *cost += F->out_cost[0];
      return 0;
    }
    b = F->fail[b];
  }
}

// n best distinct word sequences of the lattice composed with an optional
// phrase automaton. Search states are (lattice node, automaton state); the
// remaining cost h is exact (backward DP over the reachable product), so A*
// pops complete paths in cost order; a partial path is dominated once
// another reached the same search state with the same word prefix.
int lattice_nbest(const ctw_lattice* lat, const PhraseFsa* F, int32_t n, int64_t max_pops, int32_t* words,
                  int64_t words_cap, int64_t* word_off, double* costs, int32_t* n_found, int64_t* pops) {
  *n_found = 0;
  if (pops) *pops = 0;
  word_off[0] = 0;
  if (n <= 0 || lat->status == 4) return 0;
  const double INF = HUGE_VAL;
  const int64_t na = lat->n_arcs, ns = lat->n_seeds;
  const int64_t NB = F ? F->n : 1;
  // lattice nodes -> dense indices; final weight per node
  std::vector<int32_t> ids;
  ids.reserve((size_t)(2 * na + ns));
  for (int64_t k = 0; k < ns; ++k) ids.push_back((int32_t)k);
  for (int64_t k = 0; k < na; ++k) {
    ids.push_back(lat->arc_src[k]);
    ids.push_back(lat->arc_dst[k]);
  }
  std::sort(ids.begin(), ids.end());
  ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
  auto idx = [&](int32_t node) { return (int)(std::lower_bound(ids.begin(), ids.end(), node) - ids.begin()); };
  const int nn = (int)ids.size();
  std::vector<double> fin((size_t)nn, INF);
  std::vector<int> out_off((size_t)nn + 1, 0), asrc((size_t)na), adst((size_t)na);
  for (int64_t k = 0; k < na; ++k) {
    asrc[k] = idx(lat->arc_src[k]);
    adst[k] = idx(lat->arc_dst[k]);
    out_off[asrc[k] + 1]++;
    if (lat->arc_dst_final[k] < fin[adst[k]]) fin[adst[k]] = lat->arc_dst_final[k];
  }
  for (int v = 0; v < nn; ++v) out_off[v + 1] += out_off[v];
  std::vector<int> adj((size_t)na);
  {
    std::vector<int> fill(out_off.begin(), out_off.end() - 1);
    for (int64_t k = 0; k < na; ++k) adj[fill[asrc[k]]++] = (int)k;
  }
  // ---- reachable product states, forward (arcs are sorted by frame)
  std::unordered_map<int64_t, int> pid;  // node * NB + b -> product index
  std::vector<int> pnode, pb;
  std::vector<double> pstart;  // start cost (seeds only), else INF
  auto get = [&](int v, int b) {
    const int64_t key = (int64_t)v * NB + b;
    auto it = pid.find(key);
    if (it != pid.end()) return it->second;
    const int p = (int)pnode.size();
    pid.emplace(key, p);
    pnode.push_back(v);
    pb.push_back(b);
    pstart.push_back(INF);
    return p;
  };
  struct PA {
    int from, to, arc;
    double c;
  };
  std::vector<PA> parcs;
  std::vector<uint64_t> seed_h((size_t)ns);
  std::vector<int> seed_p((size_t)ns, -1);
  for (int64_t k = 0; k < ns; ++k) {
    double c = lat->seed_cost[k];
    int32_t b = 0;
    for (int64_t j = lat->seed_lab_off[k]; j < lat->seed_lab_off[k + 1]; ++j) b = fsa_step(F, b, lat->seed_lab[j], &c);
    const int p = get(idx((int32_t)k), b);
    seed_p[k] = p;
    if (c < pstart[p]) pstart[p] = c;
  }
  {
    // frontier expansion layer by layer: product states of a node are known
    // before its out-arcs are processed because arcs are frame-sorted
    std::vector<std::vector<int>> states_of((size_t)nn);
    for (int p = 0; p < (int)pnode.size(); ++p) states_of[pnode[p]].push_back(p);
    for (int64_t k = 0; k < na; ++k) {
      const int v = asrc[k];
      for (size_t q = 0; q < states_of[v].size(); ++q) {
        const int p = states_of[v][q];
        double c = lat->arc_w[k];
        int32_t b = pb[p];
        for (int64_t j = lat->arc_lab_off[k]; j < lat->arc_lab_off[k + 1]; ++j) b = fsa_step(F, b, lat->arc_lab[j], &c);
        const size_t before = pnode.size();
        const int t = get(adst[k], b);
        if (pnode.size() > before) states_of[adst[k]].push_back(t);
        parcs.push_back(PA{p, t, (int)k, c});
      }
    }
  }
  const int np = (int)pnode.size();
  // ---- exact remaining cost (backward over product arcs: frame-sorted)
  std::vector<double> h((size_t)np, INF);
  for (int p = 0; p < np; ++p)
    if (out_off[pnode[p]] == out_off[pnode[p] + 1]) h[p] = fin[pnode[p]];
  for (int64_t q = (int64_t)parcs.size() - 1; q >= 0; --q) {
    const PA& a = parcs[q];
    const double c = a.c + h[a.to];
    if (c < h[a.from]) h[a.from] = c;
  }
  std::vector<int> pout_off((size_t)np + 1, 0);
  for (const PA& a : parcs) pout_off[a.from + 1]++;
  for (int p = 0; p < np; ++p) pout_off[p + 1] += pout_off[p];
  std::vector<int> padj(parcs.size());
  {
    std::vector<int> fill(pout_off.begin(), pout_off.end() - 1);
    for (size_t q = 0; q < parcs.size(); ++q) padj[fill[parcs[q].from]++] = (int)q;
  }
  // ---- A*
  struct P {
    int parent;
    int p;
    int parc;
    int depth;
    double g;
    uint64_t hh;
  };
  struct QE {
    double f;
    int depth;
    int idx;
    bool operator>(const QE& o) const {
      if (f != o.f) return f > o.f;
      if (depth != o.depth) return depth < o.depth;
      return idx > o.idx;
    }
  };
  auto mix = [](uint64_t x, int32_t w) {
    x ^= (uint64_t)(uint32_t)w + 0x9E3779B97F4A7C15ull + (x << 6) + (x >> 2);
    return x * 0xBF58476D1CE4E5B9ull;
  };
  std::vector<P> tree;
  std::vector<QE> heap;
  auto push = [&](const P& e) {
    tree.push_back(e);
    heap.push_back(QE{e.g + h[e.p], e.depth, (int)tree.size() - 1});
    std::push_heap(heap.begin(), heap.end(), std::greater<QE>());
  };
  std::vector<int> seed_of_p((size_t)np, -1);
  for (int64_t k = 0; k < ns; ++k) {
    const int p = seed_p[k];
    uint64_t x = 0x12345678ull;
    for (int64_t j = lat->seed_lab_off[k]; j < lat->seed_lab_off[k + 1]; ++j) x = mix(x, lat->seed_lab[j]);
    double c = lat->seed_cost[k];
    int32_t b = 0;
    for (int64_t j = lat->seed_lab_off[k]; j < lat->seed_lab_off[k + 1]; ++j) b = fsa_step(F, b, lat->seed_lab[j], &c);
    seed_of_p[p] = (int)k;
    if (h[p] < INF) push(P{-1, p, -1, 0, c, x});
  }
  std::vector<std::vector<int32_t>> seen;
  std::vector<double> found_cost;
  std::unordered_set<uint64_t> expanded;
  int64_t npop = 0;
  while (!heap.empty() && (int)found_cost.size() < n && npop < max_pops) {
    std::pop_heap(heap.begin(), heap.end(), std::greater<QE>());
    const QE top = heap.back();
    heap.pop_back();
    ++npop;
    const P cur = tree[top.idx];
    const uint64_t key = mix(cur.hh, cur.p) ^ ((uint64_t)cur.p << 1);
    if (!expanded.insert(key).second) continue;  // dominated (same search state, same words so far)
    const int v = pnode[cur.p];
    if (out_off[v] == out_off[v + 1]) {
      if (!(fin[v] < INF) || cur.parc < 0) continue;
      // complete path: words = seed labels + arc labels, oldest first
      std::vector<int> arcs_rev;
      int t = top.idx, seed = -1;
      while (t >= 0) {
        if (tree[t].parc >= 0) arcs_rev.push_back(parcs[tree[t].parc].arc);
        else seed = seed_of_p[tree[t].p];
        t = tree[t].parent;
      }
      std::vector<int32_t> w;
      for (int64_t j = lat->seed_lab_off[seed]; j < lat->seed_lab_off[seed + 1]; ++j) w.push_back(lat->seed_lab[j]);
      for (auto it = arcs_rev.rbegin(); it != arcs_rev.rend(); ++it)
        for (int64_t j = lat->arc_lab_off[*it]; j < lat->arc_lab_off[*it + 1]; ++j) w.push_back(lat->arc_lab[j]);
      if (std::find(seen.begin(), seen.end(), w) == seen.end()) {
        seen.push_back(w);
        found_cost.push_back(cur.g + fin[v]);
      }
      continue;
    }
    for (int q = pout_off[cur.p]; q < pout_off[cur.p + 1]; ++q) {
      const PA& a = parcs[padj[q]];
      if (!(h[a.to] < INF)) continue;
      uint64_t x = cur.hh;
      for (int64_t j = lat->arc_lab_off[a.arc]; j < lat->arc_lab_off[a.arc + 1]; ++j) x = mix(x, lat->arc_lab[j]);
      push(P{top.idx, a.to, padj[q], cur.depth + 1, cur.g + a.c, x});
    }
  }
  if (pops) *pops = npop;
  int64_t need = 0;
  for (auto& w : seen) need += (int64_t)w.size();
  *n_found = (int32_t)seen.size();
  int64_t pos = 0;
  for (size_t k = 0; k < seen.size(); ++k) {
    costs[k] = found_cost[k];
    word_off[k] = pos;
    if (pos + (int64_t)seen[k].size() <= words_cap) std::copy(seen[k].begin(), seen[k].end(), words + pos);
    pos += (int64_t)seen[k].size();
  }
  word_off[seen.size()] = pos;
  return need > words_cap ? -2 : 0;
}

}  // namespace

int ctw_lattice_nbest(const ctw_lattice* lat, int32_t n, int64_t max_pops, int32_t* words, int64_t words_cap,
                      int64_t* word_off, double* costs, int32_t* n_found, int64_t* pops) {
  return lattice_nbest(lat, nullptr, n, max_pops, words, words_cap, word_off, costs, n_found, pops);
}

int ctw_lattice_nbest_phrases(const ctw_lattice* lat, int32_t fsa_states, const int32_t* goto_off,
                              const int32_t* goto_word, const int32_t* goto_next, const int32_t* fail_link,
                              const double* out_cost, int32_t n, int64_t max_pops, int32_t* words,
                              int64_t words_cap, int64_t* word_off, double* costs, int32_t* n_found, int64_t* pops) {
  if (fsa_states <= 0) return fail(-1, "phrase automaton needs at least the root state");
  PhraseFsa F{fsa_states, goto_off, goto_word, goto_next, fail_link, out_cost};
  return lattice_nbest(lat, &F, n, max_pops, words, words_cap, word_off, costs, n_found, pops);
}

}  // extern "C"
