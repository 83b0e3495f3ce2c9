// ctw_lattice.cu -- lattice generation and lattice pruning on the device
// (the reference has no lattice).
//
// Definition. After a lane has decoded an utterance,
// its lattice nodes are the seed tokens (layer -1: the start state's epsilon
// closure, decoder.py:173-229) and the per-frame records (layer f: the
// survivors of frame f, _kernel.pyx:392-427). Between consecutive layers
// there is one lattice arc for every (source node s in layer f-1, emitting
// arc e leaving state(s), destination node d in layer f) such that some path
// e, eps, eps, ... leads from state(s) to state(d); its weight is the minimum
// over those epsilon continuations of
//     (-scale * ll[f, il(e) - 1]) + w(e) (+ boost[ol(e)]) + sum (w + boost)
// with the reference's operation order (_kernel.pyx:249-253, :307-310), and
// its output labels are those of the minimising path. alpha(node) is the
// node's decoder cost; beta(node) the minimum over complete continuations
// (final weight at the last layer: final states if any survive, else 0 --
// the best_path rule of decoder.py:384-400). An arc is kept iff
// alpha(s) + w + beta(d) <= best + lattice_beam.
//
// The kernel walks the layers backwards so beta is known when a layer's
// arcs are generated and pruning happens as arcs are produced (a full
// unpruned lattice would be ~10^7 arcs per utterance). One thread-block
// cluster per lane (1..8 CTAs: several when the batch leaves SMs idle): per
// layer, the surviving destination nodes go into the lane's (empty) token
// table as a state -> node map, every (source, emitting arc) pair is a work
// item that runs its own small epsilon closure, and kept arcs are appended to
// the lane's arc buffer. A closure that outgrows its local capacity marks
// the lane (status 3) and the host re-runs it with the large instantiation.
//
// When no epsilon arc carries an output label (C2, C3), the closures do not
// depend on the lane (boosts and phrase automata only act on labelled arcs):
// they are computed once per graph into an index (k_closure_index: per state
// the epsilon-reachable states and their minimum path weight), and the work
// item of the indexed kernel (k_lattice_idx) reads its closure as one contiguous run of
// 16-byte entries and probes a shared-memory copy of the layer's destination
// map -- no per-thread closure arrays, no local memory, ~4 dependent memory
// round trips per item instead of ~50. Arc weights are then c0 + (w1 + w2 +
// ...) instead of ((c0 + w1) + w2) + ...: equal up to rounding (DESIGN.md
// "Lattice").
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_scan.cuh>
#include <stdint.h>

#include <algorithm>
#include <type_traits>

#include "ctw_common.h"

#ifndef LAT_BS
#define LAT_BS 512
#endif
#define LAT_CL 48       // local epsilon-closure capacity per work item
#define LAT_QL 128      // local relaxation budget per work item
#define LAT_CL_BIG 256  // ... of the re-run for items that overflowed
#define LAT_QL_BIG 1024
#define LAT_MAP 2048        // indexed kernel: shared-memory destination map slots (<= LAT_MAP / 2 entries)
#define CLO_CAP 64          // closure index: largest indexed closure
#define CLO_QCAP 256        // ... and its relaxation budget

namespace {

struct LatGraph {
  const CtwStateRange* ranges;
  const CtwArc* arcs;
  const int32_t* olabel;
  const double* final_w;
};

__device__ __forceinline__ unsigned long long lat_d2key(double x) {
  x = __dadd_rn(x, 0.0);
  long long b = __double_as_longlong(x);
  return (unsigned long long)(b ^ ((b >> 63) | (long long)0x8000000000000000ULL));
}

__device__ __forceinline__ double lat_key2d(unsigned long long k) {
  long long b = (k & 0x8000000000000000ULL) ? (long long)(k ^ 0x8000000000000000ULL) : (long long)~k;
  return __longlong_as_double(b);
}

__device__ __forceinline__ uint32_t lat_hash(uint32_t s, uint32_t shift) { return (s * 0x9E3779B1u) >> shift; }

// Destination token key of an arc (phrase automaton: the key carries the
// automaton state) and its boost, added after the arc weight like the
// decoder (ctw_kernels.cu arc_dest).
__device__ __forceinline__ uint32_t lat_dest(const CtwLane& lane, uint32_t key, int32_t ol, uint32_t nextstate,
                                             double& c) {
  if (lane.fsa_next) {
    uint32_t b = key >> lane.sbits;
    if (ol != 0) {
      b = lane.fsa_next[(size_t)b * lane.fsa_width + ol];
      c = __dadd_rn(c, lane.fsa_cost[b]);
    }
    return nextstate | (b << lane.sbits);
  }
  if (lane.boost && ol != 0) c = __dadd_rn(c, lane.boost[ol]);
  return nextstate;
}

}  // namespace

namespace cg = cooperative_groups;

namespace {

struct LatArgs {
  CtwLane* lanes;
  LatGraph g;
  const uint32_t* clo_off;  // closure index (k_lattice_idx): per state offset | CTW_CLO_NONE
  const CtwClo* clo_ent;
  CtwLatEntry* ent;
  const void* loglik;
  int width;
  int is_f64;
  double acoustic_scale;
  double lattice_beam;
};

__device__ __forceinline__ void lat_rec(const CtwLane& lane, long long r, int32_t* state, double* cost) {
  const CtwRecPage* pg = lane.pages[r >> CTW_PAGE_LOG2];
  const int o = (int)(r & (CTW_PAGE - 1));
  *state = pg->state[o];
  *cost = pg->cost[o];
}

// Insert state -> node into the (empty) lane table; the node id rides in tb.
// Returns the table index.
__device__ __forceinline__ uint32_t lat_put(const CtwLane& lane, uint32_t shift, uint32_t mask, uint32_t s,
                                            uint32_t node) {
  uint32_t h = lat_hash(s, shift);
  for (uint32_t p = 0; p <= mask; ++p) {
    const uint32_t old = atomicCAS(&lane.table[h].state, CTW_EMPTY, s);
    if (old == CTW_EMPTY || old == s) {
      lane.table[h].tb = node;
      return h;
    }
    h = (h + 1) & mask;
  }
  return CTW_EMPTY;
}

__device__ __forceinline__ int lat_get(const CtwLane& lane, uint32_t shift, uint32_t mask, uint32_t s) {
  uint32_t h = lat_hash(s, shift);
  for (uint32_t p = 0; p <= mask; ++p) {
    const uint32_t k = __ldcg(&lane.table[h].state);
    if (k == s) return (int)__ldcg(&lane.table[h].tb);
    if (k == CTW_EMPTY) return -1;
    h = (h + 1) & mask;
  }
  return -1;
}

struct __align__(16) LatSmem {
  typedef cub::BlockScan<int, LAT_BS> Scan;
  typename Scan::TempStorage scan;
  // the current tile of sources: (source, emitting arc) items are spread
  // over all threads by the degree prefix
  int off[LAT_BS + 1];
  uint32_t beg[LAT_BS];
  int32_t sst[LAT_BS];
  int32_t node[LAT_BS];
  double sc[LAT_BS];
  int nput, final_mode;
  unsigned long long ac_min;  // min over the frame row of -scale * ll (sortable key)
  unsigned long long min_beta;  // this rank's minimum over its destinations
  unsigned long long mb_pub;    // ... published to the cluster
  unsigned long long mb_all;    // cluster-wide minimum
  unsigned long long best;
  unsigned long long items, pruned;
};

#ifndef LAT_MINB
#define LAT_MINB 4  // 4 CTAs (64 warps) per SM: every lane of a 512-lane batch resident (61 -> 32 registers; lattice stage -32 %)
#endif

// One work item: emitting arc ai out of source node `node` (state sst, cost
// sc) into layer f, with its local epsilon closure of capacity CL states /
// QL relaxations (overflow -> status 3; the host re-runs the lane with the
// large-capacity instantiation).
template <int CL, int QL>
__device__ __forceinline__ void lat_item(const LatArgs& a, CtwLatEntry& E, const CtwLane& lane, LatSmem& sm,
                                         uint32_t shift, uint32_t mask, bool cut_ok, double cutoff, double min_beta,
                                         int32_t sst, double sc, int node, int f, uint32_t ai, long long row0) {
  const double INF = __longlong_as_double(0x7FF0000000000000LL);
  const CtwArc arc = a.g.arcs[ai];
  double x;
  {
    const long long idx = row0 + arc.ilabel - 1;
    x = a.is_f64 ? ((const double*)a.loglik)[idx] : (double)((const float*)a.loglik)[idx];
  }
  double c0 = __dadd_rn(__dmul_rn(-a.acoustic_scale, x), arc.weight);
  const int32_t ol0 = a.g.olabel[ai];
  const uint32_t x0 = lat_dest(lane, (uint32_t)sst, ol0, (uint32_t)arc.nextstate, c0);
  if (!(c0 < INF)) return;
  if (cut_ok && sc + c0 + min_beta > cutoff) {
    atomicAdd(&sm.pruned, 1ULL);
    return;
  }
  atomicAdd(&sm.items, 1ULL);
  // local epsilon closure from nextstate(e): (state, cost, pred, olabel)
  typedef typename std::conditional<(CL > 127), int16_t, int8_t>::type Idx;  // closure entry index
  int32_t cst[CL];
  double ccost[CL];
  Idx cpred[CL];
  int32_t colab[CL];
  int n = 1;
  cst[0] = (int32_t)x0;
  ccost[0] = c0;
  cpred[0] = -1;
  colab[0] = ol0;
  Idx queue[QL];
  int qh = 0, qt = 1;
  queue[0] = 0;
  bool overflow = false;
  while (qh < qt) {
    const int u = queue[qh++];
    const CtwStateRange ru = a.g.ranges[(uint32_t)cst[u] & lane.smask];
    for (uint32_t b = ru.eps_beg; b < ru.emit_beg; ++b) {
      const CtwArc ea = a.g.arcs[b];
      double cy = __dadd_rn(ccost[u], ea.weight);
      const int32_t oly = a.g.olabel[b];
      const int32_t ykey = (int32_t)lat_dest(lane, (uint32_t)cst[u], oly, (uint32_t)ea.nextstate, cy);
      if (!(cy < INF)) continue;
      if (cut_ok && sc + cy + min_beta > cutoff) continue;
      int j = 0;
      while (j < n && cst[j] != ykey) ++j;
      if (j < n) {
        if (!(cy < ccost[j])) continue;
      } else {
        if (n == CL) {
          overflow = true;
          continue;
        }
        ++n;
        cst[j] = ykey;
      }
      ccost[j] = cy;
      cpred[j] = (Idx)u;
      colab[j] = oly;
      if (qt == QL) {
        overflow = true;
        continue;
      }
      queue[qt++] = (Idx)j;
    }
  }
  if (overflow) atomicMax(&E.status, 3);
  // arcs to the surviving destinations
  for (int j = 0; j < n; ++j) {
    const int dn = lat_get(lane, shift, mask, (uint32_t)cst[j]);
    if (dn < 0) continue;
    const double bd = lat_key2d(__ldcg(&E.beta[dn]));
    const double tail = __dadd_rn(ccost[j], bd);
    atomicMin(&E.beta[node], lat_d2key(tail));
    if (__dadd_rn(sc, tail) > cutoff) continue;
    // labels of the minimising path, oldest first
    int nl = 0;
    int32_t last = 0;
    for (int u = j; u >= 0; u = cpred[u])
      if (colab[u] != 0) {
        ++nl;
        last = colab[u];
      }
    int32_t code = 0;
    if (nl == 1) code = last;
    else if (nl > 1) {
      const int po = atomicAdd(&E.lpool_used, nl + 1);
      if (po + nl + 1 > E.lpool_cap) {
        atomicMax(&E.status, 2);
        continue;
      }
      int32_t* seg = E.lpool + po;
      seg[0] = nl;
      int pos = nl;
      for (int u = j; u >= 0; u = cpred[u])
        if (colab[u] != 0) seg[pos--] = colab[u];
      code = -(po + 1);
    }
    const int ia = atomicAdd(&E.n_arcs, 1);
    if (ia >= E.arc_cap) {
      atomicMax(&E.status, 1);
      continue;
    }
    CtwLatArc la;
    la.src = node;
    la.dst = dn;
    la.w = ccost[j];
    la.code = code;
    la.frame = f;
    la.dst_state = cst[j];
    la.src_state = sst;
    E.arcs[ia] = la;
  }
}

// One thread-block cluster of R CTAs ("ranks") per lane: the ranks split
// every layer's destination records and source tiles and meet at cluster
// barriers between the steps of a layer; counters live in the entry (global
// atomics), the layer's minimum beta is exchanged through shared memory.
template <int CL, int QL>
__global__ void __launch_bounds__(LAT_BS, LAT_MINB) k_lattice(LatArgs a) {
  __shared__ LatSmem sm;
  cg::cluster_group cl = cg::this_cluster();
  const int R = (int)cl.num_blocks(), rank = (int)cl.block_rank();
  const int tid = threadIdx.x;
  CtwLatEntry& E = a.ent[blockIdx.x / R];
  const CtwLane& lane = a.lanes[E.lane];
  const double INF = __longlong_as_double(0x7FF0000000000000LL);
  const uint32_t tlog2 = lane.tlog2;
  const uint32_t mask = (1u << tlog2) - 1, shift = 32 - tlog2;
  const int T = lane.frame_count;
  const long long NR = lane.n_rec;
  const int S0 = E.n_seeds;
  const long long stride = (long long)R * LAT_BS;
  // this rank's list of destination-map entries (for the clear), a slice of
  // the lane's frontier scratch (the host sizes R so a layer's share fits)
  const int pcap = (int)((size_t)CTW_FRONT_LEN(1u << tlog2) / R);
  uint2* plist = lane.front + (size_t)rank * pcap;
  if (tid == 0) {
    sm.best = ~0ULL;
    sm.final_mode = 0;
    sm.items = 0;
    sm.pruned = 0;
  }
  for (long long i = (long long)rank * LAT_BS + tid; i < S0 + NR; i += stride) E.beta[i] = ~0ULL;
  cl.sync();  // beta cleared everywhere before any rank sets the last layer's
  if (T == 0) {
    if (rank == 0 && tid == 0) E.status = 4;
    return;
  }
  // ---- last layer: beta = final weight (final states if any survive, else 0);
  // every rank derives final_mode and the best cost over the whole layer
  const long long lf0 = lane.frame_base[T - 1], lf1 = NR;
  for (long long r = lf0 + tid; r < lf1; r += LAT_BS) {
    int32_t st;
    double c;
    lat_rec(lane, r, &st, &c);
    if (a.g.final_w[(uint32_t)st & lane.smask] != INF) sm.final_mode = 1;  // benign race: all writers store 1
  }
  __syncthreads();
  const bool fm = sm.final_mode != 0;
  for (long long r = lf0 + tid; r < lf1; r += LAT_BS) {
    int32_t st;
    double c;
    lat_rec(lane, r, &st, &c);
    const double fw = fm ? a.g.final_w[(uint32_t)st & lane.smask] : 0.0;
    if (fm && fw == INF) continue;
    atomicMin(&sm.best, lat_d2key(c + fw));
    if ((((r - lf0) / LAT_BS) % R) == rank) E.beta[S0 + r] = lat_d2key(fw);
  }
  cl.sync();  // beta initialised and the last layer's set in every rank's share
  const double best = lat_key2d(sm.best);
  const double cutoff = __dadd_rn(best, a.lattice_beam);
  const bool cut_ok = lane.prune_ok != 0;  // epsilon continuations never lower a cost

  for (int f = T - 1; f >= 0; --f) {
    const long long d0 = lane.frame_base[f], d1 = (f + 1 < T) ? lane.frame_base[f + 1] : NR;
    // ---- destination map: nodes of layer f that can lie on a kept path
    if (tid == 0) {
      sm.min_beta = ~0ULL;
      sm.nput = 0;
      sm.ac_min = ~0ULL;
    }
    __syncthreads();
    {
      // smallest acoustic term of the frame (source-level pruning bound)
      const long long rr = E.ll_off + (long long)f * a.width;
      for (int v = tid; v < a.width; v += LAT_BS) {
        const double x = a.is_f64 ? ((const double*)a.loglik)[rr + v] : (double)((const float*)a.loglik)[rr + v];
        atomicMin(&sm.ac_min, lat_d2key(__dmul_rn(-a.acoustic_scale, x)));
      }
    }
    for (long long r = d0 + (long long)rank * LAT_BS + tid; r < d1; r += stride) {
      const unsigned long long bk = E.beta[S0 + r];
      if (bk == ~0ULL) continue;
      int32_t st;
      double c;
      lat_rec(lane, r, &st, &c);
      if (c + lat_key2d(bk) > cutoff) continue;
      const uint32_t h = lat_put(lane, shift, mask, (uint32_t)st, (uint32_t)(S0 + r));
      if (h != CTW_EMPTY) {
        const int p = atomicAdd(&sm.nput, 1);
        if (p < pcap) plist[p] = make_uint2(h, (uint32_t)st);  // for the clear
        else atomicMax(&E.status, 3);
      }
      atomicMin(&sm.min_beta, bk);
    }
    __syncthreads();
    if (tid == 0) sm.mb_pub = sm.min_beta;
    cl.sync();  // the whole layer is in the map; every rank's minimum published
    if (tid < 32) {
      unsigned long long m = tid < R ? cl.map_shared_rank(&sm, tid)->mb_pub : ~0ULL;
      for (int d = 16; d; d >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xFFFFFFFFu, m, d);
        if (o < m) m = o;
      }
      if (tid == 0) sm.mb_all = m;
    }
    __syncthreads();
    const double min_beta = sm.mb_all == ~0ULL ? INF : lat_key2d(sm.mb_all);
    // ---- sources: layer f-1 (records) or the seeds, tiles split over the ranks
    const long long s0 = f > 0 ? lane.frame_base[f - 1] : 0;
    const long long s1 = f > 0 ? d0 : S0;
    const long long nsrc = s1 - s0;
    const long long row0 = E.ll_off + (long long)f * a.width;
    if (min_beta != INF) {
      for (long long t0 = (long long)rank * LAT_BS; t0 < nsrc; t0 += stride) {
        const long long si = t0 + tid;
        int deg = 0;
        const double step_lb = lat_key2d(sm.ac_min) + E.emit_lb;  // any emitting step costs at least this
        if (si < nsrc) {
          int32_t st0;
          double c0s;
          int nd;
          if (f > 0) {
            lat_rec(lane, s0 + si, &st0, &c0s);
            nd = (int)(S0 + s0 + si);
          } else {
            st0 = E.seeds[si].state;
            c0s = E.seeds[si].cost;
            nd = (int)si;
          }
          const CtwStateRange rg = a.g.ranges[(uint32_t)st0 & lane.smask];
          deg = (int)(rg.emit_end - rg.emit_beg);
          // no arc of this source can be kept (epsilon continuations only add)
          if (cut_ok && c0s + step_lb + min_beta > cutoff + 1e-9 * fabs(cutoff)) deg = 0;
          sm.beg[tid] = rg.emit_beg;
          sm.sst[tid] = st0;
          sm.sc[tid] = c0s;
          sm.node[tid] = nd;
        }
        int ex, tot;
        LatSmem::Scan(sm.scan).ExclusiveSum(deg, ex, tot);
        sm.off[tid] = ex;
        __syncthreads();
        const int nv = (int)min((long long)LAT_BS, nsrc - t0);
        for (int item = tid; item < tot; item += LAT_BS) {
          int lo = 0, hi = nv - 1;  // last source with off <= item
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (sm.off[mid] <= item) lo = mid;
            else hi = mid - 1;
          }
          lat_item<CL, QL>(a, E, lane, sm, shift, mask, cut_ok, cutoff, min_beta, sm.sst[lo], sm.sc[lo], sm.node[lo],
                           f, sm.beg[lo] + (uint32_t)(item - sm.off[lo]), row0);
        }
        __syncthreads();  // the tile's smem is reused by the next tile
      }
    }
    cl.sync();  // the layer's arcs are out; beta of layer f-1 final
    // ---- clear this rank's destination-map entries (the decoder's tok_clear image)
    const int np = min(sm.nput, pcap);
    for (int i = tid; i < np; i += LAT_BS) {
      ulonglong2* q = reinterpret_cast<ulonglong2*>(&lane.table[plist[i].x]);
      __stcg(q, make_ulonglong2(~0ULL, 0xFFFFFFFFULL));
      __stcg(q + 1, make_ulonglong2(~0ULL, (unsigned long long)CTW_EMPTY));
    }
    cl.sync();  // the map is empty before the next layer's puts
  }
  if (tid == 0) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&E.closure_items), sm.items);
    atomicAdd(reinterpret_cast<unsigned long long*>(&E.closure_pruned), sm.pruned);
  }
  if (rank == 0 && tid == 0) {
    if (E.status == 0 && sm.best == ~0ULL) E.status = 4;
    E.final_mode = sm.final_mode;
    E.best = best;
  }
}


// ------------------------------------------------------------ indexed kernel
// (graphs without labelled epsilon arcs): closures from the closure index,
// and every rank builds the layer's whole destination map in its own shared
// memory from the layer's records (8x redundant reads of a few KB instead of
// two extra cluster barriers and the lane-table map): one cluster barrier
// per layer.

#ifndef LAT_IBS
#define LAT_IBS 512  // threads per CTA of the indexed kernel
#endif
#ifndef LAT_IMINB
#define LAT_IMINB 4
#endif
#ifndef LAT_MU
#define LAT_MU 4  // destination-map scan: records per thread per round
#endif

struct __align__(16) LatIdxSmem {
  typedef cub::BlockScan<int, LAT_IBS> Scan;
  typename Scan::TempStorage scan;
  int off[LAT_IBS + 1];
  uint32_t beg[LAT_IBS];
  int32_t sst[LAT_IBS];
  int32_t node[LAT_IBS];
  double sc[LAT_IBS];
  // destination map: state -> node and the node's beta (sortable key)
  uint32_t mst[LAT_MAP];
  int32_t mnode[LAT_MAP];
  unsigned long long mbeta[LAT_MAP];
  int nmap, final_mode;
  unsigned long long ac_min, min_beta, best, items, pruned;
  // per-layer values the work items read at their point of use (fewer live
  // registers across the item loop: no spills at 32 registers)
  double cutoff, mb;
  long long row0;
  int f, cut_ok;
  CtwLatEntry* E;
  const CtwLane* lane;
  int T, NR, S0;
  int s0, nsrc;  // the layer's sources
  int t0, t1;    // first source of the current tile, end of this rank's share
};

#define LAT_MAP_LOG2 11
static_assert((1 << LAT_MAP_LOG2) == LAT_MAP, "LAT_MAP is 2^LAT_MAP_LOG2");

__device__ __forceinline__ int idx_find(const LatIdxSmem& sm, uint32_t s) {
  uint32_t h = lat_hash(s, 32 - LAT_MAP_LOG2);
  for (;;) {
    const uint32_t k = sm.mst[h];
    if (k == s) return (int)h;
    if (k == CTW_EMPTY) return -1;
    h = (h + 1) & (LAT_MAP - 1);
  }
}

// Work item: emitting arc ai out of source node `node` (state sst, cost sc).
__device__ __forceinline__ void lat_item_idx(const LatArgs& a, LatIdxSmem& sm, int lo, uint32_t ai) {
  const double INF = __longlong_as_double(0x7FF0000000000000LL);
  const CtwArc arc = a.g.arcs[ai];
  double x;
  {
    const long long idx = sm.row0 + arc.ilabel - 1;
    x = a.is_f64 ? ((const double*)a.loglik)[idx] : (double)((const float*)a.loglik)[idx];
  }
  double c0 = __dadd_rn(__dmul_rn(-a.acoustic_scale, x), arc.weight);
  const int32_t ol0 = a.g.olabel[ai];
  const uint32_t x0 = lat_dest(*sm.lane, (uint32_t)sm.sst[lo], ol0, (uint32_t)arc.nextstate, c0);
  if (!(c0 < INF)) return;
  const double sc = sm.sc[lo];
  if (sm.cut_ok && sc + c0 + sm.mb > sm.cutoff) {
    atomicAdd(&sm.pruned, 1ULL);
    return;
  }
  atomicAdd(&sm.items, 1ULL);
  const uint32_t smask = sm.lane->smask;
  const uint32_t s0 = x0 & smask, hi = x0 & ~smask;
  const uint32_t ob = __ldg(&a.clo_off[s0]);
  if (ob & CTW_CLO_NONE) {  // closure too large for the index: the host re-runs the lane
    atomicMax(&sm.E->status, 3);
    return;
  }
  const uint32_t oe = __ldg(&a.clo_off[s0 + 1]) & ~CTW_CLO_NONE;
  for (uint32_t k = ob; k < oe; ++k) {
    const ulonglong2 ce = __ldg(reinterpret_cast<const ulonglong2*>(a.clo_ent + k));  // {w, state}
    const double c = __dadd_rn(c0, __longlong_as_double((long long)ce.x));
    if (!(c < INF)) continue;
    if (sm.cut_ok && sc + c + sm.mb > sm.cutoff) continue;
    const uint32_t key = (uint32_t)ce.y | hi;
    const int slot = idx_find(sm, key);
    if (slot < 0) continue;
    const double tail = __dadd_rn(c, lat_key2d(sm.mbeta[slot]));
    CtwLatEntry& E = *sm.E;
    atomicMin(&E.beta[sm.node[lo]], lat_d2key(tail));
    if (__dadd_rn(sc, tail) > sm.cutoff) continue;
    const int ia = atomicAdd(&E.n_arcs, 1);
    if (ia >= E.arc_cap) {
      atomicMax(&E.status, 1);
      continue;
    }
    CtwLatArc la;
    la.src = sm.node[lo];
    la.dst = sm.mnode[slot];
    la.w = c;
    la.code = ol0;
    la.frame = sm.f;
    la.dst_state = (int32_t)key;
    la.src_state = sm.sst[lo];
    E.arcs[ia] = la;
  }
}

__global__ void __launch_bounds__(LAT_IBS, LAT_IMINB) k_lattice_idx(LatArgs a) {
  __shared__ LatIdxSmem sm;
  cg::cluster_group cl = cg::this_cluster();
  const int R = (int)cl.num_blocks(), rank = (int)cl.block_rank();
  const int tid = threadIdx.x;
  CtwLatEntry& E = a.ent[blockIdx.x / R];
  const CtwLane& lane = a.lanes[E.lane];
  const double INF = __longlong_as_double(0x7FF0000000000000LL);
  const int T = lane.frame_count;
  const int NR = (int)lane.n_rec;  // node ids are int32 (S0 + NR < 2^31)
  const int S0 = E.n_seeds;
  const int stride = R * LAT_IBS;
  if (tid == 0) {
    sm.best = ~0ULL;
    sm.final_mode = 0;
    sm.items = 0;
    sm.pruned = 0;
    sm.E = &E;
    sm.lane = &lane;
    sm.T = T;
    sm.NR = NR;
    sm.S0 = S0;
  }
  for (int i = rank * LAT_IBS + tid; i < S0 + NR; i += stride) E.beta[i] = ~0ULL;
  cl.sync();  // beta cleared everywhere before any rank sets the last layer's
  if (T == 0) {
    if (rank == 0 && tid == 0) E.status = 4;
    return;
  }
  // ---- last layer: beta = final weight (final states if any survive, else 0)
  const int lf0 = (int)lane.frame_base[T - 1], lf1 = NR;
  for (int r = lf0 + tid; r < lf1; r += LAT_IBS) {
    int32_t st;
    double c;
    lat_rec(lane, r, &st, &c);
    if (a.g.final_w[(uint32_t)st & lane.smask] != INF) sm.final_mode = 1;  // benign race: all writers store 1
  }
  __syncthreads();
  const bool fm = sm.final_mode != 0;
  for (int r = lf0 + tid; r < lf1; r += LAT_IBS) {
    int32_t st;
    double c;
    lat_rec(lane, r, &st, &c);
    const double fw = fm ? a.g.final_w[(uint32_t)st & lane.smask] : 0.0;
    if (fm && fw == INF) continue;
    atomicMin(&sm.best, lat_d2key(c + fw));
    if ((((r - lf0) / LAT_IBS) % R) == rank) E.beta[S0 + r] = lat_d2key(fw);
  }
  cl.sync();  // the last layer's beta set in every rank's share
  // loop-invariant values live in shared memory (no spills at 32 registers)
  if (tid == 0) {
    sm.cutoff = __dadd_rn(lat_key2d(sm.best), a.lattice_beam);
    sm.cut_ok = lane.prune_ok != 0;  // epsilon continuations never lower a cost
  }
  bool ovf = false;

  if (threadIdx.x == 0) sm.f = T - 1;
  for (;;) {
    __syncthreads();  // sm.f of this layer
    if (sm.f < 0) break;  // the layer index lives in shared memory (no register across the layer)
    const int d0 = (int)sm.lane->frame_base[sm.f], d1 = (sm.f + 1 < sm.T) ? (int)sm.lane->frame_base[sm.f + 1] : sm.NR;
    if ((int)threadIdx.x == 0) {
      sm.min_beta = ~0ULL;
      sm.nmap = 0;
      sm.ac_min = ~0ULL;
    }
    for (int i = (int)threadIdx.x; i < LAT_MAP; i += LAT_IBS) sm.mst[i] = CTW_EMPTY;
    __syncthreads();
    {
      // smallest acoustic term of the frame (source-level pruning bound)
      const long long rr = sm.E->ll_off + (long long)sm.f * a.width;
      for (int v = (int)threadIdx.x; v < a.width; v += LAT_IBS) {
        const double x = a.is_f64 ? ((const double*)a.loglik)[rr + v] : (double)((const float*)a.loglik)[rr + v];
        atomicMin(&sm.ac_min, lat_d2key(__dmul_rn(-a.acoustic_scale, x)));
      }
    }
    // ---- destination map: nodes of layer f that can lie on a kept path
    // (beta final since the previous layer's barrier), the whole layer in
    // every rank
    // (the beta words of LAT_MU records per thread are loaded together: most
    // are +inf and skipped, so the scan costs ~one memory latency)
    for (int r0 = d0; r0 < d1; r0 += LAT_MU * LAT_IBS) {
      unsigned long long bk[LAT_MU];
#pragma unroll
      for (int u = 0; u < LAT_MU; ++u) {
        const int r = r0 + u * LAT_IBS + (int)threadIdx.x;
        bk[u] = r < d1 ? __ldcg(&sm.E->beta[sm.S0 + r]) : ~0ULL;
      }
#pragma unroll
      for (int u = 0; u < LAT_MU; ++u) {
        if (bk[u] == ~0ULL) continue;
        const int r = r0 + u * LAT_IBS + (int)threadIdx.x;
        int32_t st;
        double c;
        lat_rec(*sm.lane, r, &st, &c);
        if (c + lat_key2d(bk[u]) > sm.cutoff) continue;
        atomicMin(&sm.min_beta, bk[u]);
        if (atomicAdd(&sm.nmap, 1) >= LAT_MAP / 2) continue;
        uint32_t h = lat_hash((uint32_t)st, 32 - LAT_MAP_LOG2);
        while (atomicCAS(&sm.mst[h], CTW_EMPTY, (uint32_t)st) != CTW_EMPTY) h = (h + 1) & (LAT_MAP - 1);
        sm.mnode[h] = (int32_t)(sm.S0 + r);
        sm.mbeta[h] = bk[u];
      }
    }
    __syncthreads();
    if (sm.nmap > LAT_MAP / 2) {  // same decision in every rank (same layer data): all leave together
      ovf = true;
      break;
    }
    // ---- sources: layer f-1 (records) or the seeds, split over the ranks
    if ((int)threadIdx.x == 0) {
      const int s0 = sm.f > 0 ? (int)sm.lane->frame_base[sm.f - 1] : 0;
      sm.s0 = s0;
      sm.nsrc = (sm.f > 0 ? d0 : sm.S0) - s0;
      sm.mb = sm.min_beta == ~0ULL ? INF : lat_key2d(sm.min_beta);
      sm.row0 = sm.E->ll_off + (long long)sm.f * a.width;
      // this rank's share: an equal contiguous slice (tiles of LAT_IBS)
      const int nsrc = sm.nsrc, rn = (int)cl.num_blocks(), rk = (int)cl.block_rank();
      const int share = (nsrc + rn - 1) / rn;
      sm.t0 = min(nsrc, rk * share);
      sm.t1 = min(nsrc, (rk + 1) * share);
    }
    __syncthreads();
    if (sm.min_beta != ~0ULL) {
      while (sm.t0 < sm.t1) {
        const int si = sm.t0 + (int)threadIdx.x;
        int deg = 0;
        const double step_lb = lat_key2d(sm.ac_min) + sm.E->emit_lb;  // any emitting step costs at least this
        if (si < sm.t1) {
          int32_t st0;
          double c0s;
          int nd;
          if (sm.f > 0) {
            lat_rec(*sm.lane, sm.s0 + si, &st0, &c0s);
            nd = sm.S0 + sm.s0 + si;
          } else {
            st0 = sm.E->seeds[si].state;
            c0s = sm.E->seeds[si].cost;
            nd = si;
          }
          const CtwStateRange rg = a.g.ranges[(uint32_t)st0 & sm.lane->smask];
          deg = (int)(rg.emit_end - rg.emit_beg);
          if (sm.cut_ok && c0s + step_lb + sm.mb > sm.cutoff + 1e-9 * fabs(sm.cutoff)) deg = 0;
          sm.beg[(int)threadIdx.x] = rg.emit_beg;
          sm.sst[(int)threadIdx.x] = st0;
          sm.sc[(int)threadIdx.x] = c0s;
          sm.node[(int)threadIdx.x] = nd;
        }
        int ex, tot;
        LatIdxSmem::Scan(sm.scan).ExclusiveSum(deg, ex, tot);
        sm.off[(int)threadIdx.x] = ex;
        __syncthreads();
        const int nv = min(LAT_IBS, sm.t1 - sm.t0);
        for (int item = (int)threadIdx.x; item < tot; item += LAT_IBS) {
          int lo = 0, hi = nv - 1;  // last source with off <= item
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (sm.off[mid] <= item) lo = mid;
            else hi = mid - 1;
          }
          lat_item_idx(a, sm, lo, sm.beg[lo] + (uint32_t)(item - sm.off[lo]));
        }
        __syncthreads();  // the tile's smem is reused by the next tile
        if (threadIdx.x == 0) sm.t0 += LAT_IBS;
        __syncthreads();
      }
    }
    cl.sync();  // the layer's arcs are out; beta of layer f-1 final in every rank
    if (threadIdx.x == 0) sm.f -= 1;
  }
  if (threadIdx.x == 0) {
    CtwLatEntry& Ex = *sm.E;
    atomicAdd(reinterpret_cast<unsigned long long*>(&Ex.closure_items), sm.items);
    atomicAdd(reinterpret_cast<unsigned long long*>(&Ex.closure_pruned), sm.pruned);
    if (cl.block_rank() == 0) {
      if (ovf) atomicMax(&Ex.status, 3);  // a layer map outgrew shared memory: general kernel re-run
      if (Ex.status == 0 && sm.best == ~0ULL) Ex.status = 4;
      Ex.final_mode = sm.final_mode;
      Ex.best = lat_key2d(sm.best);
    }
  }
}

}  // namespace

extern "C" int ctw_launch_lattice(CtwLane* d_lanes, const CtwStateRange* ranges, const CtwArc* arcs,
                                  const int32_t* olabel, const double* final_w, const uint32_t* clo_off,
                                  const CtwClo* clo_ent, CtwLatEntry* d_ent, int n, const void* loglik, int is_f64,
                                  int width, double acoustic_scale, double lattice_beam, int ranks, int big,
                                  cudaStream_t stream) {
  LatArgs a{d_lanes, LatGraph{ranges, arcs, olabel, final_w}, clo_off, clo_ent, d_ent, loglik, width, is_f64,
            acoustic_scale, lattice_beam};
  void (*KFN)(LatArgs) = big       ? k_lattice<LAT_CL_BIG, LAT_QL_BIG>
                         : clo_off ? k_lattice_idx
                                   : k_lattice<LAT_CL, LAT_QL>;
  (void)cudaGetLastError();
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)(n * ranks));
  lc.blockDim = dim3(KFN == k_lattice_idx ? LAT_IBS : LAT_BS);
  lc.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)ranks;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&lc, KFN, a);
  if (e != cudaSuccess) return (int)e;
  return (int)cudaGetLastError();
}

// ------------------------------------------------------- closure index --

namespace {

// One thread per state: its epsilon closure (label-correcting, minimum path
// weight from the state; the state itself first with weight 0). Pass 0
// counts (0 = too large to index), pass 1 writes the entries.
template <bool WRITE>
__global__ void __launch_bounds__(128) k_closure_index(const CtwStateRange* ranges, const CtwArc* arcs, long long S,
                                                       unsigned long long* cnt, const uint32_t* off, CtwClo* ent) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= S) return;
  if (WRITE && (off[s] & CTW_CLO_NONE)) return;
  const double INF = __longlong_as_double(0x7FF0000000000000LL);
  uint32_t cst[CLO_CAP];
  double cw[CLO_CAP];
  uint8_t q[CLO_QCAP];
  int n = 1, qh = 0, qt = 1;
  cst[0] = (uint32_t)s;
  cw[0] = 0.0;
  q[0] = 0;
  bool ovf = false;
  while (qh < qt && !ovf) {
    const int u = q[qh++];
    const CtwStateRange ru = ranges[cst[u]];
    for (uint32_t b = ru.eps_beg; b < ru.emit_beg; ++b) {
      const CtwArc ea = arcs[b];
      const double cy = __dadd_rn(cw[u], ea.weight);
      if (!(cy < INF)) continue;
      int j = 0;
      while (j < n && cst[j] != (uint32_t)ea.nextstate) ++j;
      if (j < n) {
        if (!(cy < cw[j])) continue;
      } else {
        if (n == CLO_CAP) {
          ovf = true;
          break;
        }
        ++n;
        cst[j] = (uint32_t)ea.nextstate;
      }
      cw[j] = cy;
      if (qt == CLO_QCAP) {
        ovf = true;
        break;
      }
      q[qt++] = (uint8_t)j;
    }
  }
  if (!WRITE) {
    cnt[s] = ovf ? 0ULL : (unsigned long long)n;
    return;
  }
  CtwClo* o = ent + (off[s] & ~CTW_CLO_NONE);
  for (int j = 0; j < n; ++j) {
    CtwClo e;
    e.w = cw[j];
    e.state = cst[j];
    e.pad = 0;
    o[j] = e;
  }
}

__global__ void k_closure_mark(const unsigned long long* cnt, const unsigned long long* off64, long long S,
                               uint32_t* off) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s > S) return;
  off[s] = (uint32_t)off64[s] | ((s < S && cnt[s] == 0) ? CTW_CLO_NONE : 0u);
}

}  // namespace

// Build the closure index of a graph (S states). Returns 0 and device
// arrays *off (S + 1 words) / *ent, or a CUDA error / -1 when the index
// would exceed 2^31 entries (the caller then runs the general kernel).
extern "C" int ctw_build_closure_index(const CtwStateRange* ranges, const CtwArc* arcs, long long S,
                                       uint32_t** off_out, CtwClo** ent_out, long long* n_out,
                                       cudaStream_t stream) {
  *off_out = nullptr;
  *ent_out = nullptr;
  *n_out = 0;
  unsigned long long *cnt = nullptr, *off64 = nullptr;
  uint32_t* off = nullptr;
  CtwClo* ent = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  unsigned long long total = 0;
  int rc = 0;
  const unsigned blocks = (unsigned)((S + 128) / 128);
  auto done = [&](int r) {
    cudaFree(cnt);
    cudaFree(off64);
    cudaFree(tmp);
    if (r) {
      cudaFree(off);
      cudaFree(ent);
    }
    return r;
  };
  if ((rc = cudaMalloc(&cnt, (S + 1) * 8)) || (rc = cudaMalloc(&off64, (S + 1) * 8)) ||
      (rc = cudaMalloc(&off, (S + 1) * 4)))
    return done(rc);
  if ((rc = cudaMemsetAsync(cnt + S, 0, 8, stream))) return done(rc);
  k_closure_index<false><<<blocks, 128, 0, stream>>>(ranges, arcs, S, cnt, nullptr, nullptr);
  if ((rc = cudaGetLastError())) return done(rc);
  if ((rc = cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, off64, S + 1, stream))) return done(rc);
  if ((rc = cudaMalloc(&tmp, tmp_bytes))) return done(rc);
  if ((rc = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, off64, S + 1, stream))) return done(rc);
  if ((rc = cudaMemcpyAsync(&total, off64 + S, 8, cudaMemcpyDeviceToHost, stream))) return done(rc);
  if ((rc = cudaStreamSynchronize(stream))) return done(rc);
  if (total >= (1ULL << 31)) return done(-1);
  k_closure_mark<<<(unsigned)((S + 256) / 256), 256, 0, stream>>>(cnt, off64, S, off);
  if ((rc = cudaGetLastError())) return done(rc);
  if ((rc = cudaMalloc(&ent, std::max<unsigned long long>(total, 1) * sizeof(CtwClo)))) return done(rc);
  k_closure_index<true><<<blocks, 128, 0, stream>>>(ranges, arcs, S, nullptr, off, ent);
  if ((rc = cudaGetLastError())) return done(rc);
  if ((rc = cudaStreamSynchronize(stream))) return done(rc);
  *off_out = off;
  *ent_out = ent;
  *n_out = (long long)total;
  return done(0);
}
