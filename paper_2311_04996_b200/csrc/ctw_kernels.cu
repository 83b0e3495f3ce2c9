// ctw_kernels.cu -- sm_100a kernels of the batched WFST beam-search decoder.
//
// One thread-block CLUSTER (1..CTW_RMAX CTAs, "ranks") owns one lane (= one
// decoding channel) for a whole chunk of frames and loops over the frames
// itself: emitting expansion -> epsilon fixpoint -> beam / max-active prune
// -> records + next sources -> table reset. The ranks of a lane share its
// token table in global memory (L2), hand out work through counters in rank
// 0's shared memory (DSMEM atomics) and meet at cluster barriers between
// stages. There is no host round trip and no grid-wide sync inside a chunk;
// the batch of lanes x ranks is the grid. Spreading a lane over several SMs
// cuts the per-frame latency (dependent L2 round trips are the bound) and
// keeps fewer lanes' token tables live in L2 at a time.
//
// Reference semantics (all paths under /root/reference/pkg/src/ctcwfst/):
//   expansion arithmetic  ((c + (-scale*ll[f, il-1])) + w) (+ boost[ol])
//                                                       _kernel.pyx:249-253
//   recombination: min cost per state, ties -> first arc in (source state,
//     arc) order == lowest global CSR arc index          _kernel.pyx:243-285
//   epsilon relaxation: Gauss-Seidel passes over the slot list until the
//     largest improvement of a pass is <= relax_eps; > max_ne_iters passes
//     -> ERR_EPS_ITERS                                    _kernel.pyx:292-355
//   no slots -> ERR_NO_SURVIVORS; keep cost <= min+beam, then the
//     max_active smallest (cost, state)                  _kernel.pyx:357-390
//   records (prev, olabels oldest-first, state, cost)    _kernel.pyx:392-427
//   seeding closure                                      decoder.py:173-229
//   best-path token choice + backtrace                   decoder.py:377-415
//
// The epsilon stage is computed as a parallel label-correcting fixpoint, not
// sequentially. Its result equals the reference's Gauss-Seidel result
// including exact-tie resolution: every slot carries its Gauss-Seidel slot
// position (gpos, see ctw_common.h) and every epsilon candidate the pass
// (pd) in which Gauss-Seidel would relax it with its final value, and equal
// costs are ordered by that event time (pd, gpos(pred), arc). The pass count
// checked against max_ne_iters is the Gauss-Seidel one (1 + max pd). See
// DESIGN.md "Epsilon closure".
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <cub/block/block_scan.cuh>
#include <stdint.h>

#include "ctw_common.h"

#ifndef CTW_BS
#define CTW_BS 512
#endif
#ifndef CTW_MINB
#define CTW_MINB (2048 / CTW_BS)  // 64 resident warps per SM: the kernel is latency-bound, occupancy pays
#endif
#ifndef CTW_DEFAULT_CLUSTER
#define CTW_DEFAULT_CLUSTER 8
#endif
#define CTW_WARPS (CTW_BS / 32)
#ifndef CTW_LD256
#define CTW_LD256 1  // token-table reads as one 256-bit load per entry (one L2 request, not two)
#endif
#ifndef CTW_EMPF
#define CTW_EMPF 1  // emitting stage: next round's arc load issued ahead (-3% emit cycles)
#endif
// Guided work chunks: chunk size once fewer than 32 items per warp of the
// lane remain (measured: 16 for the emitting stage; the epsilon passes are
// fastest without shrinking -- more claims cost more than the shorter tail)
#ifndef CTW_EMIT_TAIL_SZ
#define CTW_EMIT_TAIL_SZ 16
#endif
#ifndef CTW_EPS_TAIL_SZ
#define CTW_EPS_TAIL_SZ 32
#endif
#ifndef CTW_SRC256
#define CTW_SRC256 1  // sources read / written as one 256-bit access each (+0.8%)
#endif
#ifndef CTW_IDLE_PROF
#define CTW_IDLE_PROF 0
#endif
#ifndef CTW_EPS_INLINE
#define CTW_EPS_INLINE
#endif
#define CTW_IPT 4                        // sources per thread per expansion tile
#define CTW_TILE (CTW_BS * CTW_IPT)
#define CTW_MAX_SMEM_WIDTH 4096
#define CTW_PRED_BITS 24
#define CTW_PRED_MASK ((1u << CTW_PRED_BITS) - 1u)
#define CTW_KEY56 ((1ULL << 56) - 1ULL)
#define CTW_EIPT 2                       // frontier items per thread per epsilon tile
#define CTW_ETILE (CTW_BS * CTW_EIPT)
#define CTW_DISC 0xFFFFFFFFu             // epsilon tile item: discovery only (no value)
#ifndef CTW_NB
#define CTW_NB 1024      // cost-histogram bins over [min, min + beam] for the max-active select
#endif
#define CTW_BBUF 512     // boundary-bin capacity of the exact (cost, state) sort

namespace cg = cooperative_groups;

namespace {

struct Smem;

struct GraphDev {
  const CtwStateRange* ranges;
  const CtwArc* arcs;
  const int32_t* olabel;
  const double* final_w;
};

// ---------------------------------------------------------------- helpers --

__device__ __forceinline__ unsigned long long d2key(double x) {
  x = __dadd_rn(x, 0.0);  // -0.0 -> +0.0 (they compare equal in the reference)
  long long b = __double_as_longlong(x);
  return (unsigned long long)(b ^ ((b >> 63) | (long long)0x8000000000000000ULL));
}

__device__ __forceinline__ double key2d(unsigned long long k) {
  long long b = (k & 0x8000000000000000ULL) ? (long long)(k ^ 0x8000000000000000ULL) : (long long)~k;
  return __longlong_as_double(b);
}

__device__ __forceinline__ void cas128(void* addr, unsigned long long clo, unsigned long long chi,
                                       unsigned long long nlo, unsigned long long nhi,
                                       unsigned long long& olo, unsigned long long& ohi) {
  asm volatile(
      "{\n\t.reg .b128 c, n, o;\n\t"
      "mov.b128 c, {%2, %3};\n\t"
      "mov.b128 n, {%4, %5};\n\t"
      "atom.relaxed.gpu.global.cas.b128 o, [%6], c, n;\n\t"
      "mov.b128 {%0, %1}, o;\n\t}"
      : "=l"(olo), "=l"(ohi)
      : "l"(clo), "l"(chi), "l"(nlo), "l"(nhi), "l"(addr)
      : "memory");
}

// An atomic 128-bit snapshot: CAS with a compare value no live entry can hold
// (key 0 is the sortable image of a negative NaN, never stored).
__device__ __forceinline__ void snap128(void* addr, unsigned long long& lo, unsigned long long& hi) {
  cas128(addr, 0ULL, ~0ULL, 0ULL, ~0ULL, lo, hi);
}

__device__ __forceinline__ uint32_t tok_hash(uint32_t s, uint32_t shift) {
  return (s * 0x9E3779B1u) >> shift;
}

// Graph reads (16 B vector loads through the read-only path).
__device__ __forceinline__ CtwArc ld_arc(const CtwArc* arcs, uint32_t i) { return arcs[i]; }

__device__ __forceinline__ CtwStateRange ld_range(const CtwStateRange* ranges, uint32_t s) { return ranges[s]; }

struct LaneCtx {
  CtwTok* T;
  uint32_t mask, shift, tcap;
  uint32_t seg;        // capacity of the slot list and of each frontier set (CTW_LOAD(tcap))
  uint2* slots;        // the frame's slot list: (table index, state), cluster-wide, discovery order
  uint2* front;        // frontier sets (CTW_FRONT_LEN)
  Smem* G;             // rank 0's shared memory (cluster counters)
  int* slot_ctr;       // cluster-wide slot allocation counter of the frame (rank 0)
  int rank, nranks;
  int sw0, swstride;   // slot sweeps: this rank handles sw0 + tid + k * swstride
  int pool_cap;
  int32_t* pool;
  bool prune;    // CtwLane::prune_ok
  int* tie_ctr;  // diagnostics: epsilon/epsilon ties between distinct predecessors
  // phrase automaton (on-the-fly composition with a multi-state boost FST):
  // token key = graph state | automaton state << sbits; null fnext = none
  const uint16_t* fnext;
  const double* fcost;
  int32_t fwidth;
  uint32_t sbits, smask;
  // fast search mode (FastEnt table view of the same allocation, see below)
  ulonglong2* V;
  uint32_t tlog2, ebits;
  bool eps_lab;  // some epsilon arc of the graph carries an output label
};

// ------------------------------------------------------ fast search mode --
//
// Words-exact search (north star: best-path words bit-exact, cost within
// 1e-4) without the Gauss-Seidel slot-position machinery of the exact mode:
//  * a 16 B token entry {f64 cost key, u32 state, u32 winner} -- two entries
//    per 32 B sector, probed and relaxed with one 128-bit access each
//    (the north star's "packed atomicMin": the cost key and its backpointer
//    change together in one atom.cas.b128);
//  * candidates above the running cutoff (running min + beam) are never
//    inserted (exact for the final beam: the frame minimum only decreases and
//    epsilon increments are >= 0 -- CtwLane::prune_ok is required);
//  * the epsilon closure is a plain label-correcting fixpoint over the
//    in-beam states (full propagation: costs are the exact min over paths,
//    <= the reference's relax_eps-stopped values by at most ~relax_eps);
//  * exact-cost ties: emitting candidates by the lowest arc index (the
//    reference's first writer, _kernel.pyx:256-285), an emitting winner stays
//    against epsilon candidates (_kernel.pyx:332), epsilon candidates among
//    themselves by the lowest arc index (deterministic; the reference orders
//    them by Gauss-Seidel event time).
// Winner word: emitting = src_idx << ebits | arc offset in the source's
// emitting range; epsilon = EPS | offset << tlog2 | predecessor table index.
// The table allocation is the exact mode's (32 B x tcap); the fast view uses
// its first 16 B x tcap. A clean fast entry {~0, EMPTY, 0} is bytewise the
// clean exact pattern (every even 64-bit word ~0, every odd one 0xFFFFFFFF),
// so both views stay valid between frames and a lane set may switch modes.
#define CTW_FEPS 0x80000000u

__device__ __forceinline__ uint32_t fwin_emit(uint32_t src_idx, uint32_t off, uint32_t ebits) {
  return (src_idx << ebits) | off;
}

// Find-or-insert `d` in the fast table; *v gets a historical snapshot of the
// entry (only ever used as a CAS expected value / lower bound).
__device__ __forceinline__ uint32_t ftok_locate(const LaneCtx& L, uint32_t d, ulonglong2* v, bool& is_new) {
  uint32_t h = tok_hash(d, L.shift);
  for (uint32_t probe = 0; probe <= L.mask; ++probe) {
    const ulonglong2 val = __ldcg(&L.V[h]);
    const uint32_t k = (uint32_t)val.y;
    if (k == d) {
      *v = val;
      return h;
    }
    if (k == CTW_EMPTY) {
      const uint32_t old = atomicCAS(reinterpret_cast<uint32_t*>(&L.V[h]) + 2, CTW_EMPTY, d);
      if (old == CTW_EMPTY || old == d) {
        is_new = old == CTW_EMPTY;
        *v = make_ulonglong2(~0ULL, (unsigned long long)d);  // the claimed entry's first value
        return h;
      }
    }
    h = (h + 1) & L.mask;
  }
  return CTW_EMPTY;
}

// Arc index behind a fast winner word (exact-tie resolution, walks).
__device__ __forceinline__ uint32_t fwin_arc(const LaneCtx& L, const GraphDev& g, const CtwSrc* src, uint32_t w) {
  // (sources are written by this kernel: coherent loads, not the read-only path)
  if (!(w & CTW_FEPS)) return __ldcg(&src[w >> L.ebits].emit_beg) + (w & ((1u << L.ebits) - 1u));
  const uint32_t pred = w & L.mask;
  const uint32_t st = (uint32_t)__ldcg(&L.V[pred]).y & L.smask;
  return __ldg(&g.ranges[st].eps_beg) + ((w & ~CTW_FEPS) >> L.tlog2);
}

// Relax fast entry e with candidate (key, winner w over arc `arc`).
__device__ __forceinline__ bool ftok_relax(const LaneCtx& L, const GraphDev& g, const CtwSrc* src, ulonglong2* e,
                                           unsigned long long key, uint32_t w, uint32_t arc, ulonglong2 seen,
                                           unsigned long long* old_key) {
  if (key > seen.x) return false;
  unsigned long long clo = seen.x, chi = seen.y;
  if (key == clo) snap128(e, clo, chi);
  for (;;) {
    if (key > clo) return false;
    if (key == clo) {
      const uint32_t cw = (uint32_t)(chi >> 32);
      if (!(w & CTW_FEPS)) {
        if (!(cw & CTW_FEPS) && arc >= fwin_arc(L, g, src, cw)) return false;
      } else {
        if (!(cw & CTW_FEPS)) return false;  // an equal-cost emitting winner stays
        if (arc >= fwin_arc(L, g, src, cw)) return false;
      }
    }
    unsigned long long olo, ohi;
    const unsigned long long nhi = (chi & 0xFFFFFFFFULL) | ((unsigned long long)w << 32);
    cas128(e, clo, chi, key, nhi, olo, ohi);
    if (olo == clo && ohi == chi) {
      *old_key = clo;
      return true;
    }
    clo = olo;
    chi = ohi;
  }
}

__device__ __forceinline__ void ftok_clear(ulonglong2* e) {
  asm volatile("st.global.cg.v2.u64 [%0], {%1, %2};" ::"l"(e), "l"(~0ULL), "l"(0xFFFFFFFFULL) : "memory");
}

// The (key, winner) value of table entry h in either view: exact mode keeps
// (key, tb | aux << 32) in the first 16 B of its 32 B entry; fast mode's 16 B
// entry is (key, state | winner << 32).
template <bool FAST>
__device__ __forceinline__ ulonglong2* tval(const LaneCtx& L, uint32_t h) {
  return FAST ? L.V + h : reinterpret_cast<ulonglong2*>(&L.T[h]);
}

// Destination key and boost of an arc with output label ol leaving the token
// with key `key` (reference order: the boost is added after the arc weight,
// _kernel.pyx:251-252): the dense word table, or the phrase automaton's
// transition (the key carries the automaton state; only word arcs move it).
template <bool FSA>
__device__ __forceinline__ uint32_t arc_dest(const LaneCtx& L, const double* boost, uint32_t key, int32_t ol,
                                             uint32_t nextstate, double& nc) {
  if (FSA && L.fnext) {
    uint32_t b = key >> L.sbits;
    if (ol != 0) {
      b = L.fnext[(size_t)b * L.fwidth + ol];
      nc = __dadd_rn(nc, L.fcost[b]);
    }
    return nextstate | (b << L.sbits);
  }
  if (boost && ol != 0) nc = __dadd_rn(nc, boost[ol]);
  return nextstate;
}

// Find-or-insert `d` (linear probing). Returns the table index or CTW_EMPTY
// when the table is full.
__device__ __forceinline__ uint32_t tok_insert(const LaneCtx& L, uint32_t d, bool& is_new) {
  uint32_t h = tok_hash(d, L.shift);
  for (uint32_t probe = 0; probe <= L.mask; ++probe) {
    // one L2 round trip per probe: the CAS both claims a free entry and
    // reports an occupied one
    const uint32_t old = atomicCAS(&L.T[h].state, CTW_EMPTY, d);
    if (old == CTW_EMPTY) {
      is_new = true;
      return h;
    }
    if (old == d) return h;
    h = (h + 1) & L.mask;
  }
  return CTW_EMPTY;
}

// Fire-and-forget slot-position update (compiles to RED.MIN: no round trip).
__device__ __forceinline__ void gpos_min(CtwTok* e, unsigned long long v) {
  atomicMin(&e->gpos, v);
}

// The whole 32 B entry in one L2 request (sm_100 256-bit load, L2 only).
// 64-bit elements: each half of (key, tb|aux) stays single-copy atomic, as
// the relax logic assumes (a key read is always a historical key).
__device__ __forceinline__ void ld_tok(const CtwTok* e, ulonglong2& v, unsigned long long& gpos, uint32_t& state) {
#if CTW_LD256
  unsigned long long w3;
  asm volatile("ld.global.cg.v4.u64 {%0, %1, %2, %3}, [%4];"
               : "=l"(v.x), "=l"(v.y), "=l"(gpos), "=l"(w3)
               : "l"(e));
  state = (uint32_t)w3;  // (stamp in the upper half)
#else
  v = __ldcg(reinterpret_cast<const ulonglong2*>(e));
  gpos = __ldcg(&e->gpos);
  state = __ldcg(&e->state);
#endif
}

// Find-or-insert `d` and return a snapshot of its (key, tb|aux) in *v: the
// probe reads the entry's value and hash key together (plain loads; a
// claimed hash key never changes within a frame), so a hit costs one round
// trip and feeds the relax CAS directly; a fresh insert returns the empty
// value. The snapshot may be stale or torn -- it is only ever used as the
// expected value of a CAS, which then fails and reports the exact value.
__device__ __forceinline__ uint32_t tok_locate(const LaneCtx& L, uint32_t d, ulonglong2* v, bool& is_new) {
  uint32_t h = tok_hash(d, L.shift);
  for (uint32_t probe = 0; probe <= L.mask; ++probe) {
    const CtwTok* e = &L.T[h];
#if CTW_LD256
    ulonglong2 val;
    unsigned long long gp_;
    uint32_t k;
    ld_tok(e, val, gp_, k);
#else
    const ulonglong2 val = __ldcg(reinterpret_cast<const ulonglong2*>(e));
    const uint32_t k = __ldcg(&e->state);
#endif
    if (k == d) {
      *v = val;
      return h;
    }
    if (k == CTW_EMPTY) {
      const uint32_t old = atomicCAS(&L.T[h].state, CTW_EMPTY, d);
      if (old == CTW_EMPTY) {
        is_new = true;
        *v = make_ulonglong2(~0ULL, 0xFFFFFFFFULL);
        return h;
      }
      if (old == d) {
        *v = val;
        return h;
      }
    }
    h = (h + 1) & L.mask;
  }
  return CTW_EMPTY;
}

// Gauss-Seidel event order of two epsilon candidates with equal cost:
// (pd, slot position of the predecessor, arc).
__device__ __forceinline__ bool gs_before(const CtwTok* T, uint32_t pd_a, uint32_t pred_a, uint32_t arc_a,
                                          unsigned long long gpos_a, uint32_t aux_b, uint32_t arc_b) {
  const uint32_t pd_b = aux_b >> CTW_PRED_BITS;
  if (pd_a != pd_b) return pd_a < pd_b;
  const uint32_t pred_b = aux_b & CTW_PRED_MASK;
  if (pred_a == pred_b) return arc_a < arc_b;
  const unsigned long long gpos_b = __ldcg(&T[pred_b].gpos);
  if (gpos_a != gpos_b) return gpos_a < gpos_b;
  return pred_a < pred_b;  // only on saturated chain keys (deterministic)
}

// Relax entry e with candidate (key, tb, aux). Emitting candidates: tb = arc,
// aux = source index. Epsilon candidates: tb = EPS|arc, aux = pd<<24|pred,
// gpos_pred = gpos of the predecessor. Returns true when installed; *old_key
// gets the replaced cost key (~0 = the entry was empty).
__device__ __forceinline__ bool tok_relax_from(const LaneCtx& L, CtwTok* e, unsigned long long key, uint32_t tb,
                                               uint32_t aux, unsigned long long gpos_pred, ulonglong2 seen,
                                               unsigned long long* old_key) {
  // seen.x is a historical key (64-bit halves are single-copy atomic), and
  // keys only decrease within a frame: key > seen.x rejects safely
  if (key > seen.x) return false;
  unsigned long long clo = seen.x, chi = seen.y;
  if (key == clo) snap128(e, clo, chi);  // exact tie: need an untorn incumbent
  const unsigned long long nhi = ((unsigned long long)aux << 32) | tb;
  for (;;) {
    if (key > clo) return false;
    if (key == clo) {
      const uint32_t ctb = (uint32_t)chi;
      if (!(tb & CTW_EPS_BIT)) {
        if (tb >= ctb) return false;  // emitting: first (lowest) arc wins
      } else {
        if (!(ctb & CTW_EPS_BIT)) return false;  // equal-cost emitting / seed winner stays
        if (((uint32_t)(chi >> 32) & CTW_PRED_MASK) != (aux & CTW_PRED_MASK) && L.tie_ctr) atomicAdd(L.tie_ctr, 1);
        if (!gs_before(L.T, aux >> CTW_PRED_BITS, aux & CTW_PRED_MASK, tb & ~CTW_EPS_BIT, gpos_pred,
                       (uint32_t)(chi >> 32), ctb & ~CTW_EPS_BIT))
          return false;
      }
    }
    unsigned long long olo, ohi;
    cas128(e, clo, chi, key, nhi, olo, ohi);
    if (olo == clo && ohi == chi) {
      *old_key = clo;
      return true;
    }
    clo = olo;
    chi = ohi;
  }
}

__device__ __forceinline__ bool tok_relax(const LaneCtx& L, CtwTok* e, unsigned long long key, uint32_t tb,
                                          uint32_t aux, unsigned long long gpos_pred, unsigned long long* old_key) {
  return tok_relax_from(L, e, key, tb, aux, gpos_pred, __ldcg(reinterpret_cast<const ulonglong2*>(e)), old_key);
}

__device__ __forceinline__ void tok_clear(CtwTok* e) {
#if CTW_LD256
  // key, tb=~0, aux=0 | gpos=~0, state=EMPTY, stamp=0: one 256-bit store
  asm volatile("st.global.cg.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(e), "l"(~0ULL), "l"(0xFFFFFFFFULL), "l"(~0ULL),
               "l"((unsigned long long)CTW_EMPTY)
               : "memory");
#else
  ulonglong2* p = reinterpret_cast<ulonglong2*>(e);
  __stcg(p, make_ulonglong2(~0ULL, 0xFFFFFFFFULL));                          // key, tb=~0, aux=0
  __stcg(p + 1, make_ulonglong2(~0ULL, (unsigned long long)CTW_EMPTY));     // gpos=~0, state, stamp=0
#endif
}

// --------------------------------------------------------- shared memory --

#ifndef CTW_NBIG
#define CTW_NBIG 2048  // high out-degree sources expanded arc-parallel per frame (list capacity)
#endif
#ifndef CTW_BIG
#define CTW_BIG 16  // emitting out-degree above which a source is expanded arc-parallel (64: -2.5%)
#endif

// Per-frame cluster counters. They live in rank 0 and are double-buffered by
// frame parity: rank 0 zeroes the other parity's copy after the frame-start
// barrier, when no rank can still read it and none uses it before the next
// frame-start barrier.
struct FrameCtr {
  int work_e;   // emitting: source chunks handed out
  int work_b;   // emitting: arc chunks of the high-degree list handed out
  int nbig;     // high-degree sources listed
  int cnt;      // in-beam slots
  int max_pd;   // Gauss-Seidel pass depth of the closure
  int nbb;      // boundary-bin members collected
  int rec_ctr;  // survivors written (records of the frame)
  int nslot;    // slots allocated (the slot list's fill)
  int nib;      // in-beam slots compacted by the count pass
  uint32_t bhist[CTW_NB];      // cost histogram over [min, min + beam]
};

// One high out-degree source, listed for the arc-parallel pass (global scratch).
struct BigSrc {
  int32_t idx;  // source index (emitting winners' aux)
  uint32_t beg;
  int32_t deg;
  int32_t pad;
  double cost;
};

struct __align__(16) Smem {
  typedef cub::BlockScan<int, CTW_BS> Scan;
  typename Scan::TempStorage scan;
  union {
    struct {  // emitting expansion: each warp's current chunk of 32 sources
      double cost[CTW_WARPS][32];
      int off[CTW_WARPS][32];
      uint32_t beg[CTW_WARPS][32];
    } em;
    struct {  // epsilon closure: each warp's current chunk of 32 frontier items
      double cost[CTW_WARPS][32];
      unsigned long long gu[CTW_WARPS][32];  // the item's own slot position (tie-break)
      int off[CTW_WARPS][32];
      uint32_t beg[CTW_WARPS][32];
      uint32_t aux[CTW_WARPS][32];           // pd << 24 | table index, or CTW_DISC
    } ep;
    struct {  // arc-parallel expansion of the high-degree sources
      int pref[CTW_NBIG + 1];
    } bg;
    ulonglong2 bbuf[CTW_BBUF];  // rank 0: max-active boundary bin (cost key, state)
    struct {  // count / select stages (the expansion buffers are free then)
      uint32_t lbhist[CTW_NB];  // local cost histogram
      uint32_t hist[256];       // local digit histogram (radix select)
      uint32_t rhist[2][256];   // rank 0: merged radix digit histogram (digit parity)
    } cs;
  };
  // ---- cluster fields: meaningful in rank 0 only, reached through DSMEM ----
  FrameCtr fc[2];
  int pw[2];            // epsilon pass chunk counters (pass parity)
  int pcnt[3][2];       // frontier pushes (next, tiny) of pass p, at [p % 3]
  int pool_used;        // olabel pool fill
  int sel_bin, sel_need, sel_bcount, sel_radix;
  unsigned long long thr_key;  // survivor iff bin < sel_bin or (bin == sel_bin and (key, state) <= thr)
  uint32_t thr_state;
  unsigned long long sel_hi;  // radix-select prefix (cost-key digits)
  uint32_t sel_lo;            // radix-select prefix (state digits)
  int sel_depth;              // digits fixed; survivor iff top digits <= prefix
  int rneed;
  int sel_done;
  // ---- per-rank fields ----
  int status_l;         // sticky local status (grow requests, walk failures)
  int st_pub[2];        // status published at a barrier (barrier parity)
  unsigned long long min_pub[2];  // running minimum published at a barrier (barrier parity)
  // kernel-level bookkeeping kept by tid 0 (not live registers in every thread)
  long long tclk, src_total, rec_need, n_rec;
  int n_slots_max, err_frame;
  unsigned long long eps_idle;  // CTW_IDLE_PROF: warp-cycles waiting at the epsilon pass barriers
  unsigned long long mydiag[CTW_NPROF + 1];  // this rank's diagnostics, read by rank 0 at the end
  int epoch;            // barriers passed (all ranks pass the same sequence)
  int st_all;           // max status over the ranks at the last barrier
  int n_slots;          // slots this rank created in the frame
  int snap_slots;       // n_slots at the start of the epsilon stage
  int pc_big[2];        // this rank made a big change in the pass (pass parity)
  // the epsilon pass's parameters, read where used instead of being held in
  // registers across the chunk loop (32-register budget: +3% measured)
  int* eo_ctr;          // output counters of the pass
  uint2* eo_nxt;        // output sets of the pass
  uint2* eo_tiny;
  double eo_relax;      // relax_eps
  double eo_beam;
  int n_cur, n_first, any_big;
  uint2* in0;           // input of the current epsilon pass: in0[0, n_first) ++ in1[0, n_cur - n_first)
  uint2* in1;
  unsigned long long min_key;  // running minimum seen by this rank (>= the cluster's)
  int n_all;            // slots of all ranks (after the closure)
  int cnt_l, mpd_l, cnt_all, mpd_all;
  int nbig;
  int rbase;            // first survivor index of this rank in the frame
  int tot_surv;
  int passes;
  int eps_items, eps_arcs, eps_ties, eps_disc;
  int arcs_f;           // emitting arcs expanded in the frame (diagnostics)
  // local copies of the select result
  int l_bin, l_need, l_bcount, l_radix, l_depth;
  unsigned long long l_tk, l_ph;
  uint32_t l_ts, l_pl;
};

// Warp-aggregated append to a cluster-wide list: one DSMEM atomic per
// converged group of appending threads; returns this thread's index.
__device__ __forceinline__ int agg_alloc(int* ctr, int* local_ctr) {
  cg::coalesced_group grp = cg::coalesced_threads();
  int base = 0;
  if (grp.thread_rank() == 0) {
    base = atomicAdd(ctr, (int)grp.size());
    if (local_ctr) atomicAdd(local_ctr, (int)grp.size());
  }
  return grp.shfl(base, 0) + (int)grp.thread_rank();
}

// Append a newly inserted table index to the frame's slot list; request a
// bigger table when the list is full (the table is grown past 3/4 load).
__device__ __forceinline__ void slot_append(Smem& sm, const LaneCtx& L, uint32_t h, uint32_t state) {
  const int s = agg_alloc(L.slot_ctr, &sm.n_slots);
  if ((uint32_t)s < L.seg) L.slots[s] = make_uint2(h, state);
  else atomicMax(&sm.status_l, CTW_GROW_TABLE);
}

__device__ __forceinline__ void track_min(Smem& sm, unsigned long long k) {
  if (k < *((volatile unsigned long long*)&sm.min_key)) atomicMin(&sm.min_key, k);
}

// Running beam cutoff: the frame minimum only decreases, so a cost above
// (running min + beam) is above the final cutoff too. Each rank uses its own
// running minimum (never below the cluster's), which is looser, hence exact.
__device__ __forceinline__ double running_cut(const Smem& sm, double beam) {
  return __dadd_rn(key2d(*((volatile const unsigned long long*)&sm.min_key)), beam);
}

// Cluster barrier with a status vote and a minimum exchange: every rank
// publishes its sticky local status and its running minimum in its own
// shared memory, passes the barrier and reads everyone's, so all ranks take
// the same branch and leave with the same (cluster-wide) running minimum.
// Published values are double-buffered by barrier parity (a rank rewrites a
// slot only after every rank has passed the barrier that follows the reads
// of it). Plain stores + remote loads: shared memory has no native 64-bit
// min, and a generic 64-bit atomic min on a DSMEM address is not atomic.
__device__ __forceinline__ int csync(Smem& sm) {
  cg::cluster_group cl = cg::this_cluster();
  __syncthreads();
  const int e = sm.epoch;
  if (threadIdx.x == 0) {
    sm.st_pub[e & 1] = *((volatile int*)&sm.status_l);
    sm.min_pub[e & 1] = *((volatile unsigned long long*)&sm.min_key);
  }
  cl.sync();
  if (threadIdx.x < 32) {
    // warp 0: lane k reads rank k's published values (one DSMEM round trip
    // for all ranks), then a warp reduction
    const int k = threadIdx.x;
    int s = 0;
    unsigned long long m = ~0ULL;
    if (k < (int)cl.num_blocks()) {
      const Smem* o = cl.map_shared_rank(&sm, k);
      s = o->st_pub[e & 1];
      m = o->min_pub[e & 1];
    }
    for (int d = 16; d; d >>= 1) {
      s = max(s, __shfl_xor_sync(0xFFFFFFFFu, s, d));
      const unsigned long long mo = __shfl_xor_sync(0xFFFFFFFFu, m, d);
      if (mo < m) m = mo;
    }
    if (k == 0) {
      sm.st_all = s;
      if (m < sm.min_key) sm.min_key = m;
      sm.epoch = e + 1;
    }
  }
  __syncthreads();
  return sm.st_all;
}

// Relax one epsilon arc a (loaded: arc) of the frontier item lo of warp w:
// (c + w) (+ boost), find-or-insert the destination, update its slot
// position, install the candidate if it wins the Gauss-Seidel order, and
// queue the destination for the next pass when it changed.
template <bool FSA>
__device__ __forceinline__ void eps_arc(Smem& sm, const LaneCtx& L, const GraphDev& g, const double* boost,
                                        int w, int lo, uint32_t o, uint32_t a, const CtwArc& arc, uint32_t ikey) {
  const double INF = __longlong_as_double(0x7FF0000000000000LL);
  const uint32_t aux = sm.ep.aux[w][lo];
  const bool valued = aux != CTW_DISC;
  double nc = valued ? __dadd_rn(sm.ep.cost[w][lo], arc.weight) : arc.weight;
  uint32_t dkey = (uint32_t)arc.nextstate;
  if (FSA) {
    double nb = nc;
    dkey = arc_dest<FSA>(L, boost, ikey, g.olabel[a], (uint32_t)arc.nextstate, nb);
    if (valued) nc = nb;
  } else if (boost && valued) {
    const int32_t ol = g.olabel[a];
    if (ol != 0) nc = __dadd_rn(nc, boost[ol]);
  }
  if (!(nc < INF)) return;
  bool is_new = false;
  ulonglong2 seen;
  const uint32_t d = tok_locate(L, dkey, &seen, is_new);
  if (d == CTW_EMPTY) {
    atomicMax(&sm.status_l, CTW_GROW_TABLE);
    return;
  }
  if (is_new) slot_append(sm, L, d, dkey);
  CtwTok* ed = &L.T[d];
  // slot-position chain key handed to a discovered successor:
  // level + 1, discoverer's key << 4 | arc offset
  const unsigned long long gu = sm.ep.gu[w][lo];
  gpos_min(ed, ((((gu >> 56) + 1) << 56) | ((gu << 4) & CTW_KEY56)) | min(o, 15u));
  const uint2 item = make_uint2(d, dkey);
  bool push = false, big = false;
  if (valued) {
    unsigned long long oldk;
    const unsigned long long nk = d2key(nc);
    if (tok_relax_from(L, ed, nk, CTW_EPS_BIT | a, aux, sm.ep.gu[w][lo], seen, &oldk)) {
      track_min(sm, nk);
      push = true;
      big = is_new || oldk == ~0ULL || oldk == nk || (key2d(oldk) - nc) > sm.eo_relax;
    } else {
      push = big = is_new;
    }
  } else {
    push = big = is_new;  // discovery only: successors are discovered next pass
  }
  if (!push) return;
  // the pass's parameters come from shared memory (not registers held
  // across the chunk loop): read only on the push path
  const uint32_t epoch = (uint32_t)sm.passes;
  const int q = sm.passes & 1;
  int* ctr_out = sm.eo_ctr;
  uint2* nxt = sm.eo_nxt;
  uint2* tiny = sm.eo_tiny;
  if (big) sm.pc_big[q] = 1;
  bool first;
  if (is_new) {  // this thread created the slot: first to touch its stamp
    ed->stamp = epoch;
    first = true;
  } else {
    first = atomicExch(&ed->stamp, epoch) != epoch;
  }
  if (first) {
    int p;
    uint2* dst;
    if (big) {  // one counter per coalesced group
      p = agg_alloc(&ctr_out[0], nullptr);
      dst = nxt;
    } else {
      p = agg_alloc(&ctr_out[1], nullptr);
      dst = tiny;
    }
    if ((uint32_t)p < L.seg) dst[p] = item;
    else atomicMax(&sm.status_l, CTW_GROW_TABLE);
  }
}

// ------------------------------------------------------- epsilon fixpoint --

// Label-correcting fixpoint over epsilon arcs, frontier by frontier; the
// input of pass 1 is every slot created so far (all ranks' segments). A slot
// is re-queued when it is new, improved by more than relax_eps, or changed
// winner at equal cost (its Gauss-Seidel event time moved). Improvements <=
// relax_eps are propagated only if the pass goes on anyway, mirroring the
// Gauss-Seidel stop rule (_kernel.pyx:331, :346, :351). With L.prune, a
// predecessor whose cost is above the running cutoff (or that has no value
// yet) only *discovers* its successors -- slot positions stay exact --
// without relaxing their costs: with non-negative epsilon increments nothing
// it reaches can enter the beam. Work of a pass is handed out cluster-wide in
// 32-item chunks over the virtual concatenation of the ranks' input segments;
// every rank pushes to its own output segments. Returns CTW_OK or
// CTW_ERR_EPS_ITERS (divergence: more passes than a convergent closure needs).
template <bool FSA>
__device__ CTW_EPS_INLINE int eps_fixpoint(Smem& sm, const LaneCtx& L, const GraphDev& g, FrameCtr* fc, const double* boost,
                            double relax_eps, double beam, long long pass_cap) {
  cg::cluster_group cl = cg::this_cluster();
  const int tid = threadIdx.x;
  const int R = L.nranks, rank = L.rank;
  Smem* G = L.G;
  const double INF = __longlong_as_double(0x7FF0000000000000LL);
  for (long long pass = 1;; ++pass) {
    const int q = (int)(pass & 1);
    const int so = 2 * (int)((pass - 1) & 1);  // output sets of this pass
    uint2* nxt = L.front + (size_t)so * L.seg;
    uint2* tiny = L.front + (size_t)(so + 1) * L.seg;
    int* ctr_out = G->pcnt[pass % 3];
    if (tid == 0) {
      if (pass == 1) {
        // every slot created before the stage (the ranks' published counts)
        int tot = 0;
        for (int k = 0; k < R; ++k) tot += cl.map_shared_rank(&sm, k)->snap_slots;  // once per frame
        sm.in0 = L.slots;
        sm.n_first = min(tot, (int)L.seg);
        sm.in1 = L.slots;
        sm.n_cur = sm.n_first;
      } else {
        const int si = 2 * (int)((pass - 2) & 1);
        const int* ci = G->pcnt[(pass - 1) % 3];
        const int nn = min(*((volatile const int*)&ci[0]), (int)L.seg);
        const int nt = min(*((volatile const int*)&ci[1]), (int)L.seg);
        sm.in0 = L.front + (size_t)si * L.seg;
        sm.n_first = nn;
        sm.in1 = L.front + (size_t)(si + 1) * L.seg;
        sm.n_cur = nn + nt;
      }
      sm.pc_big[q] = 0;
      if (rank == 0) {
        sm.pw[q ^ 1] = 0;                          // the next pass's chunk counter
        sm.pcnt[(pass + 1) % 3][0] = 0;            // written in pass + 1; last read in pass - 1
        sm.pcnt[(pass + 1) % 3][1] = 0;
      }
      sm.passes = (int)pass;
      sm.eo_ctr = ctr_out;
      sm.eo_nxt = nxt;
      sm.eo_tiny = tiny;
      sm.eo_relax = relax_eps;
      sm.eo_beam = beam;
    }
    __syncthreads();
    if (pass > pass_cap) return CTW_ERR_EPS_ITERS;
    const int n_cur = sm.n_cur, n_first = sm.n_first;
    const int tail = 32 * CTW_WARPS * R;  // items left when chunks shrink
    const uint2* in0 = sm.in0;
    const uint2* in1 = sm.in1;
    // warps grab 32 frontier items at a time and spread the items' epsilon
    // arcs over their lanes
    const int lane = tid & 31, w = tid >> 5;
    // chunks of 32 items (CTW_EPS_TAIL_SZ near the end of the pass when
    // guided); a claim is (base << 1) | (size == CTW_EPS_TAIL_SZ)
    auto claim = [&]() -> int {
      int c = 0;
      if (lane == 0) {
#if CTW_EPS_TAIL_SZ < 32
        const bool small = n_cur - *((volatile int*)&G->pw[q]) < tail;
#else
        const bool small = false;  // (no remote read of the counter)
        (void)tail;
#endif
        c = (atomicAdd(&G->pw[q], small ? CTW_EPS_TAIL_SZ : 32) << 1) | (small ? 1 : 0);
      }
      return __shfl_sync(0xFFFFFFFFu, c, 0);
    };
    for (;;) {
      const int cur_claim = claim();
      const int base = cur_claim >> 1, gsz = (cur_claim & 1) ? CTW_EPS_TAIL_SZ : 32;
      if (base >= n_cur) break;
      const int nv = min(gsz, n_cur - base);
      if (lane == 0) atomicAdd(&sm.eps_items, nv);
      int deg = 0;
      uint2 it = make_uint2(0u, 0u);
      if (lane < nv) {
        const int i = base + lane;
        it = i < sm.n_first ? sm.in0[i] : sm.in1[i - sm.n_first];
      }
      if (lane < nv) {
        // the range and the entry are independent loads: issue them together
        const CtwTok* eu = &L.T[it.x];
        const CtwStateRange r = ld_range(g.ranges, FSA ? (it.y & L.smask) : it.y);
#if CTW_LD256
        ulonglong2 v;
        unsigned long long gu;
        uint32_t st_;
        ld_tok(eu, v, gu, st_);
#else
        const ulonglong2 v = __ldcg(reinterpret_cast<const ulonglong2*>(eu));
        const unsigned long long gu = __ldcg(&eu->gpos);
#endif
        deg = (int)(r.emit_beg - r.eps_beg);
        if (deg > 0) {
          const double c = key2d(v.x);
          const bool valued = v.x != ~0ULL && !(L.prune && c > running_cut(sm, sm.eo_beam));
          uint32_t aux = CTW_DISC;
          if (valued) {
            const uint32_t tbu = (uint32_t)v.y, auxu = (uint32_t)(v.y >> 32);
            uint32_t pd = 1;
            if (tbu & CTW_EPS_BIT) {
              const uint32_t pred = auxu & CTW_PRED_MASK;
              pd = (auxu >> CTW_PRED_BITS) + (gu < __ldcg(&L.T[pred].gpos) ? 1u : 0u);
              pd = min(pd, 255u);
            }
            aux = (pd << CTW_PRED_BITS) | it.x;
          }
          sm.ep.cost[w][lane] = c;
          sm.ep.gu[w][lane] = gu;
          sm.ep.beg[w][lane] = r.eps_beg;
          sm.ep.aux[w][lane] = aux;
        }
      }
      int incl = deg;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += t;
      }
      sm.ep.off[w][lane] = incl - deg;
      const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
      if (lane == 0) atomicAdd(&sm.eps_arcs, total);
      {
        int dsc = (lane < nv && deg > 0 && sm.ep.aux[w][lane] == CTW_DISC) ? deg : 0;
        for (int o = 16; o; o >>= 1) dsc += __shfl_xor_sync(0xFFFFFFFFu, dsc, o);
        if (lane == 0) atomicAdd(&sm.eps_disc, dsc);
      }
      __syncwarp();
      for (int k = lane; k < total; k += 32) {
        int lo = 0, hi = nv - 1;  // last item with off <= k
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (sm.ep.off[w][mid] <= k) lo = mid;
          else hi = mid - 1;
        }
        const uint32_t o = (uint32_t)(k - sm.ep.off[w][lo]);
        const uint32_t a = sm.ep.beg[w][lo] + o;
        const CtwArc arc = ld_arc(g.arcs, a);
        uint32_t ikey = 0;  // the item's token key (phrase automaton state)
        if (FSA) {
          const int ii = base + lo;
          ikey = (ii < n_first ? in0[ii] : in1[ii - n_first]).y;
        }
        eps_arc<FSA>(sm, L, g, boost, w, lo, o, a, arc, ikey);
      }
      __syncwarp();
    }
#if CTW_IDLE_PROF
    const long long t_done = clock64();
#endif
    // the barrier ending the pass (also merges the ranks' running minima)
    const int vst = csync(sm);
#if CTW_IDLE_PROF
    if (lane == 0) atomicAdd(&sm.eps_idle, (unsigned long long)(clock64() - t_done));
#endif
    if (vst >= CTW_GROW_TABLE) return CTW_OK;  // caller handles the grow request
    if (tid < 32) {
      const int any = __any_sync(0xFFFFFFFFu, tid < R && cl.map_shared_rank(&sm, tid)->pc_big[q]);
      if (tid == 0) sm.any_big = any;
    }
    __syncthreads();
    // a quiet pass (only <= relax_eps changes) ends the closure; otherwise the
    // parked small improvements ride along in the next pass
    if (!sm.any_big) return CTW_OK;
  }
}

// ------------------------------------------------------------- records ----

// Walk a survivor's winner chain back to its emitting arc (or the seed),
// collecting output labels. Records store them oldest-first: [pending chain
// of the source] + emitting olabel + epsilon olabels in path order
// (_kernel.pyx:400-416).
struct WalkEnd {
  int32_t bp;
  int32_t anc;   // the source's nearest labelled record (CtwSrc::anc)
  int32_t pend;  // olabel code of the source's pending chain
  int n;         // labels found on the walk (excluding pend)
  int32_t last;  // the single label when n == 1
  bool ok;
};

// One hop back along a winner chain from the value v: 0 = seed (no arc),
// 1 = emitting arc `arc` from source `idx` (the chain ends), 2 = epsilon arc
// `arc` (v becomes the predecessor's value). On a graph whose epsilon arcs
// carry no output labels an epsilon hop needs no arc (CTW_NOARC): only the
// predecessor's entry is loaded.
#define CTW_NOARC 0xFFFFFFFFu
template <bool FAST>
__device__ __forceinline__ int hop_step(const LaneCtx& L, const GraphDev& g, const CtwSrc* src, ulonglong2& v,
                                        uint32_t& arc, uint32_t& idx) {
  if (FAST) {
    const uint32_t win = (uint32_t)(v.y >> 32);
    if (!(win & CTW_FEPS)) {
      idx = win >> L.ebits;
      arc = __ldcg(&src[idx].emit_beg) + (win & ((1u << L.ebits) - 1u));
      return 1;
    }
    v = __ldcg(&L.V[win & L.mask]);
    arc = L.eps_lab ? __ldg(&g.ranges[(uint32_t)v.y & L.smask].eps_beg) + ((win & ~CTW_FEPS) >> L.tlog2)
                    : CTW_NOARC;
    return 2;
  }
  const uint32_t tb = (uint32_t)v.y, aux = (uint32_t)(v.y >> 32);
  if (tb == CTW_SEED_TB) return 0;
  arc = tb & ~CTW_EPS_BIT;
  if (!(tb & CTW_EPS_BIT)) {
    idx = aux;
    return 1;
  }
  if (!L.eps_lab) arc = CTW_NOARC;
  v = __ldcg(reinterpret_cast<const ulonglong2*>(&L.T[aux & CTW_PRED_MASK]));
  return 2;
}

// v0 = the survivor's own (key, winner), already gathered.
template <bool FAST>
__device__ __forceinline__ WalkEnd walk(const LaneCtx& L, const GraphDev& g, ulonglong2 v0, const CtwSrc* src,
                                        const int32_t* pend, int hop_cap) {
  WalkEnd w{-1, -1, 0, 0, 0, true};
  ulonglong2 v = v0;
  for (int hop = 0; hop < hop_cap; ++hop) {
    uint32_t a = 0, idx = 0;
    const int k = hop_step<FAST>(L, g, src, v, a, idx);
    if (k == 0) return w;
    const int32_t ol = a == CTW_NOARC ? 0 : g.olabel[a];
    if (ol != 0) {
      ++w.n;
      w.last = ol;
    }
    if (k == 1) {
      w.bp = src[idx].bp;
      w.anc = src[idx].anc;
      w.pend = pend ? pend[idx] : 0;
      return w;
    }
  }
  w.ok = false;
  return w;
}

__device__ __forceinline__ int code_len(const int32_t* pool, int32_t code) {
  return code == 0 ? 0 : (code > 0 ? 1 : pool[-code - 1]);
}

// Olabel code of a record: 0 none, >0 one label, <0 pool segment
// -(offset+1) holding [n, l1..ln].
template <bool FAST>
__device__ int32_t record_code(Smem& sm, const LaneCtx& L, const GraphDev& g, const CtwSrc* src, ulonglong2 v0,
                               const WalkEnd& w) {
  const int np = code_len(L.pool, w.pend);
  const int n = np + w.n;
  if (n == 0) return 0;
  if (n == 1) return np ? w.pend : w.last;
  const int off = atomicAdd(&L.G->pool_used, n + 1);  // cluster-wide pool fill (rank 0)
  if (off + n + 1 > L.pool_cap) {
    atomicMax(&sm.status_l, CTW_GROW_POOL);
    return 0;
  }
  int32_t* seg = L.pool + off;
  seg[0] = n;
  if (np == 1) seg[1] = w.pend;
  else
    for (int i = 0; i < np; ++i) seg[1 + i] = L.pool[-w.pend - 1 + 1 + i];
  int pos = n;  // walk again, writing newest-first labels from the back
  ulonglong2 v = v0;
  for (int hop = 0; hop < 1 << 20; ++hop) {
    uint32_t a = 0, idx = 0;
    const int k = hop_step<FAST>(L, g, src, v, a, idx);
    if (k == 0) break;
    const int32_t ol = a == CTW_NOARC ? 0 : g.olabel[a];
    if (ol != 0) seg[pos--] = ol;
    if (k == 1) break;
  }
  return -(off + 1);
}

// ------------------------------------------------------------- prune ------

__device__ __forceinline__ int digit_of(unsigned long long key, uint32_t state, int d) {
  return d < 8 ? (int)((key >> (56 - 8 * d)) & 255) : (int)((state >> (24 - 8 * (d - 8))) & 255);
}

// Compare the top `depth` 8-bit digits of (key, state) with the prefix.
__device__ __forceinline__ int cmp_prefix(unsigned long long key, uint32_t state, int depth,
                                          unsigned long long ph, uint32_t pl) {
  if (depth <= 8) {
    if (depth == 0) return 0;
    const unsigned long long x = key >> (64 - 8 * depth);
    return x < ph ? -1 : (x > ph ? 1 : 0);
  }
  if (key != ph) return key < ph ? -1 : 1;
  const uint32_t x = state >> (32 - 8 * (depth - 8));
  return x < pl ? -1 : (x > pl ? 1 : 0);
}

// Exact top-k by (cost, state) among in-beam slots: MSD radix select over the
// 96-bit (sortable cost, state) key, 8 bits per pass, stopping as soon as the
// prefix bucket is taken whole. Every rank histograms its own slots into rank
// 0's digit histogram; rank 0 fixes the digit. Leaves (l_ph, l_pl, l_depth)
// in every rank.
__device__ void radix_select(Smem& sm, const LaneCtx& L, const ulonglong2* sv, const uint2* ib, int n_all,
                             unsigned long long cut_key, long long k) {
  cg::cluster_group cl = cg::this_cluster();
  const int tid = threadIdx.x;
  Smem* G = L.G;
  if (L.rank == 0) {
    if (tid == 0) {
      sm.sel_hi = 0;
      sm.sel_lo = 0;
      sm.sel_depth = 0;
      sm.rneed = (int)k;
      sm.sel_done = 0;
    }
    for (int i = tid; i < 256; i += CTW_BS) sm.cs.rhist[0][i] = 0;
  }
  cl.sync();
  for (int d = 0; d < 12; ++d) {
    if (tid == 0) {
      sm.l_ph = *((volatile unsigned long long*)&G->sel_hi);
      sm.l_pl = *((volatile uint32_t*)&G->sel_lo);
    }
    for (int i = tid; i < 256; i += CTW_BS) sm.cs.hist[i] = 0;
    __syncthreads();
    const unsigned long long ph = sm.l_ph;
    const uint32_t pl = sm.l_pl;
    for (int i = L.sw0 + tid; i < n_all; i += L.swstride) {
      const unsigned long long key = sv[i].x;
      if (key > cut_key) continue;
      const uint32_t st = ib[i].y;
      if (cmp_prefix(key, st, d, ph, pl) != 0) continue;
      atomicAdd(&sm.cs.hist[digit_of(key, st, d)], 1u);
    }
    __syncthreads();
    for (int i = tid; i < 256; i += CTW_BS)
      if (sm.cs.hist[i]) atomicAdd(&G->cs.rhist[d & 1][i], sm.cs.hist[i]);
    if (L.rank == 0)
      for (int i = tid; i < 256; i += CTW_BS) sm.cs.rhist[(d + 1) & 1][i] = 0;
    cl.sync();
    if (L.rank == 0 && tid < 32) {
      // warp 0 of rank 0: locate the bucket holding the need-th smallest
      uint32_t c[8];
      uint32_t sum = 0;
      for (int j = 0; j < 8; ++j) {
        c[j] = sm.cs.rhist[d & 1][tid * 8 + j];
        sum += c[j];
      }
      uint32_t incl = sum;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (tid >= o) incl += t;
      }
      const uint32_t excl = incl - sum;
      const uint32_t need = (uint32_t)sm.rneed;
      if (excl < need && need <= incl) {
        uint32_t run = excl;
        int b = 0;
        for (int j = 0; j < 8; ++j) {
          if (run + c[j] >= need) {
            b = tid * 8 + j;
            break;
          }
          run += c[j];
        }
        const uint32_t rem = need - run;
        if (d < 8) sm.sel_hi = (sm.sel_hi << 8) | (unsigned long long)b;
        else sm.sel_lo = (sm.sel_lo << 8) | (uint32_t)b;
        sm.sel_depth = d + 1;
        sm.rneed = (int)rem;
        if (sm.cs.rhist[d & 1][b] == rem) sm.sel_done = 1;
      }
    }
    cl.sync();
    if (tid == 0) sm.l_depth = *((volatile int*)&G->sel_done);
    __syncthreads();
    if (sm.l_depth) break;
  }
  if (tid == 0) {
    sm.l_ph = *((volatile unsigned long long*)&G->sel_hi);
    sm.l_pl = *((volatile uint32_t*)&G->sel_lo);
    sm.l_depth = *((volatile int*)&G->sel_depth);
  }
  __syncthreads();
}

// --------------------------------------------------------- frame kernel ---

struct ChunkArgs {
  const void* loglik;       // [*, width] rows, f32 or f64, device
  const long long* ll_off;  // per batch entry: element offset of frame 0
  const int* nframes;       // per batch entry
  const int* lane_ids;      // per batch entry
  int width;
  int is_f64;
  int ebits;  // fast mode: bits of the emitting-arc offset in a winner word
  int eps_lab; // some epsilon arc carries an output label
  CtwDecodeCfg cfg;
};

__device__ __forceinline__ LaneCtx lane_ctx(const CtwLane& lane, int rank, int nranks, Smem* G) {
  LaneCtx L;
  L.T = lane.table;
  L.tcap = 1u << lane.tlog2;
  L.mask = L.tcap - 1;
  L.shift = 32 - lane.tlog2;
  L.seg = CTW_LOAD(L.tcap);
  L.slots = lane.slots;
  L.front = lane.front;
  L.G = G;
  L.slot_ctr = nullptr;
  L.rank = rank;
  L.nranks = nranks;
  L.sw0 = rank * CTW_BS;
  L.swstride = nranks * CTW_BS;
  L.pool = lane.pool;
  L.pool_cap = lane.pcap;
  L.prune = lane.prune_ok != 0;
  L.tie_ctr = nullptr;
  L.fnext = lane.fsa_next;
  L.fcost = lane.fsa_cost;
  L.fwidth = lane.fsa_width;
  L.sbits = lane.sbits;
  L.smask = lane.smask;
  L.V = reinterpret_cast<ulonglong2*>(lane.table);
  L.tlog2 = lane.tlog2;
  L.ebits = 0;
  L.eps_lab = true;
  return L;
}

// Epsilon-stage pass cap: a convergent closure never needs more label-
// correcting passes than slots; beyond that the closure diverges (negative
// cycle) and the reference's Gauss-Seidel loop hits max_ne_iters too.
__device__ __forceinline__ long long divergence_cap(long long max_ne_iters, uint32_t tcap) {
  return max(max_ne_iters, (long long)CTW_LOAD(tcap)) + 2;
}

__device__ __forceinline__ int cost_bin(unsigned long long key, double min_cost, double bin_scale) {
  const int b = (int)__dmul_rn(__dsub_rn(key2d(key), min_cost), bin_scale);
  return min(max(b, 0), CTW_NB - 1);
}

#ifndef CTW_UNR
#define CTW_UNR 1  // table loads in flight per thread in slot sweeps (round 2: 1 beats 2 by 2.7 % in the fast mode, neutral in the exact mode -- fewer live registers; 4 spilled in round 1)
#endif

// One sweep over this rank's slots: gathers every slot's final (key, tb|aux)
// into sv (this rank's part of the compact value array; coalesced for the
// later sweeps, CTW_UNR table loads in flight per thread), and computes the
// Gauss-Seidel pass count of the closure (= 1 + last pass that changed a
// slot, i.e. max pd over epsilon-won slots; > max_ne_iters ->
// CTW_ERR_EPS_ITERS), the in-beam count and (hist) the cost histogram over
// [min, min + beam] for the max-active select; merges them into the frame
// counters and meets the other ranks at a barrier.
// With `hist` (decoding) the in-beam slots are compacted: sv[j] = value and
// ib[j] = (table index, state) for j < in-beam count (cluster-wide list, warp-
// aggregated appends); the select and record stages then sweep only those.
// Without it (seeding) sv[i] holds slot i's value for every slot.
template <bool FAST>
__device__ int count_pass(Smem& sm, const LaneCtx& L, FrameCtr* fc, ulonglong2* sv, uint2* ib, int n_all,
                          long long max_ne_iters, unsigned long long cut_key, double min_cost, double bin_scale,
                          bool hist) {
  const int tid = threadIdx.x;
  if (hist)
    for (int i = tid; i < CTW_NB; i += CTW_BS) sm.cs.lbhist[i] = 0;
  if (tid == 0) {
    sm.cnt_l = 0;
    sm.mpd_l = 0;
  }
  __syncthreads();
  int c = 0, mpd = 0;
  for (int i0 = L.sw0 + tid; i0 < n_all; i0 += CTW_UNR * L.swstride) {
    uint2 h[CTW_UNR];
    ulonglong2 v[CTW_UNR];
#pragma unroll
    for (int u = 0; u < CTW_UNR; ++u) {
      const int i = i0 + u * L.swstride;
      h[u] = i < n_all ? L.slots[i] : make_uint2(0u, 0u);
    }
#pragma unroll
    for (int u = 0; u < CTW_UNR; ++u) {
      const int i = i0 + u * L.swstride;
      if (i < n_all) v[u] = __ldcg(tval<FAST>(L, h[u].x));
    }
#pragma unroll
    for (int u = 0; u < CTW_UNR; ++u) {
      const int i = i0 + u * L.swstride;
      if (i >= n_all) break;
      if (!hist) sv[i] = v[u];
      if (v[u].x <= cut_key) {
        ++c;
        if (hist) {
          atomicAdd(&sm.cs.lbhist[cost_bin(v[u].x, min_cost, bin_scale)], 1u);
          const int j = agg_alloc(&fc->nib, nullptr);
          sv[j] = v[u];
          ib[j] = h[u];
        }
      }
      if (!FAST && ((uint32_t)v[u].y & CTW_EPS_BIT)) mpd = max(mpd, (int)((uint32_t)(v[u].y >> 32) >> CTW_PRED_BITS));
    }
  }
  for (int o = 16; o; o >>= 1) {
    c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
    mpd = max(mpd, __shfl_xor_sync(0xFFFFFFFFu, mpd, o));
  }
  if ((tid & 31) == 0) {
    atomicAdd(&sm.cnt_l, c);
    atomicMax(&sm.mpd_l, mpd);
  }
  __syncthreads();
  if (hist)
    for (int i = tid; i < CTW_NB; i += CTW_BS) {
      const uint32_t n = sm.cs.lbhist[i];
      if (n) atomicAdd(&fc->bhist[i], n);
    }
  if (tid == 0) {
    atomicAdd(&fc->cnt, sm.cnt_l);
    atomicMax(&fc->max_pd, sm.mpd_l);
  }
  csync(sm);
  if (tid == 0) {
    sm.cnt_all = *((volatile int*)&fc->cnt);
    sm.mpd_all = *((volatile int*)&fc->max_pd);
  }
  __syncthreads();
  return (1 + (long long)sm.mpd_all > max_ne_iters) ? CTW_ERR_EPS_ITERS : CTW_OK;
}

// Reset this rank's share of the frame's table entries; slot loads batched
// ahead of the stores.
template <bool FAST>
__device__ __forceinline__ void reset_slots(const LaneCtx& L, int n_all) {
  for (int i0 = L.sw0 + threadIdx.x; i0 < n_all; i0 += CTW_UNR * L.swstride) {
    uint32_t h[CTW_UNR];
#pragma unroll
    for (int u = 0; u < CTW_UNR; ++u) {
      const int i = i0 + u * L.swstride;
      h[u] = i < n_all ? L.slots[i].x : CTW_EMPTY;
    }
#pragma unroll
    for (int u = 0; u < CTW_UNR; ++u)
      if (h[u] != CTW_EMPTY) {
        if (FAST) ftok_clear(&L.V[h[u]]);
        else tok_clear(&L.T[h[u]]);
      }
  }
}

// Exact max-active threshold by (cost, state) (decoder.py:361-374,
// _kernel.pyx:385-390): rank 0 locates the boundary bin in the merged
// histogram; every rank hands its boundary-bin members to rank 0, which sorts
// them exactly in shared memory (bitonic). Falls back to the cluster-wide
// digit-wise radix select when the boundary bin overflows CTW_BBUF. Leaves
// the threshold in every rank's l_* fields.
__device__ void select_threshold(Smem& sm, const LaneCtx& L, FrameCtr* fc, const ulonglong2* sv, const uint2* ib,
                                 int n_all,
                                 unsigned long long cut_key, double min_cost, double bin_scale, long long k) {
  cg::cluster_group cl = cg::this_cluster();
  const int tid = threadIdx.x;
  Smem* G = L.G;
  if (L.rank == 0 && tid < 32) {
    // warp 0 of rank 0: lane t owns bins [32t, 32t + 32); one warp scan of
    // the lane sums finds the lane holding the k-th smallest cost, which
    // re-reads its bins (no per-thread array: it would spill)
    const uint32_t* bh = fc->bhist + tid * (CTW_NB / 32);
    uint32_t sum = 0;
#pragma unroll 8
    for (int j = 0; j < CTW_NB / 32; ++j) sum += bh[(j + tid) & (CTW_NB / 32 - 1)];  // rotated: fewer bank conflicts
    uint32_t incl = sum;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (tid >= o) incl += t;
    }
    const uint32_t excl = incl - sum;
    const uint32_t need = (uint32_t)k;
    if (excl < need && need <= incl) {
      uint32_t run = excl;
      for (int j = 0; j < CTW_NB / 32; ++j) {
        const uint32_t c = bh[j];
        if (run + c >= need) {
          sm.sel_bin = tid * (CTW_NB / 32) + j;
          sm.sel_need = (int)(need - run);
          sm.sel_bcount = (int)c;
          break;
        }
        run += c;
      }
    }
    if (tid == 0) {
      sm.thr_key = ~0ULL;
      sm.thr_state = 0xFFFFFFFFu;
    }
  }
  cl.sync();
  if (tid == 0) {
    sm.l_bin = *((volatile int*)&G->sel_bin);
    sm.l_need = *((volatile int*)&G->sel_need);
    sm.l_bcount = *((volatile int*)&G->sel_bcount);
    sm.l_radix = 0;
    sm.l_tk = ~0ULL;
    sm.l_ts = 0xFFFFFFFFu;
  }
  __syncthreads();
  const int bsel = sm.l_bin, need = sm.l_need, bcount = sm.l_bcount;
  // (rank 0 rewrites the select fields only in a later frame, after several
  // barriers: every rank has copied them by then)
  if (bcount == need) return;  // the whole boundary bin survives
  if (bcount > CTW_BBUF) {
    if (tid == 0) sm.l_radix = 1;
    radix_select(sm, L, sv, ib, n_all, cut_key, k);
    return;
  }
  for (int i = L.sw0 + tid; i < n_all; i += L.swstride) {
    const unsigned long long key = sv[i].x;
    if (key <= cut_key && cost_bin(key, min_cost, bin_scale) == bsel) {
      const int p = atomicAdd(&fc->nbb, 1);
      G->bbuf[p] = make_ulonglong2(key, ib[i].y);
    }
  }
  cl.sync();
  if (L.rank == 0) {
    int n2 = 1;
    while (n2 < bcount) n2 <<= 1;
    for (int i = bcount + tid; i < n2; i += CTW_BS) sm.bbuf[i] = make_ulonglong2(~0ULL, ~0ULL);
    __syncthreads();
    for (int kk = 2; kk <= n2; kk <<= 1) {
      for (int j = kk >> 1; j > 0; j >>= 1) {
        for (int i = tid; i < n2; i += CTW_BS) {
          const int ixj = i ^ j;
          if (ixj > i) {
            const ulonglong2 x = sm.bbuf[i], y = sm.bbuf[ixj];
            const bool gt = x.x > y.x || (x.x == y.x && x.y > y.y);
            if (gt == ((i & kk) == 0)) {
              sm.bbuf[i] = y;
              sm.bbuf[ixj] = x;
            }
          }
        }
        __syncthreads();
      }
    }
    if (tid == 0) {
      sm.thr_key = sm.bbuf[need - 1].x;
      sm.thr_state = (uint32_t)sm.bbuf[need - 1].y;
    }
  }
  cl.sync();
  if (tid == 0) {
    sm.l_tk = *((volatile unsigned long long*)&G->thr_key);
    sm.l_ts = *((volatile uint32_t*)&G->thr_state);
  }
  __syncthreads();
}

// Relax one emitting arc: ((c + (-scale * ll)) + w) (+ boost), then
// find-or-insert the destination and install the candidate if it wins
// (_kernel.pyx:243-287). `off` = the arc's offset in its source's emitting
// range (fast mode's winner word).
template <bool FSA, bool FAST>
__device__ __forceinline__ void emit_arc_loaded(Smem& sm, const LaneCtx& L, const GraphDev& g, const ChunkArgs& a,
                                                const double* nll_s, bool smem_ll, long long row0, double neg_scale,
                                                const double* boost, uint32_t arc_i, double cost, uint32_t src_idx,
                                                uint32_t src_key, const CtwArc& arc, const CtwSrc* src, uint32_t off) {
  const double INF = __longlong_as_double(0x7FF0000000000000LL);
  double ac;
  if (smem_ll) ac = nll_s[arc.ilabel - 1];
  else {
    const long long idx = row0 + arc.ilabel - 1;
    const double x = a.is_f64 ? ((const double*)a.loglik)[idx] : (double)((const float*)a.loglik)[idx];
    ac = __dmul_rn(neg_scale, x);
  }
  double nc = __dadd_rn(__dadd_rn(cost, ac), arc.weight);
  uint32_t dkey = (uint32_t)arc.nextstate;
  if (FSA) dkey = arc_dest<FSA>(L, boost, src_key, g.olabel[arc_i], (uint32_t)arc.nextstate, nc);
  else if (boost) {
    const int32_t ol = g.olabel[arc_i];
    if (ol != 0) nc = __dadd_rn(nc, boost[ol]);
  }
  if (!(nc < INF)) return;
  if (FAST) {
    // never inserted above the running cutoff (cannot make the final beam)
    if (nc > running_cut(sm, a.cfg.beam)) return;
    bool is_new = false;
    ulonglong2 seen;
    const uint32_t d = ftok_locate(L, dkey, &seen, is_new);
    if (d == CTW_EMPTY) {
      atomicMax(&sm.status_l, CTW_GROW_TABLE);
      return;
    }
    if (is_new) slot_append(sm, L, d, dkey);
    unsigned long long oldk;
    const unsigned long long nk = d2key(nc);
    if (ftok_relax(L, g, src, &L.V[d], nk, fwin_emit(src_idx, off, L.ebits), arc_i, seen, &oldk)) track_min(sm, nk);
    return;
  }
  bool is_new = false;
  ulonglong2 seen;
  const uint32_t d = tok_locate(L, dkey, &seen, is_new);
  if (d == CTW_EMPTY) {
    atomicMax(&sm.status_l, CTW_GROW_TABLE);
    return;
  }
  if (is_new) slot_append(sm, L, d, dkey);
  CtwTok* ed = &L.T[d];
  // Gauss-Seidel slot position of an emitting-reached state = its
  // first-arrival arc (_kernel.pyx:256-272)
  gpos_min(ed, (unsigned long long)arc_i);
  if (L.prune && nc > running_cut(sm, a.cfg.beam)) return;  // cannot make the final beam
  unsigned long long oldk;
  const unsigned long long nk = d2key(nc);
  if (tok_relax_from(L, ed, nk, arc_i, src_idx, 0ULL, seen, &oldk)) track_min(sm, nk);
}

template <bool FSA, bool FAST>
__device__ __forceinline__ void emit_arc(Smem& sm, const LaneCtx& L, const GraphDev& g, const ChunkArgs& a,
                                         const double* nll_s, bool smem_ll, long long row0, double neg_scale,
                                         const double* boost, uint32_t arc_i, double cost, uint32_t src_idx,
                                         uint32_t src_key, const CtwSrc* src, uint32_t off) {
  const CtwArc arc = ld_arc(g.arcs, arc_i);
  emit_arc_loaded<FSA, FAST>(sm, L, g, a, nll_s, smem_ll, row0, neg_scale, boost, arc_i, cost, src_idx, src_key, arc,
                             src, off);
}

// Fast mode: relax one epsilon arc a (offset o) of the frontier item lo of
// warp w; queue the destination for the next pass when it improved.
template <bool FSA>
__device__ __forceinline__ void feps_arc(Smem& sm, const LaneCtx& L, const GraphDev& g, const double* boost, int w,
                                         int lo, uint32_t o, uint32_t a, const CtwArc& arc, double beam, uint2* out,
                                         int* ctr, uint32_t fcap) {
  const double INF = __longlong_as_double(0x7FF0000000000000LL);
  double nc = __dadd_rn(sm.ep.cost[w][lo], arc.weight);
  uint32_t dkey = (uint32_t)arc.nextstate;
  if (FSA) dkey = arc_dest<FSA>(L, boost, (uint32_t)sm.ep.gu[w][lo], g.olabel[a], dkey, nc);
  else if (boost) {
    const int32_t ol = g.olabel[a];
    if (ol != 0) nc = __dadd_rn(nc, boost[ol]);
  }
  if (!(nc < INF)) return;
  if (nc > running_cut(sm, beam)) return;
  bool is_new = false;
  ulonglong2 seen;
  const uint32_t d = ftok_locate(L, dkey, &seen, is_new);
  if (d == CTW_EMPTY) {
    atomicMax(&sm.status_l, CTW_GROW_TABLE);
    return;
  }
  if (is_new) slot_append(sm, L, d, dkey);
  unsigned long long oldk;
  const unsigned long long nk = d2key(nc);
  const uint32_t win = CTW_FEPS | (o << L.tlog2) | sm.ep.aux[w][lo];
  if (!ftok_relax(L, g, nullptr, &L.V[d], nk, win, a, seen, &oldk)) return;
  track_min(sm, nk);
  const int p = agg_alloc(ctr, nullptr);
  if ((uint32_t)p < fcap) out[p] = make_uint2(d, dkey);
  else atomicMax(&sm.status_l, CTW_GROW_TABLE);
}

// Fast mode epsilon closure: label-correcting passes over the states that
// improved in the previous pass (pass 1: every slot of the frame), skipping
// predecessors and candidates above the running cutoff; ends when a pass
// improves nothing. Two frontier sets of 2 x seg items (pass parity); work is
// handed out cluster-wide in 32-item chunks. Returns CTW_OK or
// CTW_ERR_EPS_ITERS (divergence).
template <bool FSA>
__device__ CTW_EPS_INLINE int eps_fast(Smem& sm, const LaneCtx& L, const GraphDev& g, const double* boost,
                                       double beam, long long pass_cap) {
  cg::cluster_group cl = cg::this_cluster();
  const int tid = threadIdx.x;
  const int R = L.nranks, rank = L.rank;
  Smem* G = L.G;
  const uint32_t fcap = 2 * L.seg;
  const int lane = tid & 31, w = tid >> 5;
  for (long long pass = 1;; ++pass) {
    const int q = (int)(pass & 1);
    uint2* out = L.front + (size_t)((pass - 1) & 1) * fcap;
    int* ctr_out = G->pcnt[pass % 3];
    if (tid == 0) {
      if (pass == 1) {
        int tot = 0;
        for (int k = 0; k < R; ++k) tot += cl.map_shared_rank(&sm, k)->snap_slots;  // once per frame
        sm.in0 = L.slots;
        sm.n_cur = min(tot, (int)L.seg);
      } else {
        sm.in0 = L.front + (size_t)((pass - 2) & 1) * fcap;
        sm.n_cur = min(*((volatile const int*)&G->pcnt[(pass - 1) % 3][0]), (int)fcap);
      }
      if (rank == 0) {
        sm.pw[q ^ 1] = 0;                // the next pass's chunk counter
        sm.pcnt[(pass + 1) % 3][0] = 0;  // written in pass + 1; last read at the start of pass - 1
      }
      sm.passes = (int)pass;
    }
    __syncthreads();
    const int n_cur = sm.n_cur;
    if (n_cur == 0) return CTW_OK;  // (the same count in every rank)
    if (pass > pass_cap) return CTW_ERR_EPS_ITERS;
    const uint2* in = sm.in0;
    for (;;) {
      int base = 0;
      if (lane == 0) base = atomicAdd(&G->pw[q], 32);
      base = __shfl_sync(0xFFFFFFFFu, base, 0);
      if (base >= n_cur) break;
      const int nv = min(32, n_cur - base);
      if (lane == 0) atomicAdd(&sm.eps_items, nv);
      int deg = 0;
      if (lane < nv) {
        const uint2 it = in[base + lane];
        // the range and the entry are independent loads: issue them together
        const CtwStateRange r = ld_range(g.ranges, FSA ? (it.y & L.smask) : it.y);
        const ulonglong2 v = __ldcg(&L.V[it.x]);
        const double c = key2d(v.x);
        if (!(c > running_cut(sm, beam))) deg = (int)(r.emit_beg - r.eps_beg);
        sm.ep.cost[w][lane] = c;
        sm.ep.beg[w][lane] = r.eps_beg;
        sm.ep.aux[w][lane] = it.x;
        sm.ep.gu[w][lane] = it.y;
      }
      int incl = deg;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += t;
      }
      sm.ep.off[w][lane] = incl - deg;
      const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
      if (lane == 0) atomicAdd(&sm.eps_arcs, total);
      __syncwarp();
      for (int k = lane; k < total; k += 32) {
        int lo = 0, hi = nv - 1;  // last item with off <= k
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (sm.ep.off[w][mid] <= k) lo = mid;
          else hi = mid - 1;
        }
        const uint32_t o = (uint32_t)(k - sm.ep.off[w][lo]);
        const uint32_t a = sm.ep.beg[w][lo] + o;
        const CtwArc arc = ld_arc(g.arcs, a);
        feps_arc<FSA>(sm, L, g, boost, w, lo, o, a, arc, beam, out, ctr_out, fcap);
      }
      __syncwarp();
    }
    // the barrier ending the pass (also merges the ranks' running minima)
    const int vst = csync(sm);
    if (vst >= CTW_GROW_TABLE) return CTW_OK;  // caller handles the grow request
  }
}

// FSA: some lane of the launch has a phrase automaton (token keys carry its
// state); the plain instantiation keeps the hot path free of it. FAST: the
// words-exact search mode (see "fast search mode" above).
template <bool FSA, bool FAST>
__global__ void __launch_bounds__(CTW_BS, CTW_MINB) k_decode_chunk(CtwLane* lanes, const __grid_constant__ GraphDev g,
                                                                const __grid_constant__ ChunkArgs a, CtwLaneOut* out) {
  extern __shared__ double nll_s[];
  __shared__ Smem sm;
  cg::cluster_group cl = cg::this_cluster();
  const int tid = threadIdx.x;
  const int R = (int)cl.num_blocks(), rank = (int)cl.block_rank();
  const int b = blockIdx.x / R;
  Smem* G = cl.map_shared_rank(&sm, 0);
  CtwLane& lane = lanes[a.lane_ids[b]];
  LaneCtx L = lane_ctx(lane, rank, R, G);
  L.tie_ctr = &sm.eps_ties;
  L.ebits = (uint32_t)a.ebits;
  L.eps_lab = a.eps_lab != 0;
  const int F = a.nframes[b];
  const double* boost = lane.boost;
  const bool smem_ll = a.width <= CTW_MAX_SMEM_WIDTH;
  const double neg_scale = -a.cfg.acoustic_scale;
  const long long pass_cap = divergence_cap(a.cfg.max_ne_iters, L.tcap);
  BigSrc* bigl = reinterpret_cast<BigSrc*>(L.front + (size_t)3 * L.seg);  // set 3: free until pass 2
  const int big_cap = (int)min((size_t)CTW_NBIG, ((size_t)L.seg * sizeof(uint2)) / sizeof(BigSrc));

  int n_src = lane.n_src;
  int cur_buf = lane.src_buf;
  const int w0 = (cur_buf + 1) % 3, w1 = (cur_buf + 2) % 3;
  const int committed = cur_buf;
  int pend_valid = lane.pend_valid;
  int status = CTW_OK;
  // stage counters: rank-local, tid 0 only, kept in shared memory (a
  // register array here would be live in every thread of the frame loop)
  long long* prof = reinterpret_cast<long long*>(sm.mydiag);
  if (tid == 0) {
    for (int k = 0; k < CTW_NPROF; ++k) prof[k] = 0;
    sm.src_total = 0;
    sm.rec_need = 0;
    sm.n_slots_max = 0;
    sm.err_frame = -1;
    sm.n_rec = lane.n_rec;
    sm.eps_idle = 0;
    sm.status_l = CTW_OK;
    sm.epoch = 0;
    sm.st_pub[0] = sm.st_pub[1] = 0;
    sm.st_all = 0;
    sm.min_pub[0] = sm.min_pub[1] = ~0ULL;
    if (rank == 0) {
      sm.pool_used = lane.pool_used;
      sm.pw[0] = sm.pw[1] = 0;
      for (int j = 0; j < 3; ++j) sm.pcnt[j][0] = sm.pcnt[j][1] = 0;
    }
  }
  if (rank == 0) {
    int* z = reinterpret_cast<int*>(&sm.fc[0]);
    for (int i = tid; i < (int)(2 * sizeof(FrameCtr) / sizeof(int)); i += CTW_BS) z[i] = 0;
  }
  cl.sync();

  for (int f = 0; f < F; ++f) {
    if (tid == 0) sm.tclk = clock64();
    FrameCtr* fc = &G->fc[f & 1];
    L.slot_ctr = &fc->nslot;
    const CtwSrc* src = lane.src[cur_buf];
    const int32_t* pend = pend_valid ? lane.pend : nullptr;
    const int nxt_buf = (f & 1) ? w1 : w0;
    CtwSrc* nsrc = lane.src[nxt_buf];
    if (tid == 0) {
      sm.n_slots = 0;
      sm.min_key = ~0ULL;
      sm.eps_items = 0;
      sm.eps_arcs = 0;
      sm.eps_ties = 0;
      sm.eps_disc = 0;
      sm.passes = 0;
      sm.arcs_f = 0;
    }
    // frame row -> -scale * ll (the reference's (-acoustic_scale * ll) term)
    const long long row0 = a.ll_off[b] + (long long)f * a.width;
    if (smem_ll) {
      for (int v = tid; v < a.width; v += CTW_BS) {
        const double x = a.is_f64 ? ((const double*)a.loglik)[row0 + v] : (double)((const float*)a.loglik)[row0 + v];
        nll_s[v] = __dmul_rn(neg_scale, x);
      }
    }
    csync(sm);  // (A) the previous frame (sources, table reset) is complete in every rank
    if (rank == 0) {
      // the other parity's counters: last read before this barrier, next used after the next frame's
      FrameCtr* nf = &sm.fc[(f + 1) & 1];
      int* z = reinterpret_cast<int*>(nf);
      for (int i = tid; i < (int)(sizeof(FrameCtr) / sizeof(int)); i += CTW_BS) z[i] = 0;
      if (tid == 0) {
        sm.pw[0] = sm.pw[1] = 0;
        for (int j = 0; j < 3; ++j) sm.pcnt[j][0] = sm.pcnt[j][1] = 0;
      }
    }
    if (tid == 0) sm.src_total += n_src;

    // ---- emitting expansion, load-balanced over out-degree ----
    const int lane_ = tid & 31, w = tid >> 5;
    // a claim is (base << 1) | (size == 8): 32 sources, 8 in the guided tail
    auto claim_e = [&]() -> int {
      int c = 0;
      if (lane_ == 0) {
        const bool small = n_src - *((volatile int*)&fc->work_e) < 32 * CTW_WARPS * R;
        c = (atomicAdd(&fc->work_e, small ? CTW_EMIT_TAIL_SZ : 32) << 1) | (small ? 1 : 0);
      }
      return __shfl_sync(0xFFFFFFFFu, c, 0);
    };
    for (;;) {
      // warps grab 32 sources at a time and spread their emitting arcs over
      // the lanes (warp scan of out-degrees); sources with more than
      // CTW_BIG arcs go to the arc-parallel list instead
      const int cur_claim = claim_e();
      const int base = cur_claim >> 1, gsz = (cur_claim & 1) ? CTW_EMIT_TAIL_SZ : 32;
      if (base >= n_src) break;
      const int nv = min(gsz, n_src - base);
      int deg = 0;
      CtwSrc t;
#if CTW_SRC256
      if (lane_ < nv) {
        unsigned long long w0, w1, w2, w3;
        asm volatile("ld.global.v4.u64 {%0, %1, %2, %3}, [%4];"
                     : "=l"(w0), "=l"(w1), "=l"(w2), "=l"(w3) : "l"(src + base + lane_));
        t.state = (int32_t)(uint32_t)w0;
        t.bp = (int32_t)(uint32_t)(w0 >> 32);
        t.cost = __longlong_as_double((long long)w1);
        t.emit_beg = (uint32_t)w2;
        t.emit_end = (uint32_t)(w2 >> 32);
        (void)w3;
      }
#else
      if (lane_ < nv) t = src[base + lane_];
#endif
      if (lane_ < nv) {
        const CtwStateRange r{0u, t.emit_beg, t.emit_end, 0u};  // cached with the token
        deg = (int)(r.emit_end - r.emit_beg);
        if (deg > CTW_BIG) {
          const int j = atomicAdd(&fc->nbig, 1);
          if (j < big_cap) {
            BigSrc bs;
            bs.idx = base + lane_;
            bs.beg = r.emit_beg;
            bs.deg = deg;
            bs.pad = 0;
            bs.cost = t.cost;
            bigl[j] = bs;
            deg = 0;
          }
        }
        sm.em.beg[w][lane_] = r.emit_beg;
        sm.em.cost[w][lane_] = t.cost;
      }
      int incl = deg;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane_ >= o) incl += t;
      }
      sm.em.off[w][lane_] = incl - deg;
      const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
      if (lane_ == 0) atomicAdd(&sm.arcs_f, total);
      __syncwarp();
#if CTW_EMPF
      // software pipeline over the rounds of 32 arcs: the next round's arc
      // load is in flight while this round's destination is located and
      // relaxed
      auto src_of = [&](int k) -> int {  // last source with off <= k
        int lo = 0, hi = nv - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (sm.em.off[w][mid] <= k) lo = mid;
          else hi = mid - 1;
        }
        return lo;
      };
      int lo = 0;
      uint32_t ai = 0;
      CtwArc arc{};
      if (lane_ < total) {
        lo = src_of(lane_);
        ai = sm.em.beg[w][lo] + (uint32_t)(lane_ - sm.em.off[w][lo]);
        arc = ld_arc(g.arcs, ai);
      }
      for (int k = lane_; k < total; k += 32) {
        const int kn = k + 32;
        int lon = 0;
        uint32_t ain = 0;
        CtwArc arcn{};
        if (kn < total) {
          lon = src_of(kn);
          ain = sm.em.beg[w][lon] + (uint32_t)(kn - sm.em.off[w][lon]);
          arcn = ld_arc(g.arcs, ain);
        }
        emit_arc_loaded<FSA, FAST>(sm, L, g, a, nll_s, smem_ll, row0, neg_scale, boost, ai, sm.em.cost[w][lo],
                                   (uint32_t)(base + lo), FSA ? (uint32_t)src[base + lo].state : 0u, arc, src,
                                   ai - sm.em.beg[w][lo]);
        lo = lon;
        ai = ain;
        arc = arcn;
      }
#else
      for (int k = lane_; k < total; k += 32) {
        int lo = 0, hi = nv - 1;  // last source with off <= k
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (sm.em.off[w][mid] <= k) lo = mid;
          else hi = mid - 1;
        }
        emit_arc<FSA, FAST>(sm, L, g, a, nll_s, smem_ll, row0, neg_scale, boost,
                            sm.em.beg[w][lo] + (uint32_t)(k - sm.em.off[w][lo]), sm.em.cost[w][lo],
                            (uint32_t)(base + lo), FSA ? (uint32_t)src[base + lo].state : 0u, src,
                            (uint32_t)(k - sm.em.off[w][lo]));
      }
#endif
      __syncwarp();
    }
    __syncthreads();
    if (tid == 0) sm.snap_slots = sm.n_slots;
    csync(sm);  // (B)
    if (tid == 0) sm.nbig = min(*((volatile int*)&fc->nbig), big_cap);
    __syncthreads();
    if (sm.nbig > 0 && sm.st_all < CTW_GROW_TABLE) {
      // arc-parallel expansion of the high out-degree sources: 32-arc chunks
      // over the degree prefix of the list
      const int nb = sm.nbig;
      for (int j0 = 0; j0 < nb; j0 += CTW_BS) {
        const int j = j0 + tid;
        int d = 0;
        if (j < nb) {
          const BigSrc bs = bigl[j];
          d = bs.deg;
        }
        const int carry = j0 == 0 ? 0 : sm.bg.pref[j0];
        int ex, tt;
        Smem::Scan(sm.scan).ExclusiveSum(d, ex, tt);
        if (j < nb) sm.bg.pref[j] = carry + ex;
        __syncthreads();
        if (tid == 0) sm.bg.pref[min(j0 + CTW_BS, nb)] = carry + tt;
        __syncthreads();
      }
      const int total = sm.bg.pref[nb];
      if (rank == 0 && tid == 0) sm.arcs_f += total;
      for (;;) {
        int base = 0;
        if (lane_ == 0) base = atomicAdd(&fc->work_b, 32);
        base = __shfl_sync(0xFFFFFFFFu, base, 0);
        if (base >= total) break;
        const int k = base + lane_;
        if (k < total) {
          int lo = 0, hi = nb - 1;  // last listed source with pref <= k
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (sm.bg.pref[mid] <= k) lo = mid;
            else hi = mid - 1;
          }
          const BigSrc bs = bigl[lo];  // (the listed source: a small, hot array)
          emit_arc<FSA, FAST>(sm, L, g, a, nll_s, smem_ll, row0, neg_scale, boost,
                              bs.beg + (uint32_t)(k - sm.bg.pref[lo]), bs.cost, (uint32_t)bs.idx,
                              FSA ? (uint32_t)src[bs.idx].state : 0u, src, (uint32_t)(k - sm.bg.pref[lo]));
        }
      }
      __syncthreads();
      if (tid == 0) sm.snap_slots = sm.n_slots;
      csync(sm);  // (C)
    }

    if (rank == 0 && tid == 0) {
      const long long t = clock64();
      prof[0] += t - sm.tclk;
      sm.tclk = t;
    }
    // ---- epsilon closure ----
    int st = CTW_OK;
    if (sm.st_all < CTW_GROW_TABLE)
      st = FAST ? eps_fast<FSA>(sm, L, g, boost, a.cfg.beam, pass_cap)
                : eps_fixpoint<FSA>(sm, L, g, fc, boost, a.cfg.relax_eps, a.cfg.beam, pass_cap);
    const int vote = sm.st_all;
    if (tid < 32) {
      int tot = tid < R ? cl.map_shared_rank(&sm, tid)->n_slots : 0;  // stable: the closure is over
      for (int d = 16; d; d >>= 1) tot += __shfl_xor_sync(0xFFFFFFFFu, tot, d);
      if (tid == 0) sm.n_all = tot;
    }
    __syncthreads();
    const int n_alloc = sm.n_all;
    const int n_all = min(n_alloc, (int)L.seg);
    if (tid == 0) {
      if (rank == 0) {
        const long long t = clock64();
        prof[1] += t - sm.tclk;
        sm.tclk = t;
        prof[6] += sm.passes;
        prof[8] += n_all;
      }
      prof[9] += sm.eps_items;
      prof[10] += sm.eps_arcs;
      prof[12] += sm.eps_ties > 0;
      prof[13] += sm.eps_ties;
      prof[14] += sm.eps_disc;
      prof[15] += sm.arcs_f;  // (moved to arcs_expanded at the end)
    }
    if (tid == 0) sm.n_slots_max = max(sm.n_slots_max, n_all);
    if (st != CTW_OK) status = st;
    else if (vote >= CTW_GROW_TABLE) status = vote;
    else if (n_alloc == 0) status = CTW_ERR_NO_SURVIVORS;
    else if ((uint32_t)n_alloc > L.seg) status = CTW_GROW_TABLE;

    // ---- prune: beam cutoff from the frame minimum, exact max_active ----
    const double min_cost = key2d(sm.min_key);
    const double cutoff = __dadd_rn(min_cost, a.cfg.beam);
    const unsigned long long cut_key = d2key(cutoff);
    const double bin_scale = (double)CTW_NB / a.cfg.beam;
    // in-beam values and (table index, state) pairs, compacted by the count
    // pass into the (now free) frontier sets
    ulonglong2* sv = reinterpret_cast<ulonglong2*>(L.front);
    uint2* ib = L.front + 2 * (size_t)L.seg;
    if (status == CTW_OK)
      status = count_pass<FAST>(sm, L, fc, sv, ib, n_all, a.cfg.max_ne_iters, cut_key, min_cost, bin_scale, true);
    const int n_ib = sm.cnt_all;
    if (rank == 0 && tid == 0) {
      const long long t = clock64();
      prof[2] += t - sm.tclk;
      sm.tclk = t;
    }
    if (status == CTW_OK) {
      const int in_beam = sm.cnt_all;
      if (rank == 0 && tid == 0) prof[11] += in_beam;
      const bool select = (long long)in_beam > a.cfg.max_active;
      const int n_surv = select ? (int)a.cfg.max_active : in_beam;
      if (select) select_threshold(sm, L, fc, sv, ib, n_ib, cut_key, min_cost, bin_scale, a.cfg.max_active);
      if (rank == 0 && tid == 0) {
        const long long t = clock64();
        prof[3] += t - sm.tclk;
        prof[7] += select;
        sm.tclk = t;
      }
      if (sm.n_rec + n_surv > lane.rcap) {
        status = CTW_GROW_HIST;
        if (tid == 0) sm.rec_need = sm.n_rec + n_surv;
      } else if (n_surv > lane.scap) {
        status = CTW_GROW_SRC;
        if (tid == 0) sm.rec_need = n_surv;
      } else {
        // ---- records + next sources: per-thread counts, one block scan,
        // one cluster counter for the rank's base, then independent
        // per-survivor writes (record order inside a frame is free: the
        // export orders by state) ----
        // the select result is read from shared memory where it is used: held
        // in registers it would stay live across the whole survivor loop
        auto keep = [&](unsigned long long key, uint32_t state) -> bool {
          if (key > cut_key) return false;
          if (!select) return true;
          if (sm.l_radix) return cmp_prefix(key, state, sm.l_depth, sm.l_ph, sm.l_pl) <= 0;
          const int bb = cost_bin(key, min_cost, bin_scale);
          const unsigned long long tk = sm.l_tk;
          return bb < sm.l_bin || (bb == sm.l_bin && (key < tk || (key == tk && state <= sm.l_ts)));
        };
        int mine = 0;
        for (int i = L.sw0 + tid; i < n_ib; i += L.swstride) mine += keep(sv[i].x, ib[i].y);
        int pos, tot;
        Smem::Scan(sm.scan).ExclusiveSum(mine, pos, tot);
        if (tid == 0) sm.rbase = atomicAdd(&fc->rec_ctr, tot);
        __syncthreads();
        pos += sm.rbase;
        const int hop_cap = n_all + 2;
        for (int i = L.sw0 + tid; i < n_ib; i += L.swstride) {
          const ulonglong2 v0 = sv[i];
          const unsigned long long key = v0.x;
          const uint2 it = ib[i];
          const uint32_t st2 = it.y;
          if (!keep(key, st2)) continue;
          const CtwStateRange rg = ld_range(g.ranges, FSA ? (st2 & L.smask) : st2);  // independent of the walk: overlaps it
          const WalkEnd wk = walk<FAST>(L, g, v0, src, pend, hop_cap);
          if (!wk.ok) atomicMax(&sm.status_l, CTW_ERR_EPS_ITERS);
          const int32_t code = record_code<FAST>(sm, L, g, src, v0, wk);
          const long long r = sm.n_rec + pos;
          CtwRecPage* pg = lane.pages[r >> CTW_PAGE_LOG2];
          const int ro = (int)(r & (CTW_PAGE - 1));
          pg->link[ro] = make_int2(wk.bp, code);
          pg->plab[ro] = wk.anc;
          pg->state[ro] = (int32_t)st2;
          const double cost = key2d(key);
          pg->cost[ro] = cost;
          CtwSrc ns;
          ns.state = (int32_t)st2;
          ns.bp = (int32_t)r;
          ns.cost = cost;
          ns.emit_beg = rg.emit_beg;
          ns.emit_end = rg.emit_end;
          ns.anc = code != 0 ? (int32_t)r : wk.anc;
#if CTW_SRC256
          asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(nsrc + pos),
                       "l"(((unsigned long long)(uint32_t)ns.bp << 32) | (uint32_t)ns.state),
                       "l"((unsigned long long)__double_as_longlong(ns.cost)),
                       "l"(((unsigned long long)ns.emit_end << 32) | ns.emit_beg),
                       "l"((unsigned long long)(uint32_t)ns.anc)
                       : "memory");
#else
          nsrc[pos] = ns;
#endif
          ++pos;
        }
        if (rank == 0 && tid == 0) lane.frame_base[lane.frame_count + f] = sm.n_rec;
        const int v2 = csync(sm);  // (H)
        if (tid == 0) {
          sm.tot_surv = *((volatile int*)&fc->rec_ctr);
          sm.n_rec += sm.tot_surv;
        }
        __syncthreads();
        n_src = sm.tot_surv;
        if (v2 != CTW_OK) status = v2;  // grow request (>= 16) or a failed walk (ERR_EPS_ITERS)
      }
    }
    if (rank == 0 && tid == 0) {
      const long long t = clock64();
      prof[4] += t - sm.tclk;
      sm.tclk = t;
    }

    // ---- reset every table entry this rank created (also on failure) ----
    reset_slots<FAST>(L, n_all);
    __syncthreads();
    if (rank == 0 && tid == 0) prof[5] += clock64() - sm.tclk;
    if (status != CTW_OK) {
      if (tid == 0) sm.err_frame = f;
      break;
    }
    cur_buf = nxt_buf;
    pend_valid = 0;
  }

  // per-rank diagnostics -> rank 0 (plain stores + remote loads between two
  // barriers; the second keeps every rank's shared memory alive until rank 0
  // has read it)
  cl.sync();
  long long dsum[7] = {0, 0, 0, 0, 0, 0, 0};
  if (rank == 0 && tid == 0)
    for (int r = 0; r < R; ++r) {
      const Smem* o = cl.map_shared_rank(&sm, r);
      const int ks[6] = {9, 10, 12, 13, 14, 15};
      for (int j = 0; j < 6; ++j) dsum[j] += (long long)o->mydiag[ks[j]];
      dsum[6] += (long long)o->eps_idle;
    }
  cl.sync();
  if (rank == 0 && tid == 0) {
    CtwLaneOut o;
    o.status = status;
    o.err_frame = sm.err_frame;
    o.n_slots_max = sm.n_slots_max;
    o.arcs_expanded = dsum[5];
    o.src_total = sm.src_total;
    o.rec_need = sm.rec_need;
    for (int k = 0; k < CTW_NPROF; ++k) o.prof[k] = prof[k];
    o.prof[9] = dsum[0];
    o.prof[10] = dsum[1];
    o.prof[12] = dsum[2];
    o.prof[13] = dsum[3];
    o.prof[14] = dsum[4];
    o.prof[15] = dsum[6];  // epsilon-barrier idle warp-cycles (CTW_IDLE_PROF builds), else 0
    if (status == CTW_OK) {
      lane.n_src = n_src;
      lane.src_buf = (F > 0) ? cur_buf : committed;
      lane.frame_count += F;
      lane.pool_used = sm.pool_used;
      lane.n_rec = sm.n_rec;
      lane.pend_valid = pend_valid;
    }
    o.n_src = lane.n_src;
    o.src_buf = lane.src_buf;
    o.frame_count = lane.frame_count;
    o.pool_used = lane.pool_used;
    o.n_rec = lane.n_rec;
    o.pend_valid = lane.pend_valid;
    out[b] = o;
  }
}

#ifndef CTW_WIDE  // (the wide translation unit carries only the frame kernel)
// ------------------------------------------------------------ seeding ----

// Fresh channel: token at the start state plus its epsilon closure
// (decoder.py:173-229, same pass discipline: the start slot is slot 0). All
// closure states become sources with bp = -1 and their pending olabel chains
// (no pruning at seed time, as in the reference). One CTA per lane (a cluster
// of one rank).
__global__ void __launch_bounds__(CTW_BS) k_seed(CtwLane* lanes, GraphDev g, const int* lane_ids, int start,
                                                 CtwDecodeCfg cfg, CtwLaneOut* out) {
  __shared__ Smem sm;
  cg::cluster_group cl = cg::this_cluster();
  const int tid = threadIdx.x;
  const int R = (int)cl.num_blocks();
  CtwLane& lane = lanes[lane_ids[blockIdx.x / R]];
  LaneCtx L = lane_ctx(lane, 0, 1, &sm);
  L.prune = false;  // no beam at seed time: the whole closure is kept
  if (R != 1) return;  // launched as single-CTA clusters only
  FrameCtr* fc = &sm.fc[0];
  L.slot_ctr = &fc->nslot;
  if (tid == 0) {
    sm.status_l = CTW_OK;
    sm.epoch = 0;
    sm.st_pub[0] = sm.st_pub[1] = 0;
    sm.st_all = 0;
    sm.pool_used = 0;
    sm.n_slots = 0;
    sm.min_key = ~0ULL;
    sm.pw[0] = sm.pw[1] = 0;
    sm.eps_items = sm.eps_arcs = sm.eps_ties = sm.eps_disc = 0;
    sm.min_pub[0] = sm.min_pub[1] = ~0ULL;
    for (int j = 0; j < 3; ++j) sm.pcnt[j][0] = sm.pcnt[j][1] = 0;
    fc->cnt = 0;
    fc->max_pd = 0;
    fc->nslot = 0;
    bool is_new = false;
    const uint32_t h = tok_insert(L, (uint32_t)start, is_new);
    slot_append(sm, L, h, (uint32_t)start);
    L.T[h].gpos = 0ULL;
    unsigned long long oldk;
    tok_relax(L, &L.T[h], d2key(0.0), CTW_SEED_TB, 0, 0ULL, &oldk);
    sm.snap_slots = sm.n_slots;
  }
  __syncthreads();
  int status = eps_fixpoint<true>(sm, L, g, fc, lane.boost, cfg.relax_eps, cfg.beam,
                            divergence_cap(cfg.max_ne_iters, L.tcap));
  const int n_own = min(sm.n_slots, (int)L.seg);
  if (status == CTW_OK && sm.st_all >= CTW_GROW_TABLE) status = sm.st_all;
  if (status == CTW_OK && (uint32_t)sm.n_slots > L.seg) status = CTW_GROW_TABLE;
  if (status == CTW_OK && n_own > lane.scap) status = CTW_GROW_SRC;
  ulonglong2* sv = reinterpret_cast<ulonglong2*>(lane.front);
  if (status == CTW_OK)
    status = count_pass<false>(sm, L, fc, sv, nullptr, n_own, cfg.max_ne_iters, 0ULL, 0.0, 1.0, false);
  if (status == CTW_OK) {
    CtwSrc* dst = lane.src[0];
    for (int i = tid; i < n_own; i += CTW_BS) {
      const ulonglong2 v0 = sv[i];
      const WalkEnd w = walk<false>(L, g, v0, nullptr, nullptr, n_own + 2);
      if (!w.ok) atomicMax(&sm.status_l, CTW_ERR_EPS_ITERS);
      CtwSrc s;
      s.state = (int32_t)L.slots[i].y;
      s.bp = -1;
      s.anc = -1;
      s.pad = 0;
      s.cost = key2d(v0.x);
      const CtwStateRange rg = g.ranges[(uint32_t)s.state & L.smask];
      s.emit_beg = rg.emit_beg;
      s.emit_end = rg.emit_end;
      dst[i] = s;
      lane.pend[i] = record_code<false>(sm, L, g, nullptr, v0, w);
    }
    __syncthreads();
    if (sm.status_l != CTW_OK) status = sm.status_l;
  }
  reset_slots<false>(L, n_own);
  __syncthreads();
  if (tid == 0) {
    CtwLaneOut o = {};
    o.status = status;
    o.err_frame = -1;
    if (status == CTW_OK) {
      lane.n_src = n_own;
      lane.src_buf = 0;
      lane.frame_count = 0;
      lane.pool_used = sm.pool_used;
      lane.n_rec = 0;
      lane.pend_valid = 1;
    }
    o.n_src = lane.n_src;
    o.src_buf = lane.src_buf;
    o.frame_count = lane.frame_count;
    o.pool_used = lane.pool_used;
    o.n_rec = lane.n_rec;
    o.pend_valid = lane.pend_valid;
    out[blockIdx.x] = o;
  }
}


// ------------------------------------------------------- best path -------

// One CTA per lane: best token (final states preferred, ties -> lowest
// state; decoder.py:384-400), then the backpointer walk over the lane's
// records. Words are written oldest-first into words[woff[b] .. + cap[b]);
// nwords[b] always receives the true length (host retries when too small).
#define CTW_BPB 256  // best path: threads per lane (the argmin over up to max_active tokens)
#define CTW_BPC_NEW 512  // best-path cache: records walked per call that can be cached
#define CTW_BPU 4  // best path: tokens per thread per round of the argmin
__global__ void __launch_bounds__(CTW_BPB) k_best_path(const CtwLane* lanes, GraphDev g, const int* lane_ids, int n,
                                                      int32_t* words, const long long* woff, const int* wcap,
                                                      int* nwords, double* total_cost, int* status, CtwBpCache bc) {
  __shared__ double s_best[CTW_BPB / 32];
  __shared__ int s_state[CTW_BPB / 32], s_i[CTW_BPB / 32];
  __shared__ int32_t s_crec[CTW_BPC_REC];             // the lane's cached best path (record indices, ascending)
  __shared__ int32_t s_new[CTW_BPC_NEW], s_cnt[CTW_BPC_NEW];  // records walked this time (newest first), words each
  const int warp = blockIdx.x;  // (the batch entry)
  const int ln = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (warp >= n) return;
  const CtwLane& lane = lanes[lane_ids[warp]];
  const CtwSrc* src = lane.src[lane.src_buf];
  const double INF = __longlong_as_double(0x7FF0000000000000LL);
  // pass 0: final tokens; pass 1 (only if none final): all tokens
  double best = INF;
  int best_state = 0x7FFFFFFF, best_i = -1;
  auto better = [](double ob, int os, int oi, double b, int bs, int bi) {
    return oi >= 0 && (bi < 0 || ob < b || (ob == b && os < bs));
  };
  const int nsrc = lane.n_src;
  for (int pass = 0; pass < 2 && best_i < 0; ++pass) {
    // CTW_BPU tokens per thread per round, their loads issued together (the
    // scan is a few dependent round trips instead of one per token)
    for (int i0 = threadIdx.x; i0 < nsrc; i0 += CTW_BPB * CTW_BPU) {
      int st[CTW_BPU];
      double c[CTW_BPU], fw[CTW_BPU];
#pragma unroll
      for (int u = 0; u < CTW_BPU; ++u) {
        const int i = i0 + u * CTW_BPB;
        st[u] = i < nsrc ? src[i].state : 0;
        c[u] = i < nsrc ? src[i].cost : INF;
      }
#pragma unroll
      for (int u = 0; u < CTW_BPU; ++u)
        fw[u] = (pass == 0 && i0 + u * CTW_BPB < nsrc) ? g.final_w[(uint32_t)st[u] & lane.smask] : 0.0;
#pragma unroll
      for (int u = 0; u < CTW_BPU; ++u) {
        const int i = i0 + u * CTW_BPB;
        if (i >= nsrc) continue;
        double tot;
        if (pass == 0) {
          if (fw[u] == INF) continue;
          tot = c[u] + fw[u];
        } else {
          tot = c[u];
          if (!(tot < INF)) continue;
        }
        if (tot < best || (tot == best && st[u] < best_state)) {
          best = tot;
          best_state = st[u];
          best_i = i;
        }
      }
    }
    for (int o = 16; o; o >>= 1) {
      const double ob = __shfl_xor_sync(0xFFFFFFFFu, best, o);
      const int os = __shfl_xor_sync(0xFFFFFFFFu, best_state, o);
      const int oi = __shfl_xor_sync(0xFFFFFFFFu, best_i, o);
      if (better(ob, os, oi, best, best_state, best_i)) {
        best = ob;
        best_state = os;
        best_i = oi;
      }
    }
    if (ln == 0) {
      s_best[wid] = best;
      s_state[wid] = best_state;
      s_i[wid] = best_i;
    }
    __syncthreads();
    best = s_best[0];
    best_state = s_state[0];
    best_i = s_i[0];
    for (int k = 1; k < CTW_BPB / 32; ++k)
      if (better(s_best[k], s_state[k], s_i[k], best, best_state, best_i)) {
        best = s_best[k];
        best_state = s_state[k];
        best_i = s_i[k];
      }
    __syncthreads();  // (the slots are rewritten by the next pass)
  }
  if (threadIdx.x >= 32) return;  // the walk and the word move: warp 0
  if (best_i < 0) {
    if (ln == 0) {
      status[warp] = 1;
      nwords[warp] = 0;
      total_cost[warp] = INF;
    }
    return;
  }
  // one walk of the labelled-record chain (lane 0): words are written
  // newest-first at the end of the lane's window, then the warp moves them
  // into place. With a best-path cache (streaming: ctw_advance_best), the
  // walk stops at the first record on the lane's previous best path -- its
  // ancestry is that path's prefix, whose words are copied from the cache --
  // so a step costs one hop per new word instead of one per word so far.
  const int lid = lane_ids[warp];
  const bool cached = bc.n != nullptr && lid < bc.lanes;
  const int cn = cached ? bc.n[lid] : 0;
  const int32_t* crec = cached ? bc.rec + (size_t)lid * CTW_BPC_REC : nullptr;
  for (int k = ln; k < cn; k += 32) s_crec[k] = crec[k];
  __syncwarp();
  const int cap = wcap[warp];
  int32_t* w = words + woff[warp];
  int pos = cap, count = 0, hit = -1, nnew = 0, pre = 0;
  if (ln == 0) {
    status[warp] = 0;
    total_cost[warp] = best;
    // labelled records only: anc / plab skip the frames without output labels
    for (int r = src[best_i].anc; r >= 0;) {
      if (cn > 0 && r <= s_crec[cn - 1]) {
        int lo = 0, hi = cn - 1;  // binary search of r in the cached path
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (s_crec[mid] < r) lo = mid + 1;
          else hi = mid;
        }
        if (s_crec[lo] == r) {
          hit = lo;
          break;
        }
      }
      const CtwRecPage* pg = lane.pages[r >> CTW_PAGE_LOG2];
      const int2 lk = pg->link[r & (CTW_PAGE - 1)];
      const int nxt = pg->plab[r & (CTW_PAGE - 1)];
      const int c = lk.y;
      int m = 0;
      if (c > 0) {
        if (pos > 0) w[pos - 1] = c;
        --pos;
        m = 1;
      } else if (c < 0) {
        const int32_t* seg = lane.pool + (-c - 1);
        m = seg[0];
        for (int j = m - 1; j >= 0; --j) {
          if (pos > 0) w[pos - 1] = seg[1 + j];
          --pos;
        }
      }
      count += m;
      if (nnew < CTW_BPC_NEW) {
        s_new[nnew] = r;
        s_cnt[nnew] = m;
      }
      ++nnew;
      r = nxt;
    }
    pre = hit >= 0 ? bc.cum[(size_t)lid * CTW_BPC_REC + hit] : 0;
    nwords[warp] = pre + count;  // > cap: the host retries with a bigger window
  }
  count = __shfl_sync(0xFFFFFFFFu, count, 0);
  pos = __shfl_sync(0xFFFFFFFFu, pos, 0);
  pre = __shfl_sync(0xFFFFFFFFu, pre, 0);
  hit = __shfl_sync(0xFFFFFFFFu, hit, 0);
  nnew = __shfl_sync(0xFFFFFFFFu, nnew, 0);
  if (pre + count > cap) return;
  __syncwarp();
  // new words to [pre, pre + count) (forward, chunk read before written:
  // the destination never overtakes the unread source)
  if (pos != pre)
    for (int k = 0; k < count; k += 32) {
      const int32_t v = (k + ln < count) ? w[pos + k + ln] : 0;
      __syncwarp();
      if (k + ln < count) w[pre + k + ln] = v;
      __syncwarp();
    }
  if (!cached) return;
  int32_t* cw = bc.words + (size_t)lid * CTW_BPC_WORDS;
  for (int k = ln; k < pre; k += 32) w[k] = cw[k];
  // the new path into the cache: the kept prefix, then the walked records
  // oldest first (a path too long for the cache leaves it empty)
  const int base = hit + 1;
  const bool fits = nnew <= CTW_BPC_NEW && base + nnew <= CTW_BPC_REC && pre + count <= CTW_BPC_WORDS;
  if (fits) {
    int32_t* rec = bc.rec + (size_t)lid * CTW_BPC_REC;
    int32_t* cum = bc.cum + (size_t)lid * CTW_BPC_REC;
    if (ln == 0) {
      int acc = pre;
      for (int j = 0; j < nnew; ++j) {
        const int k = nnew - 1 - j;
        acc += s_cnt[k];
        rec[base + j] = s_new[k];
        cum[base + j] = acc;
      }
    }
    for (int k = ln; k < count; k += 32) cw[pre + k] = w[pre + k];
  }
  __syncwarp();
  if (ln == 0) bc.n[lid] = fits ? base + nnew : 0;
}

__global__ void k_clear_table(CtwTok* T, uint32_t n) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) tok_clear(&T[i]);
}
#endif  // CTW_WIDE

}  // namespace

// ------------------------------------------------------ launch wrappers ---

// The frame kernel over n lanes with R CTAs (ranks) per lane, CTW_BS
// threads per CTA (this translation unit's block size).
static int launch_decode_r(CtwLane* d_lanes, const CtwStateRange* ranges, const CtwArc* arcs,
                           const int32_t* olabel, const double* final_w, const void* loglik, int is_f64, int width,
                           const long long* ll_off, const int* nframes, const int* lane_ids, int n,
                           const CtwDecodeCfg* cfg, CtwLaneOut* out, int any_fsa, int fast, int ebits, int eps_lab,
                           cudaStream_t stream, int R) {
  GraphDev g{ranges, arcs, olabel, final_w};
  void (*KFN)(CtwLane*, GraphDev, ChunkArgs, CtwLaneOut*) =
      fast ? (any_fsa ? k_decode_chunk<true, true> : k_decode_chunk<false, true>)
           : (any_fsa ? k_decode_chunk<true, false> : k_decode_chunk<false, false>);
  ChunkArgs a{loglik, ll_off, nframes, lane_ids, width, is_f64, ebits, eps_lab, *cfg};
  const size_t dyn = (width <= CTW_MAX_SMEM_WIDTH ? (size_t)width : 0) * sizeof(double);
  if (dyn + sizeof(Smem) > 48 * 1024)
    cudaFuncSetAttribute(KFN, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  (void)cudaGetLastError();  // drop stale errors of unchecked calls
  if (R > 8) cudaFuncSetAttribute(KFN, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)(n * R));
  lc.blockDim = dim3(CTW_BS);
  lc.dynamicSmemBytes = dyn;
  lc.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)R;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&lc, KFN, d_lanes, g, a, out);
  if (e != cudaSuccess) return (int)e;
  return (int)cudaGetLastError();
}

#ifdef CTW_WIDE
#ifndef CTW_WIDE_FN
#define CTW_WIDE_FN ctw_launch_decode_wide
#define CTW_WIDE_MAXC ctw_wide_max_clusters
#else
#define CTW_WIDE_MAXC ctw_wide64_max_clusters
#endif
// How many 16-CTA clusters of this build can be resident at once (a lane is
// one cluster: a launch of more lanes than this runs in waves), for a
// launch of the given frame width.
extern "C" int CTW_WIDE_MAXC(int width) {
  static int last_dyn = -1, last = 0;
  const size_t dyn = (width <= CTW_MAX_SMEM_WIDTH ? (size_t)width : 0) * sizeof(double);
  if ((int)dyn == last_dyn) return last;
  void (*KFN)(CtwLane*, GraphDev, ChunkArgs, CtwLaneOut*) = k_decode_chunk<false, true>;
  if (dyn + sizeof(Smem) > 48 * 1024)
    cudaFuncSetAttribute(KFN, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  cudaFuncSetAttribute(KFN, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(16 * 64);
  lc.blockDim = dim3(CTW_BS);
  lc.dynamicSmemBytes = dyn;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 16;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  int m = 0;
  if (cudaOccupancyMaxActiveClusters(&m, (void*)KFN, &lc) != cudaSuccess) {
    (void)cudaGetLastError();
    m = 0;
  }
  last = m;
  last_dyn = (int)dyn;
  return m;
}
// 1024-thread CTAs, 16 per lane: twice the threads of a 512 x 16 lane, for
// launches too small to fill the GPU (streaming steps: per-lane latency)
extern "C" int CTW_WIDE_FN(CtwLane* d_lanes, const CtwStateRange* ranges, const CtwArc* arcs,
                                      const int32_t* olabel, const double* final_w, const void* loglik, int is_f64,
                                      int width, const long long* ll_off, const int* nframes, const int* lane_ids,
                                      int n, const CtwDecodeCfg* cfg, CtwLaneOut* out, int any_fsa, int fast,
                                      int ebits, int eps_lab, cudaStream_t stream) {
  return launch_decode_r(d_lanes, ranges, arcs, olabel, final_w, loglik, is_f64, width, ll_off, nframes, lane_ids, n,
                         cfg, out, any_fsa, fast, ebits, eps_lab, stream, 16);
}
#else
extern "C" int ctw_launch_decode_wide(CtwLane*, const CtwStateRange*, const CtwArc*, const int32_t*, const double*,
                                      const void*, int, int, const long long*, const int*, const int*, int,
                                      const CtwDecodeCfg*, CtwLaneOut*, int, int, int, int, cudaStream_t);
extern "C" int ctw_launch_decode_wide64(CtwLane*, const CtwStateRange*, const CtwArc*, const int32_t*, const double*,
                                        const void*, int, int, const long long*, const int*, const int*, int,
                                        const CtwDecodeCfg*, CtwLaneOut*, int, int, int, int, cudaStream_t);
extern "C" int ctw_wide_max_clusters(int);
extern "C" int ctw_wide64_max_clusters(int);

// Ranks (CTAs) per lane for a launch of n lanes: CTW_CLUSTER overrides.
// Otherwise 8 x 512 threads (best throughput when lanes fill the GPU: 74
// clusters resident); launches too small to fill the GPU -- streaming steps,
// where per-lane latency is the metric -- take 16 CTAs per lane, of 1024
// threads while all its 16 x 1024-thread clusters can be resident at once
// (C4: p50 2.79 -> 2.30 ms, p99 4.13 -> 3.34 ms against 512-thread CTAs),
// else of 512; while the clusters of the build with 64 registers per thread
// (one CTA per SM, no spills) all fit, that build (C4 p50 -1.8 %).
extern "C" int ctw_launch_decode(CtwLane* d_lanes, const CtwStateRange* ranges, const CtwArc* arcs,
                                 const int32_t* olabel, const double* final_w, const void* loglik, int is_f64,
                                 int width, const long long* ll_off, const int* nframes, const int* lane_ids, int n,
                                 const CtwDecodeCfg* cfg, CtwLaneOut* out, int any_fsa, int fast, int ebits,
                                 int eps_lab, cudaStream_t stream) {
  static int env = -1;
  if (env < 0) {
    const char* s = getenv("CTW_CLUSTER");
    env = s ? atoi(s) : 0;
    if (env < 0 || env > CTW_RMAX) env = 0;
  }
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int R = CTW_DEFAULT_CLUSTER;
  if (env) {
    R = env;
  } else if (n <= ctw_wide64_max_clusters(width) && !getenv("CTW_NO_WIDE") && !getenv("CTW_NO_WIDE64")) {
    return ctw_launch_decode_wide64(d_lanes, ranges, arcs, olabel, final_w, loglik, is_f64, width, ll_off, nframes,
                                    lane_ids, n, cfg, out, any_fsa, fast, ebits, eps_lab, stream);
  } else if (n <= ctw_wide_max_clusters(width) && !getenv("CTW_NO_WIDE")) {
    return ctw_launch_decode_wide(d_lanes, ranges, arcs, olabel, final_w, loglik, is_f64, width, ll_off, nframes,
                                  lane_ids, n, cfg, out, any_fsa, fast, ebits, eps_lab, stream);
  } else if ((long long)n * 16 <= (long long)sms * CTW_MINB) {
    R = 16;
  }
  return launch_decode_r(d_lanes, ranges, arcs, olabel, final_w, loglik, is_f64, width, ll_off, nframes, lane_ids, n,
                         cfg, out, any_fsa, fast, ebits, eps_lab, stream, R);
}

extern "C" int ctw_launch_seed(CtwLane* d_lanes, const CtwStateRange* ranges, const CtwArc* arcs,
                               const int32_t* olabel, const double* final_w, const int* lane_ids, int n, int start,
                               const CtwDecodeCfg* cfg, CtwLaneOut* out, cudaStream_t stream) {
  GraphDev g{ranges, arcs, olabel, final_w};
  (void)cudaGetLastError();
  k_seed<<<n, CTW_BS, 0, stream>>>(d_lanes, g, lane_ids, start, *cfg, out);
  return (int)cudaGetLastError();
}

extern "C" int ctw_launch_best(const CtwLane* d_lanes, const CtwStateRange* ranges, const CtwArc* arcs,
                               const int32_t* olabel, const double* final_w, const int* lane_ids, int n,
                               int32_t* words, const long long* woff, const int* wcap, int* nwords, double* total_cost,
                               int* status, CtwBpCache bc, cudaStream_t stream) {
  GraphDev g{ranges, arcs, olabel, final_w};
  (void)cudaGetLastError();
  k_best_path<<<n, CTW_BPB, 0, stream>>>(d_lanes, g, lane_ids, n, words, woff, wcap, nwords, total_cost, status, bc);
  return (int)cudaGetLastError();
}

extern "C" int ctw_launch_clear(CtwTok* T, uint32_t n, cudaStream_t stream) {
  (void)cudaGetLastError();
  k_clear_table<<<(n + 255) / 256, 256, 0, stream>>>(T, n);
  return (int)cudaGetLastError();
}
#endif  // CTW_WIDE
