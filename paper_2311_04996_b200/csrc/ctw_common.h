// ctw_common.h -- data layout shared by the host C-ABI layer and the sm_100a
// kernels of the batched WFST beam-search decoder.
//
// Reference being replaced: the per-channel frame kernel
// /root/reference/pkg/src/ctcwfst/_kernel.pyx:115-502 (== _pykernel.py:28-248)
// and the CSR graph view decoder.py:70-127. See DESIGN.md for the layout
// rationale and the per-unit byte counts used by the roofline.
#pragma once
#include <stdint.h>

// Kernel/lane status words. 0..2 mirror the reference codes
// (_pykernel.py:22-25); 3 mirrors C_ERR_OOM (_kernel.pyx:22). 16..18 are
// internal "grow and re-run the chunk" requests handled by the host layer.
enum {
  CTW_OK = 0,
  CTW_ERR_EPS_ITERS = 1,
  CTW_ERR_NO_SURVIVORS = 2,
  CTW_ERR_OOM = 3,
  CTW_GROW_TABLE = 16,
  CTW_GROW_HIST = 17,
  CTW_GROW_POOL = 18,
  CTW_GROW_SRC = 19,
};

// Per-state arc ranges (16 B, one vector load): epsilon arcs occupy
// [eps_beg, emit_beg), emitting arcs [emit_beg, emit_end) -- the
// FlatGraph invariant of decoder.py:108-116.
struct __align__(16) CtwStateRange {
  uint32_t eps_beg, emit_beg, emit_end, pad;
};

// One arc (16 B, one vector load). Output labels live in a separate int32
// array: they are read only for winners (records) and when a boost vector is
// attached.
struct __align__(16) CtwArc {
  double weight;
  int32_t nextstate;
  int32_t ilabel;
};

// Token-table entry (32 B = one L2 sector), one per state reached in the
// current frame (open addressing on `state`).
//  key, tb, aux  -- updated together by one 128-bit CAS. `key` is the
//     order-preserving bit image of the f64 cost; ties on `key` are broken
//     exactly as the reference's sequential Gauss-Seidel order would:
//       emitting winner: tb = arc index (lowest arc = first writer,
//         _kernel.pyx:243-285), aux = source token index;
//       epsilon winner:  tb = EPS_BIT | arc, aux = pd << 24 | pred table
//         index, where pd is the Gauss-Seidel pass in which the predecessor
//         was processed holding its final value; epsilon candidates never
//         displace an equal-cost emitting / seed winner (strict '<',
//         _kernel.pyx:332) and among themselves order by (pd, gpos(pred), arc).
//  gpos -- the state's position in the reference's slot list
//     (_kernel.pyx:266, :324): level << 56 | chain key, where level 0 =
//     reached by an emitting arc (key = first-arrival arc index) and level L
//     = first discovered by the epsilon closure from a level L-1 slot
//     (key = discoverer's key << 4 | epsilon-arc offset).
//  state -- hash key (CTW_EMPTY when free); stamp -- frontier dedupe epoch.
struct __align__(32) CtwTok {
  unsigned long long key;
  uint32_t tb;
  uint32_t aux;
  unsigned long long gpos;
  uint32_t state;
  uint32_t stamp;
};

#define CTW_EMPTY 0xFFFFFFFFu
#define CTW_EPS_BIT 0x80000000u
#define CTW_SEED_TB 0x7FFFFFFFu

// Lattice history page: CTW_PAGE records in struct-of-arrays layout. A
// lane's history is a table of pages, so it grows by appending pages (no
// copy of the records already written).
#define CTW_PAGE_LOG2 16
#define CTW_PAGE (1 << CTW_PAGE_LOG2)
struct CtwRecPage {
  int2 link[CTW_PAGE];      // {prev record, olabel code}
  int32_t state[CTW_PAGE];
  double cost[CTW_PAGE];
  int32_t plab[CTW_PAGE];   // nearest strict ancestor record with output labels (-1: none)
};

// Active token (32 B): the frame's sources / survivors.
struct __align__(16) CtwSrc {
  int32_t state;
  int32_t bp;  // record index in this lane's history, -1 root, <= -2: external (compat)
  double cost;
  // the state's emitting arc range, cached with the token so the expansion
  // reads arcs without a dependent range lookup
  uint32_t emit_beg, emit_end;
  // nearest record at or before bp that carries output labels (-1: none):
  // best-path walks follow these links, one hop per word instead of per frame
  int32_t anc;
  int32_t pad;
};

// Device-side descriptor of one lane (= one decoding channel). The host owns
// the authoritative copy; kernels read it and write the committed fields back.
// A lane is decoded by one thread-block cluster of up to CTW_RMAX CTAs
// ("ranks") that share one slot list and four epsilon frontier sets
// (warp-aggregated appends through counters in rank 0's shared memory). The
// token table is grown once a frame fills more than CTW_LOAD(tcap) entries
// (3/4 load), so lists of CTW_LOAD(tcap) entries never overflow in a frame
// that commits.
#define CTW_RMAX 16  // 8 portable; 16 with the non-portable cluster attribute
#ifndef CTW_LOAD_DIV
#define CTW_LOAD_DIV 4
#endif
#define CTW_LOAD(tcap) ((tcap) - (tcap) / CTW_LOAD_DIV)
#define CTW_SLOTS_LEN(tcap) ((uint64_t)CTW_LOAD(tcap))
#define CTW_FRONT_LEN(tcap) (4 * (uint64_t)CTW_LOAD(tcap))

struct CtwLane {
  // token hash table: capacity 1 << tlog2
  CtwTok* table;
  uint2* slots;      // [CTW_SLOTS_LEN] (table index, state) per slot of the frame
  uint2* front;      // [CTW_FRONT_LEN] 4 frontier sets (same pairs); also scratch
  CtwSrc* src[3];    // [scap] each: committed + two working buffers
  int32_t* pend;     // [scap] pending olabel segment of seeded sources
  CtwRecPage** pages;  // history pages: record r lives in pages[r >> CTW_PAGE_LOG2]
  int64_t* frame_base;  // [fcap] first record of each frame
  int32_t* pool;        // [pcap] multi-label olabel segments: [n, l1..ln]
  const double* boost;  // dense f64[boost_len] or null
  uint32_t tlog2;
  int32_t boost_len;
  int64_t rcap;        // records the pages hold (pages x CTW_PAGE)
  int32_t fcap, pcap;
  int32_t scap;      // source capacity: >= max_active (survivors) and the seed closure
  // committed channel state
  int32_t n_src, src_buf, frame_count, pool_used;
  int64_t n_rec;
  int32_t pend_valid;  // committed sources carry pending olabel chains
  // 1 = candidates provably outside the final beam may skip value work:
  // epsilon increments are >= 0 (graph weights and, when epsilon arcs carry
  // olabels, the boost) and max_ne_iters is not a tight cap. Set by the host.
  int32_t prune_ok;
  // phrase automaton (ctw_lane_set_fsa): token keys = graph state | automaton
  // state << sbits; smask recovers the graph state (all ones without one)
  const uint16_t* fsa_next;  // [fsa_states x fsa_width] next automaton state per word label
  const double* fsa_cost;    // [fsa_states] cost of entering the state (negative = boost)
  int32_t fsa_states, fsa_width;
  uint32_t sbits, smask;
};

// Per-launch result of one lane.
struct CtwLaneOut {
  int32_t status;
  int32_t err_frame;   // chunk-relative
  int32_t n_src, src_buf, frame_count, pool_used;
  int64_t n_rec;
  int32_t pend_valid;
  int32_t n_slots_max;  // diagnostics: max slots seen in a frame
  int64_t arcs_expanded;  // diagnostics: emitting arcs relaxed (E_emit)
  int64_t src_total;      // diagnostics: sum of sources over frames (N_src)
  int64_t rec_need;       // CTW_GROW_HIST: records needed through the failing frame
  // stage profile (SM cycles summed over the chunk's frames, thread 0):
  // [0] emitting expansion, [1] epsilon closure, [2] beam count + pass check,
  // [3] max-active select, [4] records, [5] table reset, [6] epsilon passes,
  // [7] frames that needed the select, [8] slots, [9] epsilon frontier items,
  // [10] epsilon arcs relaxed, [11] in-beam slots, [12] frames with an
  // equal-cost epsilon/epsilon tie between distinct predecessors, [13] such ties,
  // [14] epsilon arcs from predecessors outside the running beam (discovery only)
  int64_t prof[16];
};
#define CTW_NPROF 16

struct CtwDecodeCfg {
  double beam;
  double acoustic_scale;
  double relax_eps;
  long long max_active;
  long long max_ne_iters;
};

// ------------------------------------------------------------- lattice ----

// One kept lattice arc (ctw_lattice.cu): nodes are numbered seeds first
// (0 .. n_seeds-1), then n_seeds + record index.
struct CtwLatArc {
  int32_t src, dst;
  double w;       // emitting arc + epsilon continuation cost (reference operation order)
  int32_t code;   // output labels: 0 none, > 0 one label, < 0 segment -(off+1) [n, l1..ln] of the lattice pool
  int32_t frame;  // layer of dst
  int32_t dst_state;
  int32_t src_state;
};

// One lane's seed-token copy (kept for lattices) in a batched reset.
struct CtwSeedCopy {
  CtwSrc* dst_src;
  const CtwSrc* src_src;
  int32_t* dst_pend;
  const int32_t* src_pend;
  int32_t n;
  int32_t pad;
};

// Best-path cache (streaming partial hypotheses): per lane the labelled
// records of the previous best path (ascending), the word count through each
// and its words, in fixed-size per-lane slices of three slabs; n[lane] = 0
// means empty. Written by k_best_path only; the host empties a lane's cache
// when its history is reset or renumbered.
#define CTW_BPC_REC 2048
#define CTW_BPC_WORDS 8192
struct CtwBpCache {
  int32_t* n;      // [lanes]
  int32_t* rec;    // [lanes * CTW_BPC_REC]
  int32_t* cum;    // [lanes * CTW_BPC_REC]
  int32_t* words;  // [lanes * CTW_BPC_WORDS]
  int32_t lanes;   // lanes covered (a lane id >= lanes has no cache)
};

// Epsilon-closure index entry (lattice kernel): for every state s, the
// states reachable from s over epsilon arcs (s itself first) with the
// minimum path weight from s. Built on the device once per graph when no
// epsilon arc carries an output label (then the closure is the same for
// every lane, boost and phrase automaton).
struct __align__(16) CtwClo {
  double w;
  uint32_t state;
  uint32_t pad;
};
#define CTW_CLO_NONE 0x80000000u  // flag in the offset word: closure not indexed (too large)

// Per batch entry (lane) arguments and outputs, device pointers.
struct CtwLatEntry {
  int32_t lane;
  int32_t n_seeds;
  const CtwSrc* seeds;        // seed tokens (state, cost)
  long long ll_off;           // element offset of frame 0 in the log-likelihood buffer
  CtwLatArc* arcs;            // kept arcs
  int32_t arc_cap;
  int32_t* lpool;             // label segments [n, l1..ln]
  int32_t lpool_cap;
  unsigned long long* beta;   // per node (seeds first, then records): sortable key
  double emit_lb;             // lower bound of an emitting arc's weight (+ boost), <= 0
  // outputs
  int32_t n_arcs, lpool_used;
  int32_t status;             // 0 ok, 1 arc buffer full, 2 label pool full, 3 closure overflow, 4 no final path
  int32_t final_mode;         // 1 = final states present at the last layer
  double best;                // best complete path cost (alpha + final)
  long long closure_items, closure_pruned;  // diagnostics
};

