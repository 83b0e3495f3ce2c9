/*
 * ctcwfst_b200.h -- C-ABI of the B200-native batched WFST beam-search decoder
 * (libctcwfst_b200.so). Plain pointers and sizes only; no torch types.
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/ctcwfst/):
 *   ctw_graph_create / ctw_graph_destroy
 *       FlatGraph(Wfst) + flatten()                decoder.py:70-138
 *       (graph load: CSR arrays in HBM, ranges of epsilon / emitting arcs)
 *   ctw_lanes_create / ctw_lane_reset
 *       create_channel / DecodeState.__init__ ->
 *       _seed_initial_tokens, set_boost            decoder.py:150-238, :344-350
 *   ctw_advance
 *       DecodeState.advance_frames -> kernels.advance_chunk
 *                                                   decoder.py:264-341,
 *                                                   _kernel.pyx:115-502
 *       (batched: many channels per call; chunk-atomic per channel)
 *   ctw_best_path
 *       best_path                                  decoder.py:377-415
 *   ctw_lane_export
 *       DecodeState.history_records / active_tokens decoder.py:240-260
 *   ctw_advance_chunk_compat
 *       the kernel plug-in seam itself: _pykernel.advance_chunk's 19-argument
 *       / 8-tuple contract (_pykernel.py:28-248), so the GPU path can be
 *       injected as DecodeState(graph, config, kernel=...)  (decoder.py:154)
 *
 * Return codes: 0 OK; 1 CTW_ERR_EPS_ITERS; 2 CTW_ERR_NO_SURVIVORS (mirroring
 * _pykernel.py:22-25); 3 CTW_ERR_OOM (_kernel.pyx:22 -> MemoryError);
 * negative: argument / CUDA error, message in ctw_last_error() (thread-local).
 * Per-channel statuses of batched calls are written to status arrays using
 * the same 0/1/2/3 codes.
 */
#ifndef CTCWFST_B200_H
#define CTCWFST_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CTW_ABI_VERSION 1

typedef struct ctw_graph ctw_graph;
typedef struct ctw_lanes ctw_lanes;

/* DecoderConfig (decoder.py:34-48) with max_nonemitting_iters resolved
 * (None -> 2 x num_states, decoder.py:164-168) and max_active clamped to
 * 2**60 (decoder.py:31). */
typedef struct {
  double beam;
  int64_t max_active;
  double acoustic_scale;
  double relax_eps;
  int64_t max_ne_iters;
} ctw_config;

/* Reference-layout history / token export (the arrays returned by
 * _pykernel.advance_chunk, plus the active token set). Arrays are malloc'd by
 * the library and released by ctw_export_free. */
typedef struct {
  int64_t n_frames, n_records, n_olab;
  int64_t* counts;        /* [n_frames] survivors per frame */
  int64_t* rec_prev;      /* [n_records] global record index of predecessor */
  int32_t* rec_state;     /* [n_records] state-ascending within a frame */
  double* rec_cost;       /* [n_records] */
  int64_t* rec_olab_off;  /* [n_records + 1] */
  int32_t* rec_olab_pool; /* [n_olab] olabels, oldest first */
  int64_t n_tok;
  int32_t* tok_state;       /* [n_tok] active tokens, state-ascending */
  double* tok_cost;
  int64_t* tok_bp;          /* global record index, -1 at the root */
  int64_t* tok_chain_off;   /* [n_tok + 1] pending olabels (fresh channels) */
  int32_t* tok_chain_pool;
  int64_t n_chain;
} ctw_export;

/* Pruned lattice of one decoded lane (ctw_lane_lattice).
 * Nodes: seeds 0..n_seeds-1 (the start closure), then n_seeds + record index.
 * Arrays are malloc'd by the library and released by ctw_lattice_free. */
typedef struct {
  int32_t status;      /* 0 ok; 1/2 buffers (internal); 3 closure overflow; 4 no complete path */
  int32_t final_mode;  /* 1: the last layer holds final states (their weights end paths) */
  int32_t frame_count;
  double best;         /* best complete path cost (== best_path's total_cost) */
  double lattice_beam;
  int64_t n_seeds;
  int32_t* seed_state;
  double* seed_cost;
  int64_t* seed_lab_off; /* [n_seeds + 1] pending output labels of each seed */
  int32_t* seed_lab;
  int64_t n_arcs;
  int32_t* arc_src;
  int32_t* arc_dst;
  int32_t* arc_frame;     /* layer of dst */
  int32_t* arc_src_state;
  int32_t* arc_dst_state;
  double* arc_w;
  double* arc_dst_final;  /* final weight of dst when arc_frame is the last layer, else +inf */
  int64_t* arc_lab_off;   /* [n_arcs + 1] */
  int32_t* arc_lab;
  int64_t closure_items, closure_pruned;
} ctw_lattice;

int ctw_abi_version(void);
const char* ctw_last_error(void);
int ctw_device_count(void);

/* Graph load: CSR arrays exactly as FlatGraph holds them (decoder.py:89-127):
 * per state s, arcs [off[s], off[s+1]) stably sorted by ilabel so epsilon
 * arcs are [off[s], eps_end[s]). final_w[s] = +inf for non-final states. The
 * graph is uploaded once into HBM of `device`. */
int ctw_graph_create(const int64_t* off, const int64_t* eps_end, const int32_t* ilabel,
                     const int32_t* olabel, const double* weight, const int32_t* nextstate,
                     const double* final_w, int64_t num_states, int64_t num_arcs, int64_t start,
                     int32_t device, ctw_graph** out);
/* The same from a binary .ctwg file (paper_2311_04996_b200/graphio.py
 * layout: "CTWGRAPH", version 1, then the flattened CSR arrays), memory-
 * mapped -- the graph load path without text parsing (replaces
 * read_fst_text + flatten, wfst.py:213-268, decoder.py:130-138). */
int ctw_graph_load(const char* path, int32_t device, ctw_graph** out);
void ctw_graph_destroy(ctw_graph* g);
/* bytes: device bytes of the resident graph. */
int ctw_graph_info(const ctw_graph* g, int64_t* num_states, int64_t* num_arcs, int64_t* max_ilabel,
                   int64_t* max_olabel, int64_t* bytes);

/* A lane set: n_lanes decoding channels resident on the graph's device,
 * driven by one host thread. `stream` is a cudaStream_t (NULL: the library
 * creates its own non-blocking stream). */
int ctw_lanes_create(ctw_graph* g, int32_t n_lanes, const ctw_config* cfg, void* stream,
                     ctw_lanes** out);
void ctw_lanes_destroy(ctw_lanes* l);
/* Number of lanes; grows the set to at least n (new lanes start unseeded). */
int ctw_lanes_reserve(ctw_lanes* l, int32_t n);

/* Search mode of the lane set (default 0):
 *   0 exact -- the reference's kernel reproduced record for record
 *     (_kernel.pyx:233-444: Gauss-Seidel epsilon order, every slot, every
 *     prev pointer), the mode behind ctw_lane_export / history parity;
 *   1 fast  -- words-exact search for throughput: best-path words identical,
 *     costs the exact min over paths (within the reference's relax_eps stop
 *     rule), out-of-beam candidates never inserted, 16 B token entries.
 * A launch falls back to exact when a lane does not meet the fast mode's
 * preconditions (negative epsilon increments, tight max_ne_iters caps).
 * ctw_lanes_search_info: out3 = {mode, fast launches, decode launches}. */
int ctw_lanes_set_search(ctw_lanes* l, int32_t mode);
int ctw_lanes_search_info(ctw_lanes* l, int64_t* out3);
/* ctw_lanes_graph_info: out3 = {CUDA-graph step launches, graphs captured,
 * 1 if step graphs were turned off (CTW_NO_GRAPH or a capture failure)}.
 * ctw_advance_best runs a step's first round (parameter uploads, frame
 * kernel, partial best paths, result copies) as one graph launch. */
int ctw_lanes_graph_info(ctw_lanes* l, int64_t* out3);

/* Seed lanes: fresh channel = start token + epsilon closure, zero frames, empty
 * history (decoder.py:173-229). boosts[i] is a host f64 vector of
 * boost_lens[i] >= max_olabel + 1 entries or NULL (no boost: bit-identical to
 * the unboosted path, boosting.py:58-62). status[i]: 0 OK or 1 (epsilon cap
 * exceeded while seeding). */
int ctw_lane_reset(ctw_lanes* l, const int32_t* lane_ids, int32_t n, const double* const* boosts,
                   const int64_t* boost_lens, int32_t* status);

/* Replace a lane's boost vector without re-seeding (the reference reads
 * DecodeState.boost at every advance, decoder.py:287-305, so assigning
 * ch.boost between chunks takes effect from the next frame). */
/* Phrase boosting inside the search (on-the-fly composition with a
 * multi-state boost FST; beyond the reference's one-state word boost,
 * boosting.py:75-86). A deterministic automaton over word labels:
 * next[b * (max_olabel + 1) + w] is the state after word w from state b,
 * cost[b] the cost paid on entering b (negative = boost). Token keys become
 * (graph state | automaton state << ceil(log2 num_states)); recorded and
 * exported states are those keys. Takes effect at the next ctw_lane_reset;
 * n_states = 0 removes it. */
int ctw_lane_set_fsa(ctw_lanes* l, int32_t lane, int32_t n_states, const uint16_t* next, const double* cost);
int ctw_lane_set_boost(ctw_lanes* l, int32_t lane, const double* boost, int64_t boost_len);

/* Advance n lanes by one chunk each. loglik rows are `width` wide, dtype 0 =
 * f32, 1 = f64; location 0 = host memory (copied to HBM inside the call),
 * 1 = device memory of the graph's device. Lane i consumes frames[i] rows
 * starting at element offset ll_offsets[i]. A lane whose chunk fails keeps its
 * pre-call state (chunk atomicity, decoder.py:264-267, :307-315); status[i]
 * gets 0/1/2 and err_frame[i] the chunk-relative failing frame. */
int ctw_advance(ctw_lanes* l, const int32_t* lane_ids, int32_t n, const void* loglik, int32_t dtype,
                int32_t location, const int64_t* ll_offsets, const int32_t* frames, int32_t width,
                int32_t* status, int32_t* err_frame);

/* Best path of n lanes. Words of lane i land in words[word_off[i] ..
 * word_off[i+1]) (oldest first); word_off has n + 1 entries. If words_cap is
 * too small, returns -2 and word_off[n] holds the required capacity.
 * status[i]: 0 OK, 1 no surviving hypotheses, 2 no frames decoded. */
int ctw_best_path(ctw_lanes* l, const int32_t* lane_ids, int32_t n, int32_t* words, int64_t words_cap,
                  int64_t* word_off, double* total_cost, int64_t* frame_count, int32_t* status);

/* ctw_advance followed by ctw_best_path of the same lanes in one call: the
 * best-path kernel is enqueued right behind the frame kernel and both come
 * back with one synchronisation (streaming partial hypotheses per chunk,
 * streaming.py:114-137). Outputs as ctw_advance (status, err_frame) and
 * ctw_best_path (words .. bstatus); a lane whose chunk failed keeps its
 * committed state, and its best path is that of the committed frames. */
int ctw_advance_best(ctw_lanes* l, const int32_t* lane_ids, int32_t n, const void* loglik, int32_t dtype,
                     int32_t location, const int64_t* ll_offsets, const int32_t* frames, int32_t width,
                     int32_t* status, int32_t* err_frame, int32_t* words, int64_t words_cap, int64_t* word_off,
                     double* total_cost, int64_t* frame_count, int32_t* bstatus);

/* Channel introspection: committed frame count, active tokens, records. */
/* Partial-history garbage collection (long-running streams; SURVEY 8(f)
 * item 2): keep only the records reachable from each lane's active tokens
 * (everything best_path or a later partial hypothesis can reach), renumber
 * them in frame order and release the rest. kept[i] = records kept. After
 * it, history export returns the kept records only and lattices are not
 * available for the lane. */
int ctw_lane_compact(ctw_lanes* l, const int32_t* lane_ids, int32_t n, int64_t* kept);
/* Grow the lanes' token tables now to the largest size any lane of the set
 * has needed (a streaming server does this when it opens a stream, so no
 * chunk has to be re-run mid-stream for a bigger table). Call between
 * ctw_lane_reset and the first ctw_advance. */
int ctw_lanes_presize(ctw_lanes* l, const int32_t* lane_ids, int32_t n);
int ctw_lane_info(ctw_lanes* l, int32_t lane, int64_t* frame_count, int64_t* n_tokens,
                  int64_t* n_records);
/* Capacities of one lane's device buffers: out6 = {token-table log2 size,
 * source capacity, history record capacity, frame capacity, olabel pool
 * capacity, device bytes held by the lane}. */
int ctw_lane_capacity(ctw_lanes* l, int32_t lane, int64_t* out6);
/* Reference-layout export of frames [frame_from, frame_count) of one lane.
 * Records get global indices base, base+1, ... in (frame, state) order;
 * predecessors inside the exported range are renumbered, external
 * predecessors (compat sources) map through ext_bp. */
int ctw_lane_export(ctw_lanes* l, int32_t lane, int64_t frame_from, int64_t base, const int64_t* ext_bp,
                    int64_t n_ext, ctw_export* out);
void ctw_export_free(ctw_export* e);

/* Lattice generation + pruning for lanes that have decoded a whole
 * utterance (no reference counterpart: SPEC.md:312).
 * `loglik` / `ll_offsets` / `width` / `dtype` / `location` address the same
 * log-likelihood rows the lanes were advanced over (frame 0 .. frame_count-1
 * contiguous per lane). out[i] receives lane i's pruned lattice: arcs with
 * alpha(src) + w + beta(dst) <= best + lattice_beam. */
int ctw_lane_lattice(ctw_lanes* l, const int32_t* lane_ids, int32_t n, const void* loglik, int32_t dtype,
                int32_t location, const int64_t* ll_offsets, int32_t width, double lattice_beam,
                ctw_lattice* out);
void ctw_lattice_free(ctw_lattice* lat);

/* n lowest-cost DISTINCT word sequences of a lattice (A* over the kept arcs
 * with exact remaining costs; at most max_pops partial paths expanded).
 * words[word_off[k] .. word_off[k+1]) and costs[k] for k < *n_found; returns
 * -2 when words_cap is too small (word_off[n] then holds the need). */
int ctw_lattice_nbest(const ctw_lattice* lat, int32_t n, int64_t max_pops, int32_t* words, int64_t words_cap,
                      int64_t* word_off, double* costs, int32_t* n_found, int64_t* pops);

/* The same over the lattice composed with a phrase automaton (multi-word
 * boosting by lattice rescoring): a deterministic
 * Aho-Corasick automaton over word ids -- state 0 the root, per state a
 * goto list sorted by word (goto_off[fsa_states + 1], goto_word, goto_next),
 * a failure link and out_cost[state] = summed cost of the phrases completed
 * on entering it (negative = boost). */
int ctw_lattice_nbest_phrases(const ctw_lattice* lat, int32_t fsa_states, const int32_t* goto_off,
                              const int32_t* goto_word, const int32_t* goto_next, const int32_t* fail_link,
                              const double* out_cost, int32_t n, int64_t max_pops, int32_t* words,
                              int64_t words_cap, int64_t* word_off, double* costs, int32_t* n_found, int64_t* pops);

/* Counters since creation (or the last reset): all kernel launches, launches
 * of the frame kernel and their total device milliseconds (CUDA events on the
 * lane stream around each launch), emitting arcs relaxed (E_emit), source
 * tokens expanded (N_src), lane-frames advanced, max slots seen in a frame. */
int ctw_lanes_stats(ctw_lanes* l, int64_t* launches, int64_t* decode_launches, double* decode_ms,
                    int64_t* arcs, int64_t* src_tokens, int64_t* frames, int64_t* max_slots);
int ctw_lanes_reset_stats(ctw_lanes* l);
/* Per-stage profile of the frame kernel summed over lanes and frames since
 * the last reset (16 counters): SM cycles of [0] emitting expansion, [1]
 * epsilon closure, [2] beam count, [3] max-active select, [4] records, [5]
 * table reset; [6] epsilon passes, [7] frames needing the select, [8] slots,
 * [9] epsilon frontier items, [10] epsilon arcs relaxed, [11] in-beam slots,
 * [12] frames with an epsilon/epsilon tie between distinct predecessors,
 * [13] such ties, [14] epsilon arcs relaxed for discovery only, [15] reserved. */
int ctw_lanes_profile(ctw_lanes* l, int64_t* out16);
/* Host-side breakdown of ctw_advance since the last reset: out10 =
 * {staging H2D s, capacity pre-sizing s, launch-to-completion wait s,
 * post-processing s, grow re-runs, calls, lanes re-run for a bigger token
 * table / history / olabel pool / source buffer}. Diagnostics. */
int ctw_lanes_host_timing(ctw_lanes* l, double* out10);
void* ctw_lanes_stream(ctw_lanes* l);

/* The reference kernel contract (_pykernel.py:28-248) on the GPU: same inputs
 * (host arrays), same outputs (in `out`, counts/rec_* fields; tok_* unused).
 * Returns 0, 1, 2 like the reference (3 -> MemoryError); err_frame is
 * chunk-relative. */
int ctw_advance_chunk_compat(const int64_t* off, const int64_t* eps_end, const int32_t* ilabel,
                             const int32_t* olabel, const double* weight, const int32_t* nextstate,
                             int64_t num_states, int64_t num_arcs, const int32_t* act_state,
                             const double* act_cost, const int64_t* act_bp, const int64_t* act_chain_off,
                             const int32_t* act_chain_pool, int64_t n_src, const double* loglik,
                             int64_t num_frames, int64_t width, double acoustic_scale, double beam,
                             int64_t max_active, double relax_eps, int64_t max_ne_iters,
                             const double* boost, int64_t boost_len, int64_t base, int32_t device,
                             int64_t* err_frame, ctw_export* out);

#ifdef __cplusplus
}
#endif
#endif /* CTCWFST_B200_H */
