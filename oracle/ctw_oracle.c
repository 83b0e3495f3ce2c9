/*
 * ctw_oracle.c -- CPU restatement of the reference's frame-synchronous WFST
 * beam search, used ONLY as a test oracle and as the CPU "port" baseline.
 *
 * TEST INFRASTRUCTURE. Nothing on the product path (paper_2311_04996_b200/)
 * links, loads or calls this file; only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may.
 *
 * What it restates (all paths under /root/reference/pkg/src/ctcwfst/):
 *   ctwo_advance_chunk   _pykernel.py:28-248  (== _kernel.pyx:115-502)
 *     seed sources + pending olabel chains      _pykernel.py:66-79
 *     emitting expansion + recombination        _pykernel.py:103-139
 *     epsilon Gauss-Seidel relaxation           _pykernel.py:141-195
 *     prune: beam cutoff, max_active by (cost,  _pykernel.py:197-213
 *            state), survivors in state order
 *     records + next sources                    _pykernel.py:215-237
 *   ctwo_seed            decoder.py:173-229   (initial epsilon closure)
 *   ctwo_best            decoder.py:377-415   (final-state preference + fallback;
 *                                              the backtrace itself is done by the
 *                                              Python wrapper over the records)
 *
 * Float operations are performed in exactly the reference's order, in IEEE
 * double, and this file must be compiled without FP contraction
 * (-ffp-contract=off) so no FMA fuses a multiply into an add.
 *
 * Parity pinning: tests/test_oracle.py checks this file against the golden
 * vectors in tests/golden/ (made by tests/golden/make_golden.py from the
 * reference itself) and, when oracle/_ref is built, against the compiled
 * reference kernel on random systems.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define CTWO_OK 0
#define CTWO_ERR_EPS_ITERS 1
#define CTWO_ERR_NO_SURVIVORS 2
#define CTWO_ERR_OOM 3

typedef struct {
  void* p;
  size_t n, cap, item;
} vec_t;

static int vec_reserve(vec_t* v, size_t want) {
  if (want <= v->cap) return 0;
  size_t nc = v->cap ? v->cap : 64;
  while (nc < want) nc *= 2;
  void* np = realloc(v->p, nc * v->item);
  if (!np) return -1;
  v->p = np;
  v->cap = nc;
  return 0;
}
#define VPUSH(v, T, x) \
  (vec_reserve(&(v), (v).n + 1) ? -1 : (((T*)(v).p)[(v).n++] = (x), 0))
#define VAT(v, T) ((T*)(v).p)

/* Output of one chunk: arrays owned by the oracle until ctwo_result_free. */
typedef struct {
  int64_t status, err_frame;
  int64_t n_frames, n_records, n_olab;
  int64_t* counts;
  int64_t* rec_prev;
  int32_t* rec_state;
  double* rec_cost;
  int64_t* rec_olab_off; /* n_records + 1 */
  int32_t* rec_olab_pool;
} ctwo_result;

typedef struct {
  double cost;
  int32_t state, slot;
} rank_t;

static int cmp_cost_state(const void* a, const void* b) {
  const rank_t* x = (const rank_t*)a;
  const rank_t* y = (const rank_t*)b;
  if (x->cost < y->cost) return -1;
  if (x->cost > y->cost) return 1;
  return (x->state > y->state) - (x->state < y->state);
}
static int cmp_state(const void* a, const void* b) {
  const rank_t* x = (const rank_t*)a;
  const rank_t* y = (const rank_t*)b;
  return (x->state > y->state) - (x->state < y->state);
}

/* Slot table for one frame: dense state -> slot map with generation stamps. */
typedef struct {
  vec_t state, cost, prev, chain; /* i32, f64, i64, i64 */
} slots_t;

/* Chain arena: olabel + parent (newest-first links). */
typedef struct {
  vec_t ol, parent; /* i32, i64 */
} chains_t;

static inline int64_t chain_push(chains_t* c, int32_t ol, int64_t parent) {
  if (VPUSH(c->ol, int32_t, ol) || VPUSH(c->parent, int64_t, parent)) return -2;
  return (int64_t)c->ol.n - 1;
}

/* Relax one candidate (dest d, cost nc, backpointer bp, chain ch, olabel ol)
 * into the frame's slot table; mirrors _pykernel.py:117-139 / :158-189.
 * Returns -1 on OOM, else 1 when a new slot was created, 0 otherwise;
 * *improve receives (old - new) when an existing slot improved. */
static int relax(slots_t* sl, int32_t* slot_of, int64_t* slot_gen, int64_t gen, chains_t* cs,
                 int32_t d, double nc, int64_t bp, int64_t ch, int32_t ol, double* improve) {
  *improve = 0.0;
  if (slot_gen[d] != gen) {
    int64_t node = ch;
    if (ol != 0) {
      node = chain_push(cs, ol, ch);
      if (node == -2) return -1;
    }
    slot_gen[d] = gen;
    slot_of[d] = (int32_t)sl->state.n;
    if (VPUSH(sl->state, int32_t, d) || VPUSH(sl->cost, double, nc) ||
        VPUSH(sl->prev, int64_t, bp) || VPUSH(sl->chain, int64_t, node))
      return -1;
    return 1;
  }
  int32_t j = slot_of[d];
  double old = VAT(sl->cost, double)[j];
  if (nc < old) {
    int64_t node = ch;
    if (ol != 0) {
      node = chain_push(cs, ol, ch);
      if (node == -2) return -1;
    }
    *improve = old - nc;
    VAT(sl->cost, double)[j] = nc;
    VAT(sl->prev, int64_t)[j] = bp;
    VAT(sl->chain, int64_t)[j] = node;
  }
  return 0;
}

/* Gauss-Seidel epsilon passes over the growing slot list until the largest
 * improvement of a pass is <= relax_eps (a new slot counts as +inf).
 * _pykernel.py:141-195; seeding uses the same discipline (decoder.py:185-219).
 * Returns CTWO_OK, CTWO_ERR_EPS_ITERS or CTWO_ERR_OOM. */
static int eps_closure(const int64_t* off, const int64_t* eps_end, const int32_t* olabel,
                       const double* weight, const int32_t* nextstate, const double* boost,
                       double relax_eps, int64_t max_ne_iters, slots_t* sl, int32_t* slot_of,
                       int64_t* slot_gen, int64_t gen, chains_t* cs) {
  int64_t iters = 0;
  for (;;) {
    iters++;
    if (iters > max_ne_iters) return CTWO_ERR_EPS_ITERS;
    double max_improve = 0.0;
    for (size_t j = 0; j < sl->state.n; j++) {
      int32_t s = VAT(sl->state, int32_t)[j];
      double c = VAT(sl->cost, double)[j];
      int64_t bp = VAT(sl->prev, int64_t)[j];
      int64_t ch = VAT(sl->chain, int64_t)[j];
      for (int64_t a = off[s]; a < eps_end[s]; a++) {
        double nc = c + weight[a];
        int32_t ol = olabel[a];
        if (boost && ol != 0) nc = nc + boost[ol];
        if (!(nc < INFINITY)) continue;
        double imp;
        int r = relax(sl, slot_of, slot_gen, gen, cs, nextstate[a], nc, bp, ch, ol, &imp);
        if (r < 0) return CTWO_ERR_OOM;
        if (r == 1) max_improve = INFINITY;
        else if (imp > max_improve) max_improve = imp;
      }
    }
    if (max_improve <= relax_eps) return CTWO_OK;
  }
}

static void free_vecs(vec_t* vs, int n) {
  for (int i = 0; i < n; i++) free(vs[i].p);
}

static void* dup_out(const vec_t* v, size_t min_items) {
  size_t n = v->n > min_items ? v->n : min_items;
  void* p = malloc((n ? n : 1) * v->item);
  if (p && v->n) memcpy(p, v->p, v->n * v->item);
  return p;
}

int64_t ctwo_advance_chunk(const int64_t* off, const int64_t* eps_end, const int32_t* ilabel,
                           const int32_t* olabel, const double* weight, const int32_t* nextstate,
                           int64_t num_states, const int32_t* act_state, const double* act_cost,
                           const int64_t* act_bp, const int64_t* act_chain_off,
                           const int32_t* act_chain_pool, int64_t n_src, const double* loglik,
                           int64_t num_frames, int64_t width, double acoustic_scale, double beam,
                           int64_t max_active, double relax_eps, int64_t max_ne_iters,
                           const double* boost, int64_t base, ctwo_result* out) {
  memset(out, 0, sizeof(*out));
  int status = CTWO_OK;
  int64_t err_frame = -1;
  int32_t* slot_of = (int32_t*)malloc((size_t)(num_states ? num_states : 1) * sizeof(int32_t));
  int64_t* slot_gen = (int64_t*)malloc((size_t)(num_states ? num_states : 1) * sizeof(int64_t));
  vec_t v[17];
  memset(v, 0, sizeof(v));
  slots_t* sl = (slots_t*)&v[0];
  sl->state.item = 4; sl->cost.item = 8; sl->prev.item = 8; sl->chain.item = 8;
  chains_t* cs = (chains_t*)&v[4];
  cs->ol.item = 4; cs->parent.item = 8;
  vec_t *src_state = &v[6], *src_cost = &v[7], *src_bp = &v[8], *src_chain = &v[9];
  src_state->item = 4; src_cost->item = 8; src_bp->item = 8; src_chain->item = 8;
  vec_t *rec_prev = &v[10], *rec_state = &v[11], *rec_cost = &v[12], *rec_off = &v[13],
        *rec_pool = &v[14], *counts = &v[15], *rank = &v[16];
  rec_prev->item = 8; rec_state->item = 4; rec_cost->item = 8; rec_off->item = 8;
  rec_pool->item = 4; counts->item = 8; rank->item = sizeof(rank_t);
  if (!slot_of || !slot_gen) { status = CTWO_ERR_OOM; goto done; }
  for (int64_t i = 0; i < num_states; i++) slot_gen[i] = -1;
  if (VPUSH(*rec_off, int64_t, 0)) { status = CTWO_ERR_OOM; goto done; }

  /* Sources plus their pending olabel chains (_pykernel.py:66-79). */
  for (int64_t i = 0; i < n_src; i++) {
    int64_t head = -1;
    for (int64_t k = act_chain_off[i]; k < act_chain_off[i + 1]; k++) {
      head = chain_push(cs, act_chain_pool[k], head);
      if (head == -2) { status = CTWO_ERR_OOM; goto done; }
    }
    if (VPUSH(*src_state, int32_t, act_state[i]) || VPUSH(*src_cost, double, act_cost[i]) ||
        VPUSH(*src_bp, int64_t, act_bp[i]) || VPUSH(*src_chain, int64_t, head)) {
      status = CTWO_ERR_OOM; goto done;
    }
  }

  int64_t gen = -1;
  for (int64_t f = 0; f < num_frames; f++) {
    const double* row = loglik + f * width;
    size_t chain_base = cs->ol.n;
    gen++;
    sl->state.n = sl->cost.n = sl->prev.n = sl->chain.n = 0;

    /* Emitting expansion: sources in order x emitting arcs in ilabel order. */
    for (size_t i = 0; i < src_state->n; i++) {
      int32_t s = VAT(*src_state, int32_t)[i];
      double c = VAT(*src_cost, double)[i];
      int64_t bp = VAT(*src_bp, int64_t)[i];
      int64_t ch = VAT(*src_chain, int64_t)[i];
      for (int64_t a = eps_end[s]; a < off[s + 1]; a++) {
        double nc = c + (-acoustic_scale * row[ilabel[a] - 1]) + weight[a];
        int32_t ol = olabel[a];
        if (boost && ol != 0) nc = nc + boost[ol];
        if (!(nc < INFINITY)) continue;
        double imp;
        if (relax(sl, slot_of, slot_gen, gen, cs, nextstate[a], nc, bp, ch, ol, &imp) < 0) {
          status = CTWO_ERR_OOM; err_frame = f; goto done;
        }
      }
    }

    status = eps_closure(off, eps_end, olabel, weight, nextstate, boost, relax_eps, max_ne_iters,
                         sl, slot_of, slot_gen, gen, cs);
    if (status != CTWO_OK) { err_frame = f; goto done; }

    size_t n_slots = sl->state.n;
    if (n_slots == 0) { status = CTWO_ERR_NO_SURVIVORS; err_frame = f; goto done; }

    /* Prune (_pykernel.py:197-213, decoder.py:361-374). */
    const double* scost = VAT(sl->cost, double);
    double min_cost = INFINITY;
    for (size_t j = 0; j < n_slots; j++)
      if (scost[j] < min_cost) min_cost = scost[j];
    double cutoff = min_cost + beam;
    rank->n = 0;
    if (vec_reserve(rank, n_slots)) { status = CTWO_ERR_OOM; err_frame = f; goto done; }
    rank_t* ent = VAT(*rank, rank_t);
    for (size_t j = 0; j < n_slots; j++) {
      if (scost[j] <= cutoff) {
        ent[rank->n].cost = scost[j];
        ent[rank->n].state = VAT(sl->state, int32_t)[j];
        ent[rank->n].slot = (int32_t)j;
        rank->n++;
      }
    }
    int64_t n_surv = (int64_t)rank->n;
    if (n_surv > max_active) {
      qsort(ent, rank->n, sizeof(rank_t), cmp_cost_state);
      n_surv = max_active;
    }
    qsort(ent, (size_t)n_surv, sizeof(rank_t), cmp_state);

    /* Records, oldest-first olabel segments (_pykernel.py:215-228). */
    size_t rec_first = rec_state->n;
    for (int64_t j = 0; j < n_surv; j++) {
      int32_t k = ent[j].slot;
      if (VPUSH(*rec_prev, int64_t, VAT(sl->prev, int64_t)[k]) ||
          VPUSH(*rec_state, int32_t, VAT(sl->state, int32_t)[k]) ||
          VPUSH(*rec_cost, double, VAT(sl->cost, double)[k])) {
        status = CTWO_ERR_OOM; err_frame = f; goto done;
      }
      size_t seg0 = rec_pool->n;
      for (int64_t node = VAT(sl->chain, int64_t)[k]; node >= 0;
           node = VAT(cs->parent, int64_t)[node]) {
        if (VPUSH(*rec_pool, int32_t, VAT(cs->ol, int32_t)[node])) {
          status = CTWO_ERR_OOM; err_frame = f; goto done;
        }
      }
      int32_t* pool = VAT(*rec_pool, int32_t);
      for (size_t lo = seg0, hi = rec_pool->n; lo + 1 < hi; lo++, hi--) {
        int32_t t = pool[lo]; pool[lo] = pool[hi - 1]; pool[hi - 1] = t;
      }
      if (VPUSH(*rec_off, int64_t, (int64_t)rec_pool->n)) {
        status = CTWO_ERR_OOM; err_frame = f; goto done;
      }
    }
    if (VPUSH(*counts, int64_t, n_surv)) { status = CTWO_ERR_OOM; err_frame = f; goto done; }

    /* Survivors become the next sources (_pykernel.py:230-237). */
    src_state->n = src_cost->n = src_bp->n = src_chain->n = 0;
    for (int64_t j = 0; j < n_surv; j++) {
      size_t r = rec_first + (size_t)j;
      if (VPUSH(*src_state, int32_t, VAT(*rec_state, int32_t)[r]) ||
          VPUSH(*src_cost, double, VAT(*rec_cost, double)[r]) ||
          VPUSH(*src_bp, int64_t, base + (int64_t)r) || VPUSH(*src_chain, int64_t, -1)) {
        status = CTWO_ERR_OOM; err_frame = f; goto done;
      }
    }
    cs->ol.n = cs->parent.n = chain_base;
  }

done:
  out->status = status;
  out->err_frame = err_frame;
  out->n_frames = (int64_t)counts->n;
  out->n_records = (int64_t)rec_state->n;
  out->n_olab = (int64_t)rec_pool->n;
  out->counts = (int64_t*)dup_out(counts, 0);
  out->rec_prev = (int64_t*)dup_out(rec_prev, 0);
  out->rec_state = (int32_t*)dup_out(rec_state, 0);
  out->rec_cost = (double*)dup_out(rec_cost, 0);
  out->rec_olab_off = (int64_t*)dup_out(rec_off, 1);
  if (rec_off->n == 0) out->rec_olab_off[0] = 0;
  out->rec_olab_pool = (int32_t*)dup_out(rec_pool, 0);
  free(slot_of);
  free(slot_gen);
  free_vecs(v, 17);
  return status;
}

void ctwo_result_free(ctwo_result* r) {
  free(r->counts); free(r->rec_prev); free(r->rec_state); free(r->rec_cost);
  free(r->rec_olab_off); free(r->rec_olab_pool);
  memset(r, 0, sizeof(*r));
}

/* Initial epsilon closure of {start} (decoder.py:173-229): same pass
 * discipline as the kernels, boost-aware, result sorted by state. Output is
 * written into a ctwo_result with one "frame": rec_state/rec_cost hold the
 * tokens, rec_olab_off/pool their pending chains (oldest-first). Returns
 * CTWO_OK or CTWO_ERR_EPS_ITERS. */
int64_t ctwo_seed(const int64_t* off, const int64_t* eps_end, const int32_t* olabel,
                  const double* weight, const int32_t* nextstate, int64_t num_states,
                  int64_t start, double relax_eps, int64_t max_ne_iters, const double* boost,
                  ctwo_result* out) {
  memset(out, 0, sizeof(*out));
  int32_t* slot_of = (int32_t*)malloc((size_t)num_states * sizeof(int32_t));
  int64_t* slot_gen = (int64_t*)malloc((size_t)num_states * sizeof(int64_t));
  vec_t v[8];
  memset(v, 0, sizeof(v));
  slots_t* sl = (slots_t*)&v[0];
  sl->state.item = 4; sl->cost.item = 8; sl->prev.item = 8; sl->chain.item = 8;
  chains_t* cs = (chains_t*)&v[4];
  cs->ol.item = 4; cs->parent.item = 8;
  vec_t* rank = &v[6];
  rank->item = sizeof(rank_t);
  vec_t* pool = &v[7];
  pool->item = 4;
  int status = CTWO_OK;
  if (!slot_of || !slot_gen) { status = CTWO_ERR_OOM; goto done; }
  for (int64_t i = 0; i < num_states; i++) slot_gen[i] = -1;
  double imp;
  if (relax(sl, slot_of, slot_gen, 0, cs, (int32_t)start, 0.0, -1, -1, 0, &imp) < 0) {
    status = CTWO_ERR_OOM; goto done;
  }
  status = eps_closure(off, eps_end, olabel, weight, nextstate, boost, relax_eps, max_ne_iters,
                       sl, slot_of, slot_gen, 0, cs);
  if (status != CTWO_OK) goto done;
  size_t n = sl->state.n;
  if (vec_reserve(rank, n)) { status = CTWO_ERR_OOM; goto done; }
  rank_t* ent = VAT(*rank, rank_t);
  for (size_t j = 0; j < n; j++) {
    ent[j].cost = VAT(sl->cost, double)[j];
    ent[j].state = VAT(sl->state, int32_t)[j];
    ent[j].slot = (int32_t)j;
  }
  qsort(ent, n, sizeof(rank_t), cmp_state);
  out->n_frames = 1;
  out->n_records = (int64_t)n;
  out->counts = (int64_t*)malloc(sizeof(int64_t));
  out->counts[0] = (int64_t)n;
  out->rec_prev = (int64_t*)malloc((n ? n : 1) * sizeof(int64_t));
  out->rec_state = (int32_t*)malloc((n ? n : 1) * sizeof(int32_t));
  out->rec_cost = (double*)malloc((n ? n : 1) * sizeof(double));
  out->rec_olab_off = (int64_t*)malloc((n + 1) * sizeof(int64_t));
  out->rec_olab_off[0] = 0;
  for (size_t j = 0; j < n; j++) {
    out->rec_prev[j] = -1;
    out->rec_state[j] = ent[j].state;
    out->rec_cost[j] = ent[j].cost;
    size_t seg0 = pool->n;
    for (int64_t node = VAT(sl->chain, int64_t)[ent[j].slot]; node >= 0;
         node = VAT(cs->parent, int64_t)[node]) {
      if (VPUSH(*pool, int32_t, VAT(cs->ol, int32_t)[node])) { status = CTWO_ERR_OOM; goto done; }
    }
    int32_t* pp = VAT(*pool, int32_t);
    for (size_t lo = seg0, hi = pool->n; lo + 1 < hi; lo++, hi--) {
      int32_t t = pp[lo]; pp[lo] = pp[hi - 1]; pp[hi - 1] = t;
    }
    out->rec_olab_off[j + 1] = (int64_t)pool->n;
  }
  out->n_olab = (int64_t)pool->n;
  out->rec_olab_pool = (int32_t*)dup_out(pool, 0);
done:
  out->status = status;
  free(slot_of);
  free(slot_gen);
  free_vecs(v, 8);
  return status;
}

/* best_path token choice (decoder.py:384-400): min cost+final over final
 * states, else min cost over all; strict '<' so ties go to the earlier
 * (lower-state) token. Returns the token index or -1; *total gets the cost. */
int64_t ctwo_best(const int32_t* act_state, const double* act_cost, int64_t n,
                  const double* final_w, double* total) {
  int64_t best = -1;
  double best_cost = INFINITY;
  int any_final = 0;
  for (int64_t i = 0; i < n; i++) {
    double fw = final_w[act_state[i]];
    if (fw != INFINITY) {
      double t = act_cost[i] + fw;
      if (!any_final || t < best_cost) { any_final = 1; best_cost = t; best = i; }
    }
  }
  if (!any_final) {
    for (int64_t i = 0; i < n; i++) {
      if (act_cost[i] < best_cost) { best_cost = act_cost[i]; best = i; }
    }
  }
  *total = best_cost;
  return best;
}
