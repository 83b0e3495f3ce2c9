/* examples/c_decode.c -- the C-ABI with no Python: load a .ctwg graph, decode
 * a batch of log-likelihood matrices (raw f32 file: n x frames x width), print
 * each utterance's best word ids and cost. What a non-Python host (cgo, JNI,
 * N-API) binds; see INTEGRATION.md.
 *
 *   gcc -O2 -I include examples/c_decode.c -L paper_2311_04996_b200 \
 *       -lctcwfst_b200 -Wl,-rpath,$PWD/paper_2311_04996_b200 -o c_decode
 *   ./c_decode graph.ctwg loglik.f32 n frames width
 */
#include <stdio.h>
#include <stdlib.h>

#include "ctcwfst_b200.h"

#define CHECK(x)                                                  \
  do {                                                            \
    int rc_ = (x);                                                \
    if (rc_ < 0) {                                                \
      fprintf(stderr, "%s failed (%d): %s\n", #x, rc_, ctw_last_error()); \
      return 1;                                                   \
    }                                                             \
  } while (0)

int main(int argc, char** argv) {
  if (argc != 6) {
    fprintf(stderr, "usage: %s graph.ctwg loglik.f32 n frames width\n", argv[0]);
    return 2;
  }
  const int n = atoi(argv[3]), frames = atoi(argv[4]), width = atoi(argv[5]);
  const size_t cells = (size_t)n * frames * width;
  float* ll = (float*)malloc(cells * sizeof(float));
  FILE* f = fopen(argv[2], "rb");
  if (!f || fread(ll, sizeof(float), cells, f) != cells) {
    fprintf(stderr, "cannot read %s\n", argv[2]);
    return 1;
  }
  fclose(f);
  ctw_graph* g = NULL;
  CHECK(ctw_graph_load(argv[1], 0, &g));
  int64_t S, A, mil, mol, bytes;
  CHECK(ctw_graph_info(g, &S, &A, &mil, &mol, &bytes));
  /* DecoderConfig defaults (decoder.py:34-48): beam 17, max_active 10000,
   * acoustic scale 1, relax epsilon 1e-9, max_nonemitting_iters 2 x states */
  ctw_config cfg = {17.0, 10000, 1.0, 1e-9, 2 * S};
  ctw_lanes* lanes = NULL;
  CHECK(ctw_lanes_create(g, n, &cfg, NULL, &lanes));
  int32_t* ids = (int32_t*)malloc(n * sizeof(int32_t));
  int32_t* st = (int32_t*)malloc(n * sizeof(int32_t));
  int32_t* ef = (int32_t*)malloc(n * sizeof(int32_t));
  int32_t* fr = (int32_t*)malloc(n * sizeof(int32_t));
  int64_t* off = (int64_t*)malloc(n * sizeof(int64_t));
  for (int i = 0; i < n; ++i) {
    ids[i] = i;
    fr[i] = frames;
    off[i] = (int64_t)i * frames * width;
  }
  CHECK(ctw_lane_reset(lanes, ids, n, NULL, NULL, st));
  CHECK(ctw_advance(lanes, ids, n, ll, 0 /* f32 */, 0 /* host */, off, fr, width, st, ef));
  const int64_t cap = (int64_t)n * (frames + 8);
  int32_t* words = (int32_t*)malloc(cap * sizeof(int32_t));
  int64_t* woff = (int64_t*)malloc((n + 1) * sizeof(int64_t));
  double* cost = (double*)malloc(n * sizeof(double));
  int64_t* fcount = (int64_t*)malloc(n * sizeof(int64_t));
  CHECK(ctw_best_path(lanes, ids, n, words, cap, woff, cost, fcount, st));
  for (int i = 0; i < n; ++i) {
    printf("%d %.17g", i, cost[i]);
    for (int64_t k = woff[i]; k < woff[i + 1]; ++k) printf(" %d", words[k]);
    printf("\n");
  }
  ctw_lanes_destroy(lanes);
  ctw_graph_destroy(g);
  return 0;
}
