/*
 * oracle/oracle.c — plain, slow, obviously-correct CPU oracle for round-synchronous
 * speculative-greedy (SGR) vertex colouring, arXiv 1606.06025.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this library.  It shares no
 * code, header, table or helper with the CUDA path (paper_1606_06025_b200/) and the
 * CUDA path never calls it.
 *
 * Single-threaded C99, std arrays only, no bit tricks.  Every function follows the
 * paper's algorithm in the paper's order and notation:
 *   PAPER.md:117-131  Alg. 1 "Sequential Greedy Algorithm" (colorMask stamping)
 *   PAPER.md:141-167  Alg. 2 "Parallel GM Algorithm"
 *   PAPER.md:327-338  Alg. 4 "FirstFit routine"
 *   PAPER.md:340-351  Alg. 5 "ConflictResolve routine"
 *   PAPER.md:421-442  Alg. 7 "Data-driven Parallel Graph Coloring" (W_in / W_out)
 *   PAPER.md:545-557  §3.2 "Heuristic Conflict Resolve" (degree policy)
 * with the readings C1-C17 of DESIGN.md ("Readings of the paper").  Pins (what each
 * function is checked against, other than itself) are listed in DESIGN.md "Oracle pins"
 * and exercised by tests/test_oracle.py.  No function here is "parity unpinned".
 *
 * Return codes: 0 ok, 1 invalid argument, 3 no convergence (rounds > max_rounds),
 * 4 out of memory.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { OR_OK = 0, OR_BAD_ARG = 1, OR_NO_CONVERGENCE = 3, OR_OOM = 4 };
enum { POLICY_HIGHER_ID = 0, POLICY_LOWER_ID = 1, POLICY_DEGREE = 2 };

static int64_t degree_of(const int64_t* R, int64_t v) { return R[v + 1] - R[v]; }

/*
 * recolors(v, w): true when, of a same-colour edge {v, w}, v is the endpoint that is
 * re-queued (its colour cleared).
 *   HIGHER_ID : v > w   (BASELINE.json north star: "the higher vertex id recolors"; reading C1)
 *   LOWER_ID  : v < w   (Alg. 5 literal: "color[v] = color[w] and v < w" clears v)
 *   DEGREE    : deg v < deg w, or deg v = deg w and v > w
 *               (§3.2: larger degree keeps its colour; on a tie "the one
 *                with smaller vertex id is picked" -> keeps it; reading C8)
 */
static int recolors(int policy, const int64_t* R, int64_t v, int64_t w) {
  if (policy == POLICY_HIGHER_ID) return v > w;
  if (policy == POLICY_LOWER_ID) return v < w;
  int64_t dv = degree_of(R, v), dw = degree_of(R, w);
  return dv < dw || (dv == dw && v > w);
}

/*
 * Round-synchronous Data-GC (Alg. 7) = GM (Alg. 2) with W-scan
 * (reading C3).  Per round, with the snapshot reading C2/C4:
 *   Phase A (FirstFit): every v in W_in takes
 *       tent[v] = min{ c >= 1 : colorMask[c] != stamp } after stamping colorMask[color[w]]
 *       for every neighbour w coloured (committed) before this round.  Pending
 *       neighbours have colour 0 (colour clearing) and colour 0
 *       never forbids anything (reading C6).
 *   Phase B (ConflictResolve): v in W_in is conflicting iff some
 *       neighbour w in W_in has tent[w] = tent[v] and recolors(v, w).  Conflicting v are
 *       pushed to W_out; the others keep tent[v] as their colour.
 *   swap(W_in, W_out); loop while W_in is non-empty.
 * W is kept in ascending id order (reading C12).  rounds = number of Phase-A passes
 * (reading C11); num_colors = max colour.
 * trace_w (optional, may be NULL): trace_w[r-1] = |W_in| at round r, for r <= trace_cap.
 */
int oracle_sgr(int64_t n, const int64_t* R, const int32_t* C, int policy, int64_t max_rounds,
               uint32_t* color_out, uint32_t* num_colors, uint32_t* rounds, int64_t* trace_w,
               int64_t trace_cap) {
  if (n < 0 || (n > 0 && (!R || !color_out)) || !num_colors || !rounds) return OR_BAD_ARG;
  if (policy < 0 || policy > 2) return OR_BAD_ARG;
  *num_colors = 0;
  *rounds = 0;
  if (n == 0) return OR_OK;
  if (max_rounds <= 0) max_rounds = n + 1; /* reading C13 */

  int64_t maxdeg = 0;
  for (int64_t v = 0; v < n; ++v)
    if (degree_of(R, v) > maxdeg) maxdeg = degree_of(R, v);

  uint32_t* color = (uint32_t*)calloc((size_t)n, sizeof(uint32_t));   /* 0 = not coloured */
  uint32_t* tent = (uint32_t*)calloc((size_t)n, sizeof(uint32_t));
  char* inW = (char*)calloc((size_t)n, 1);
  int64_t* W_in = (int64_t*)malloc((size_t)n * sizeof(int64_t));
  int64_t* W_out = (int64_t*)malloc((size_t)n * sizeof(int64_t));
  int64_t* colorMask = (int64_t*)malloc((size_t)(maxdeg + 2) * sizeof(int64_t));
  if (!color || !tent || !inW || !W_in || !W_out || !colorMask) {
    free(color); free(tent); free(inW); free(W_in); free(W_out); free(colorMask);
    return OR_OOM;
  }
  /* colorMask initialised with a value a not in V: -1 */
  for (int64_t i = 0; i < maxdeg + 2; ++i) colorMask[i] = -1;
  int64_t stamp = 0; /* unique per (round, vertex): see SURVEY.md Appendix A pitfall */

  int64_t nW = n;
  for (int64_t v = 0; v < n; ++v) W_in[v] = v; /* W_in <- V */
  int64_t r = 0;
  int rc = OR_OK;
  while (nW > 0) { /* while W_in != empty */
    ++r;
    if (r > max_rounds) { rc = OR_NO_CONVERGENCE; break; }
    if (trace_w && r <= trace_cap) trace_w[r - 1] = nW;

    /* Phase A: FirstFit(v) for each v in W_in on the round-start colours */
    for (int64_t i = 0; i < nW; ++i) {
      int64_t v = W_in[i];
      ++stamp;
      for (int64_t e = R[v]; e < R[v + 1]; ++e) {
        int64_t w = C[e];
        colorMask[color[w]] = stamp; /* colorMask[color[w]] <- v */
      }
      uint32_t c = 1; /* c <- min{i > 0 : colorMask[i] != v} */
      while (colorMask[c] == stamp) ++c;
      tent[v] = c;
    }

    /* Phase B: ConflictResolve(v) for each v in W_in on the round's tentative colours */
    for (int64_t i = 0; i < nW; ++i) inW[W_in[i]] = 1;
    int64_t nOut = 0; /* W_out <- empty */
    for (int64_t i = 0; i < nW; ++i) {
      int64_t v = W_in[i];
      int conflicting = 0;
      for (int64_t e = R[v]; e < R[v + 1]; ++e) {
        int64_t w = C[e];
        if (inW[w] && tent[w] == tent[v] && recolors(policy, R, v, w)) { conflicting = 1; break; }
      }
      if (conflicting) W_out[nOut++] = v; /* W_out <- W_out U {v} */
    }
    /* winners keep their colour; losers stay 0 (colour clearing) */
    int64_t j = 0;
    for (int64_t i = 0; i < nW; ++i) {
      int64_t v = W_in[i];
      if (j < nOut && W_out[j] == v) { ++j; continue; }
      color[v] = tent[v];
    }
    for (int64_t i = 0; i < nW; ++i) inW[W_in[i]] = 0;

    /* swap(W_in, W_out) */
    int64_t* t = W_in; W_in = W_out; W_out = t;
    nW = nOut;
  }

  uint32_t mx = 0;
  for (int64_t v = 0; v < n; ++v) {
    color_out[v] = color[v];
    if (color[v] > mx) mx = color[v];
  }
  if (rc == OR_OK) {
    *num_colors = mx;
    *rounds = (uint32_t)r;
  }
  free(color); free(tent); free(inW); free(W_in); free(W_out); free(colorMask);
  return rc;
}

/*
 * Alg. 1 Sequential Greedy, vertices visited in ascending id order
 * (reading C16).  colorMask[color[w]] <- v; c <- min{i > 0 : colorMask[i] != v}.
 */
int oracle_greedy_alg1(int64_t n, const int64_t* R, const int32_t* C, uint32_t* color_out,
                       uint32_t* num_colors) {
  if (n < 0 || (n > 0 && (!R || !color_out)) || !num_colors) return OR_BAD_ARG;
  *num_colors = 0;
  if (n == 0) return OR_OK;
  int64_t maxdeg = 0;
  for (int64_t v = 0; v < n; ++v)
    if (degree_of(R, v) > maxdeg) maxdeg = degree_of(R, v);
  int64_t* colorMask = (int64_t*)malloc((size_t)(maxdeg + 2) * sizeof(int64_t));
  if (!colorMask) return OR_OOM;
  for (int64_t i = 0; i < maxdeg + 2; ++i) colorMask[i] = -1; /* a not in V */
  for (int64_t v = 0; v < n; ++v) color_out[v] = 0;
  uint32_t mx = 0;
  for (int64_t v = 0; v < n; ++v) {
    for (int64_t e = R[v]; e < R[v + 1]; ++e) colorMask[color_out[C[e]]] = v;
    uint32_t c = 1;
    while (colorMask[c] == v) ++c;
    color_out[v] = c;
    if (c > mx) mx = c;
  }
  free(colorMask);
  *num_colors = mx;
  return OR_OK;
}

/*
 * Verifier (SPEC.md:407-415 verify_coloring + SURVEY.md pin P9).  Returns
 *   0 proper, complete and First-Fit fixpoint,
 *   1 incomplete (a colour 0),  2 improper (an edge with equal colours),
 *   3 not a First-Fit fixpoint (color[v] != min{c >= 1 : c not among neighbour colours}).
 * *bad_vertex receives the first offending vertex, or -1.
 */
int oracle_verify(int64_t n, const int64_t* R, const int32_t* C, const uint32_t* color,
                  int64_t* bad_vertex) {
  *bad_vertex = -1;
  for (int64_t v = 0; v < n; ++v)
    if (color[v] == 0) { *bad_vertex = v; return 1; }
  for (int64_t v = 0; v < n; ++v)
    for (int64_t e = R[v]; e < R[v + 1]; ++e)
      if (color[C[e]] == color[v]) { *bad_vertex = v; return 2; }
  int64_t maxdeg = 0;
  for (int64_t v = 0; v < n; ++v)
    if (degree_of(R, v) > maxdeg) maxdeg = degree_of(R, v);
  char* seen = (char*)calloc((size_t)(maxdeg + 2), 1);
  if (!seen) return OR_OOM;
  int rc = 0;
  for (int64_t v = 0; v < n && !rc; ++v) {
    for (int64_t e = R[v]; e < R[v + 1]; ++e)
      if (color[C[e]] <= (uint32_t)(maxdeg + 1)) seen[color[C[e]]] = 1;
    uint32_t c = 1;
    while (seen[c]) ++c;
    if (c != color[v]) { *bad_vertex = v; rc = 3; }
    for (int64_t e = R[v]; e < R[v + 1]; ++e)
      if (color[C[e]] <= (uint32_t)(maxdeg + 1)) seen[color[C[e]]] = 0;
  }
  free(seen);
  return rc;
}

/* backtracking k-colourability test for the brute-force chromatic number */
static int try_color(int64_t v, int64_t n, const int64_t* R, const int32_t* C, int k, int* col) {
  if (v == n) return 1;
  for (int c = 1; c <= k; ++c) {
    int ok = 1;
    for (int64_t e = R[v]; e < R[v + 1]; ++e)
      if (C[e] < v && col[C[e]] == c) { ok = 0; break; }
    if (!ok) continue;
    col[v] = c;
    if (try_color(v + 1, n, R, C, k, col)) return 1;
  }
  col[v] = 0;
  return 0;
}

/* chi(G) by exhaustive backtracking; only for n <= 16 (BASELINE.json: "brute-force
 * chromatic number on graphs with <= 10 vertices").  Returns -1 if n is too large. */
int oracle_chromatic_bruteforce(int64_t n, const int64_t* R, const int32_t* C) {
  if (n < 0 || n > 16) return -1;
  if (n == 0) return 0;
  int col[16];
  for (int k = 1; k <= n; ++k) {
    memset(col, 0, sizeof(col));
    if (try_color(0, n, R, C, k, col)) return k;
  }
  return (int)n;
}
