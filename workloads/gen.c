/*
 * workloads/gen.c — seeded synthetic graph generators (test/bench INPUT infrastructure).
 *
 * This module holds NONE of the coloring method's arithmetic.  It only builds the
 * undirected CSR inputs (row_ptr int64[n+1], col_idx int32[m]) that the CPU oracle
 * (oracle/) and the CUDA path (paper_1606_06025_b200/) both consume.  The recipes are
 * the ones fixed in DESIGN.md §"Input recipe" (SURVEY.md §8(d) W1–W3):
 *
 *   W1 R-MAT  (§4 "Rmat-er and Rmat-g", (a,b,c,d) quadrant descent)
 *   W2 27-point stencil N^3 (HPCG-shaped, BASELINE.json configs[1])
 *   W3 R x C 4-neighbour mesh with i.i.d. edge deletion (road/mesh-like, configs[3])
 *
 * Every output is canonical CSR: rows sorted strictly increasing,
 * deduplicated, no self loops, symmetric.  All outputs are bit-identical for a fixed
 * seed regardless of the OpenMP thread count (row contents are sorted after a racy
 * scatter; everything else is computed per index).
 *
 * Ownership: every gen_* function returns malloc'd arrays through out-pointers; the
 * caller releases them with gen_free().  Return value 0 = ok, nonzero = error
 * (1 bad argument, 2 out of memory).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

uint64_t gen_splitmix64(uint64_t x) { return splitmix64(x); }

void gen_free(void* p) { free(p); }

static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

/* insertion sort for short rows, qsort for long ones */
static void sort_row(int32_t* a, int64_t len) {
  if (len < 48) {
    for (int64_t i = 1; i < len; ++i) {
      int32_t x = a[i];
      int64_t j = i - 1;
      while (j >= 0 && a[j] > x) { a[j + 1] = a[j]; --j; }
      a[j + 1] = x;
    }
  } else {
    qsort(a, (size_t)len, sizeof(int32_t), cmp_i32);
  }
}

/* exclusive prefix sum of cnt[0..n) into off[0..n] (off[n] = total); parallel two-pass */
static void prefix_sum(const int64_t* cnt, int64_t* off, int64_t n) {
#ifdef _OPENMP
  int nt = omp_get_max_threads();
#else
  int nt = 1;
#endif
  if (n < (1 << 20) || nt == 1) {
    int64_t s = 0;
    for (int64_t i = 0; i < n; ++i) { off[i] = s; s += cnt[i]; }
    off[n] = s;
    return;
  }
  int64_t* part = (int64_t*)calloc((size_t)nt + 1, sizeof(int64_t));
#pragma omp parallel num_threads(nt)
  {
#ifdef _OPENMP
    int t = omp_get_thread_num();
#else
    int t = 0;
#endif
    int64_t lo = n * t / nt, hi = n * (t + 1) / nt, s = 0;
    for (int64_t i = lo; i < hi; ++i) s += cnt[i];
    part[t + 1] = s;
#pragma omp barrier
#pragma omp single
    for (int k = 1; k <= nt; ++k) part[k] += part[k - 1];
    s = part[t];
    for (int64_t i = lo; i < hi; ++i) { off[i] = s; s += cnt[i]; }
  }
  off[n] = part[nt];
  free(part);
}

/*
 * Build canonical CSR from an arc list (src[i] -> dst[i]) of length k that already holds
 * BOTH directions of every undirected edge and no self loops.  Duplicates are removed
 * (dedupe without redraw).
 */
static int csr_from_arcs(int64_t n, const int32_t* src, const int32_t* dst, int64_t k,
                         int64_t** row_ptr_out, int32_t** col_out, int64_t* m_out) {
  int64_t* deg = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  int64_t* off = (int64_t*)malloc(((size_t)n + 1) * sizeof(int64_t));
  if (!deg || !off) { free(deg); free(off); return 2; }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < k; ++i) {
#pragma omp atomic
    deg[src[i]]++;
  }
  prefix_sum(deg, off, n);
  int32_t* col = (int32_t*)malloc((size_t)(k > 0 ? k : 1) * sizeof(int32_t));
  int64_t* cur = (int64_t*)malloc(((size_t)n + 1) * sizeof(int64_t));
  if (!col || !cur) { free(deg); free(off); free(col); free(cur); return 2; }
  memcpy(cur, off, (size_t)n * sizeof(int64_t));
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < k; ++i) {
    int64_t p;
#pragma omp atomic capture
    p = cur[src[i]]++;
    col[p] = dst[i];
  }
  free(cur);
  /* sort + dedupe each row in place, record new degree */
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t v = 0; v < n; ++v) {
    int32_t* a = col + off[v];
    int64_t len = off[v + 1] - off[v];
    sort_row(a, len);
    int64_t w = 0;
    for (int64_t i = 0; i < len; ++i)
      if (w == 0 || a[i] != a[w - 1]) a[w++] = a[i];
    deg[v] = w;
  }
  int64_t* rp = (int64_t*)malloc(((size_t)n + 1) * sizeof(int64_t));
  if (!rp) { free(deg); free(off); free(col); return 2; }
  prefix_sum(deg, rp, n);
  int64_t m = rp[n];
  int32_t* out = (int32_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(int32_t));
  if (!out) { free(deg); free(off); free(col); free(rp); return 2; }
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t v = 0; v < n; ++v)
    memcpy(out + rp[v], col + off[v], (size_t)deg[v] * sizeof(int32_t));
  free(col); free(deg); free(off);
  *row_ptr_out = rp; *col_out = out; *m_out = m;
  return 0;
}

/*
 * W1: R-MAT.  Recipe:
 *   samples = edge_factor * 2^scale; sample i, level l draws
 *   r = (splitmix64(seed*2^40 + 64*i + l) >> 11) * 2^-53 and picks the quadrant from the
 *   cumulative (a, a+b, a+b+c); u,v built MSB first; both ends relabelled by the seeded
 *   Fisher-Yates permutation pi; both directions added, self loops dropped, deduped.
 *
 * gen_rmat_range builds only the rows [vb, ve) (column ids global), without ever holding the
 * arc list: every sample is recomputed from its counter in two passes (degree count, then
 * scatter), so the memory is the rows' own CSR plus n int32 for pi.  The rows are identical
 * to the same rows of the whole graph (each row is the sorted, deduplicated set of its
 * neighbours), so ranges can be generated independently per rank (BASELINE configs[4],
 * scale 27: 4.3e9 entries).
 */
static inline void rmat_sample(int32_t scale, uint64_t base, int64_t i, double a, double ab, double abc,
                               uint64_t* u_out, uint64_t* v_out) {
  uint64_t u = 0, v = 0;
  for (int l = 0; l < scale; ++l) {
    double r = (double)(splitmix64(base + 64ULL * (uint64_t)i + (uint64_t)l) >> 11) * 0x1.0p-53;
    uint64_t bu, bv;
    if (r < a) { bu = 0; bv = 0; }
    else if (r < ab) { bu = 0; bv = 1; }
    else if (r < abc) { bu = 1; bv = 0; }
    else { bu = 1; bv = 1; }
    u = (u << 1) | bu;
    v = (v << 1) | bv;
  }
  *u_out = u;
  *v_out = v;
}

/* The seeded Fisher-Yates relabelling pi of gen_rmat_range (pi_out: int32[2^scale]); the GPU
 * generator (gen_gpu.cu) takes it as input so both sides use one permutation routine. */
int gen_rmat_perm(int32_t scale, uint64_t seed, int32_t* pi_out) {
  if (scale < 1 || scale > 30 || !pi_out) return 1;
  const int64_t n = (int64_t)1 << scale;
  for (int64_t i = 0; i < n; ++i) pi_out[i] = (int32_t)i;
  for (int64_t i = n - 1; i >= 1; --i) {
    uint64_t j = splitmix64((seed ^ 0x5851F42D4C957F2DULL) + (uint64_t)(n - 1 - i)) % (uint64_t)(i + 1);
    int32_t t = pi_out[i]; pi_out[i] = pi_out[j]; pi_out[j] = t;
  }
  return 0;
}

int gen_rmat_range(int32_t scale, int64_t edge_factor, double a, double b, double c, uint64_t seed,
                   int64_t vb, int64_t ve, int64_t* m_out, int64_t** row_ptr_out, int32_t** col_out) {
  if (scale < 1 || scale > 30 || edge_factor < 0) return 1;
  const int64_t n = (int64_t)1 << scale;
  if (vb < 0 || ve < vb || ve > n) return 1;
  const int64_t nl = ve - vb;
  const int64_t ns = edge_factor * n;
  int32_t* pi = (int32_t*)malloc((size_t)n * sizeof(int32_t));
  int64_t* off = (int64_t*)calloc((size_t)nl + 1, sizeof(int64_t));
  int64_t* cur = (int64_t*)calloc((size_t)nl + 1, sizeof(int64_t));
  if (!pi || !off || !cur) { free(pi); free(off); free(cur); return 2; }
  gen_rmat_perm(scale, seed, pi);
  const double ab = a + b, abc = a + b + c;
  const uint64_t base = seed << 40;
  /* pass 1: arcs per local row (both directions of every non-loop sample, duplicates kept) */
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < ns; ++i) {
    uint64_t u, v;
    rmat_sample(scale, base, i, a, ab, abc, &u, &v);
    const int64_t pu = pi[u], pv = pi[v];
    if (pu == pv) continue;
    if (pu >= vb && pu < ve) {
#pragma omp atomic
      cur[pu - vb]++;
    }
    if (pv >= vb && pv < ve) {
#pragma omp atomic
      cur[pv - vb]++;
    }
  }
  prefix_sum(cur, off, nl);
  const int64_t k = off[nl];
  int32_t* col = (int32_t*)malloc((size_t)(k > 0 ? k : 1) * sizeof(int32_t));
  if (!col) { free(pi); free(off); free(cur); return 2; }
  memcpy(cur, off, (size_t)nl * sizeof(int64_t));
  /* pass 2: scatter */
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < ns; ++i) {
    uint64_t u, v;
    rmat_sample(scale, base, i, a, ab, abc, &u, &v);
    const int64_t pu = pi[u], pv = pi[v];
    if (pu == pv) continue;
    int64_t p;
    if (pu >= vb && pu < ve) {
#pragma omp atomic capture
      p = cur[pu - vb]++;
      col[p] = (int32_t)pv;
    }
    if (pv >= vb && pv < ve) {
#pragma omp atomic capture
      p = cur[pv - vb]++;
      col[p] = (int32_t)pu;
    }
  }
  free(pi);
  /* sort + dedupe every row in place; cur[v] = new degree */
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t v = 0; v < nl; ++v) {
    int32_t* r = col + off[v];
    const int64_t len = off[v + 1] - off[v];
    sort_row(r, len);
    int64_t w = 0;
    for (int64_t i = 0; i < len; ++i)
      if (w == 0 || r[i] != r[w - 1]) r[w++] = r[i];
    cur[v] = w;
  }
  int64_t* rp = (int64_t*)malloc(((size_t)nl + 1) * sizeof(int64_t));
  if (!rp) { free(off); free(cur); free(col); return 2; }
  prefix_sum(cur, rp, nl);
  /* compact in place, ascending rows (rp[v] <= off[v], so a row never overwrites a later one) */
  for (int64_t v = 0; v < nl; ++v)
    if (rp[v] != off[v] && cur[v]) memmove(col + rp[v], col + off[v], (size_t)cur[v] * sizeof(int32_t));
  const int64_t m = rp[nl];
  int32_t* shrunk = (int32_t*)realloc(col, (size_t)(m > 0 ? m : 1) * sizeof(int32_t));
  if (shrunk) col = shrunk;
  free(off); free(cur);
  *row_ptr_out = rp; *col_out = col; *m_out = m;
  return 0;
}

int gen_rmat(int32_t scale, int64_t edge_factor, double a, double b, double c, uint64_t seed,
             int64_t* n_out, int64_t* m_out, int64_t** row_ptr_out, int32_t** col_out) {
  if (scale < 1 || scale > 30) return 1;
  const int64_t n = (int64_t)1 << scale;
  int rc = gen_rmat_range(scale, edge_factor, a, b, c, seed, 0, n, m_out, row_ptr_out, col_out);
  if (rc == 0) *n_out = n;
  return rc;
}

/*
 * W2: 27-point stencil on an nx x ny x nz box, id = x + nx*(y + ny*z) (x fastest,
 * HPCG's natural order); every vertex is adjacent to its up-to-26 in-box neighbours.
 */
int gen_stencil27(int32_t nx, int32_t ny, int32_t nz, int64_t* n_out, int64_t* m_out,
                  int64_t** row_ptr_out, int32_t** col_out) {
  if (nx < 0 || ny < 0 || nz < 0) return 1;
  int64_t n = (int64_t)nx * ny * nz;
  if (n > 0x7fffffffLL) return 1;
  int64_t* rp = (int64_t*)malloc(((size_t)n + 1) * sizeof(int64_t));
  int64_t* deg = (int64_t*)malloc(((size_t)n + 1) * sizeof(int64_t));
  if (!rp || !deg) { free(rp); free(deg); return 2; }
#pragma omp parallel for schedule(static)
  for (int64_t id = 0; id < n; ++id) {
    int64_t x = id % nx, y = (id / nx) % ny, z = id / ((int64_t)nx * ny);
    int64_t cx = 1 + (x > 0) + (x < nx - 1), cy = 1 + (y > 0) + (y < ny - 1), cz = 1 + (z > 0) + (z < nz - 1);
    deg[id] = cx * cy * cz - 1;
  }
  prefix_sum(deg, rp, n);
  int64_t m = rp[n];
  int32_t* col = (int32_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(int32_t));
  if (!col) { free(rp); free(deg); return 2; }
#pragma omp parallel for schedule(static)
  for (int64_t id = 0; id < n; ++id) {
    int64_t x = id % nx, y = (id / nx) % ny, z = id / ((int64_t)nx * ny);
    int64_t p = rp[id];
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          if (!dx && !dy && !dz) continue;
          int64_t X = x + dx, Y = y + dy, Z = z + dz;
          if (X < 0 || X >= nx || Y < 0 || Y >= ny || Z < 0 || Z >= nz) continue;
          col[p++] = (int32_t)(X + nx * (Y + (int64_t)ny * Z));
        }
  }
  free(deg);
  *n_out = n; *m_out = m; *row_ptr_out = rp; *col_out = col;
  return 0;
}

/*
 * W3: R x C 4-neighbour mesh, id = i*C + j.  Undirected edges are numbered horizontal
 * first, e = i*(C-1) + j for {(i,j),(i,j+1)}, then vertical, e = R*(C-1) + i*C + j for
 * {(i,j),(i+1,j)}.  Edge e is kept iff splitmix64(seed ^ e) >= keep_threshold, where
 * keep_threshold = floor(p_delete * 2^64) (0 keeps every edge).
 */
static inline int mesh_keep(uint64_t seed, uint64_t e, uint64_t thr) {
  return thr == 0 || splitmix64(seed ^ e) >= thr;
}

int gen_mesh2d(int32_t R, int32_t C, uint64_t keep_threshold, uint64_t seed, int64_t* n_out,
               int64_t* m_out, int64_t** row_ptr_out, int32_t** col_out) {
  if (R < 0 || C < 0) return 1;
  int64_t n = (int64_t)R * C;
  if (n > 0x7fffffffLL) return 1;
  int64_t* rp = (int64_t*)malloc(((size_t)n + 1) * sizeof(int64_t));
  int64_t* deg = (int64_t*)malloc(((size_t)n + 1) * sizeof(int64_t));
  if (!rp || !deg) { free(rp); free(deg); return 2; }
  const uint64_t H = (uint64_t)R * (uint64_t)(C > 0 ? C - 1 : 0);
#define EDGE_H(i, j) ((uint64_t)(i) * (uint64_t)(C - 1) + (uint64_t)(j))
#define EDGE_V(i, j) (H + (uint64_t)(i) * (uint64_t)C + (uint64_t)(j))
#pragma omp parallel for schedule(static)
  for (int64_t id = 0; id < n; ++id) {
    int64_t i = id / C, j = id % C, d = 0;
    if (i > 0 && mesh_keep(seed, EDGE_V(i - 1, j), keep_threshold)) ++d;
    if (j > 0 && mesh_keep(seed, EDGE_H(i, j - 1), keep_threshold)) ++d;
    if (j < C - 1 && mesh_keep(seed, EDGE_H(i, j), keep_threshold)) ++d;
    if (i < R - 1 && mesh_keep(seed, EDGE_V(i, j), keep_threshold)) ++d;
    deg[id] = d;
  }
  prefix_sum(deg, rp, n);
  int64_t m = rp[n];
  int32_t* col = (int32_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(int32_t));
  if (!col) { free(rp); free(deg); return 2; }
#pragma omp parallel for schedule(static)
  for (int64_t id = 0; id < n; ++id) {
    int64_t i = id / C, j = id % C, p = rp[id];
    if (i > 0 && mesh_keep(seed, EDGE_V(i - 1, j), keep_threshold)) col[p++] = (int32_t)(id - C);
    if (j > 0 && mesh_keep(seed, EDGE_H(i, j - 1), keep_threshold)) col[p++] = (int32_t)(id - 1);
    if (j < C - 1 && mesh_keep(seed, EDGE_H(i, j), keep_threshold)) col[p++] = (int32_t)(id + 1);
    if (i < R - 1 && mesh_keep(seed, EDGE_V(i, j), keep_threshold)) col[p++] = (int32_t)(id + C);
  }
#undef EDGE_H
#undef EDGE_V
  free(deg);
  *n_out = n; *m_out = m; *row_ptr_out = rp; *col_out = col;
  return 0;
}

/*
 * Generic: canonical CSR from an undirected edge list (u[i], v[i]) of length k on n
 * vertices (SPEC.md:50-68 canonicalize + build_csr).  Self loops dropped, both
 * directions added, duplicates removed.  Returns 1 if an endpoint is out of range.
 */
int gen_from_edges(int64_t n, const int32_t* u, const int32_t* v, int64_t k, int64_t* m_out,
                   int64_t** row_ptr_out, int32_t** col_out) {
  if (n < 0 || k < 0) return 1;
  for (int64_t i = 0; i < k; ++i)
    if (u[i] < 0 || u[i] >= n || v[i] < 0 || v[i] >= n) return 1;
  int32_t* src = (int32_t*)malloc((size_t)(2 * k + 1) * sizeof(int32_t));
  int32_t* dst = (int32_t*)malloc((size_t)(2 * k + 1) * sizeof(int32_t));
  if (!src || !dst) { free(src); free(dst); return 2; }
  int64_t a = 0;
  for (int64_t i = 0; i < k; ++i) {
    if (u[i] == v[i]) continue;
    src[a] = u[i]; dst[a] = v[i]; ++a;
    src[a] = v[i]; dst[a] = u[i]; ++a;
  }
  int rc = csr_from_arcs(n, src, dst, a, row_ptr_out, col_out, m_out);
  free(src); free(dst);
  return rc;
}
