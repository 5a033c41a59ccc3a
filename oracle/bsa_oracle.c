/*
 * bsa_oracle.c — plain, slow, fp64 CPU oracle for BSA (Bidirectional Sparse Attention,
 * arXiv 2509.01085). TEST INFRASTRUCTURE ONLY: it may be called only by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs. It shares no
 * code with the CUDA path (paper_2509_01085_b200/csrc) and the product never calls it.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n, "C<k>" = the
 * reading table of DESIGN.md §3. Every function follows the paper's
 * definition step by step in fp64, on bf16 input values widened exactly to fp64 (C25).
 *
 * Parity pins (tests/test_oracle_pins.py) and their status:
 *   geometry ............ pinned (flatten example S:120, centre offsets, exhaustive partition)
 *   pooling ............. pinned (constant, [1,0],[3,2]->[2,1], linearity)
 *   query selection ..... pinned (worked example E-q, tie example S:219, brute force, invariants)
 *   donor / restore ..... pinned (restore example S:228, brute force argmax)
 *   quantile ............ pinned (Phi^-1(.5)=0, Phi^-1(.975) vs statistics.NormalDist, symmetry)
 *   threshold + admission pinned (worked row E-kv, S:315 example, brute force 2^|C| subsets)
 *   attention forward ... pinned (torch SDPA fp64 with dense / boolean masks, invariants)
 *   attention backward .. pinned (finite differences, sum dK = 0, sum dV = sum dO, dQ pruned = 0)
 *   Parity with the paper's own Triton kernels is unpinned (no numeric example is printed).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
  int T, H, W;    /* latent grid */
  int ct, ch, cw; /* cuboid block (C_t, C_h, C_w) */
  int ut, uh, uw; /* query-selection unit = window (w_t, w_h, w_w); == block => block centre */
} or_geom;

static int cdiv(int a, int b) { return (a + b - 1) / b; }
static int imin(int a, int b) { return a < b ? a : b; }

/* 3D -> 1D flattening n = tHW + hW + w. */
int or_flatten(int t, int h, int w, int H, int W) { return t * H * W + h * W + w; }

/* Number of blocks N = ceil(T/C_t) ceil(H/C_h) ceil(W/C_w) (P:140 with truncated edge blocks, C1). */
int or_num_blocks(const or_geom* g) { return cdiv(g->T, g->ct) * cdiv(g->H, g->ch) * cdiv(g->W, g->cw); }

/* Block b (row-major over (N_t, N_h, N_w), C2): origin and actual extent. */
static void block_box(const or_geom* g, int b, int* o, int* e) {
  int Nh = cdiv(g->H, g->ch), Nw = cdiv(g->W, g->cw);
  int bt = b / (Nh * Nw), bh = (b / Nw) % Nh, bw = b % Nw;
  o[0] = bt * g->ct; o[1] = bh * g->ch; o[2] = bw * g->cw;
  e[0] = imin(g->ct, g->T - o[0]); e[1] = imin(g->ch, g->H - o[1]); e[2] = imin(g->cw, g->W - o[2]);
}

/* Per-unit keep count m_u = clamp(ceil(r*|u| - 1e-9), 1, |u|)  (Eq.2, C6). */
int or_keep_count(double r, int n) {
  int m = (int)ceil(r * (double)n - 1e-9);
  if (m < 1) m = 1;
  if (m > n) m = n;
  return m;
}

/* Units of a block: sub-grid of the block's actual extent with nominal unit dims, truncated (C8).
 * Writes the tokens of unit u (ascending) into toks and returns the count; *centre receives the
 * unit's centre token: local (floor(e_t/2), floor(e_h/2), floor(e_w/2)) of the unit extent (C3). */
static int unit_count(const or_geom* g, const int* e) {
  return cdiv(e[0], g->ut) * cdiv(e[1], g->uh) * cdiv(e[2], g->uw);
}
static int unit_tokens(const or_geom* g, const int* o, const int* e, int u, int* toks, int* centre) {
  int nuh = cdiv(e[1], g->uh), nuw = cdiv(e[2], g->uw);
  int ut_i = u / (nuh * nuw), uh_i = (u / nuw) % nuh, uw_i = u % nuw;
  int uo[3] = {o[0] + ut_i * g->ut, o[1] + uh_i * g->uh, o[2] + uw_i * g->uw};
  int ue[3] = {imin(g->ut, e[0] - ut_i * g->ut), imin(g->uh, e[1] - uh_i * g->uh), imin(g->uw, e[2] - uw_i * g->uw)};
  int n = 0;
  for (int a = 0; a < ue[0]; ++a)
    for (int b = 0; b < ue[1]; ++b)
      for (int c = 0; c < ue[2]; ++c) toks[n++] = or_flatten(uo[0] + a, uo[1] + b, uo[2] + c, g->H, g->W);
  *centre = or_flatten(uo[0] + ue[0] / 2, uo[1] + ue[1] / 2, uo[2] + ue[2] / 2, g->H, g->W);
  return n;
}

/* Block tokens in ascending raster order (C2). Returns |b|. */
static int block_tokens(const or_geom* g, int b, int* toks) {
  int o[3], e[3];
  block_box(g, b, o, e);
  int n = 0;
  for (int a = 0; a < e[0]; ++a)
    for (int bb = 0; bb < e[1]; ++bb)
      for (int c = 0; c < e[2]; ++c) toks[n++] = or_flatten(o[0] + a, o[1] + bb, o[2] + c, g->H, g->W);
  return n;
}

static int block_kept(const or_geom* g, double r, int b) {
  int o[3], e[3];
  block_box(g, b, o, e);
  int nu = unit_count(g, e), k = 0;
  int* toks = (int*)malloc(sizeof(int) * g->ct * g->ch * g->cw);
  for (int u = 0; u < nu; ++u) {
    int c, n = unit_tokens(g, o, e, u, toks, &c);
    k += or_keep_count(r, n);
  }
  free(toks);
  return k;
}

/* Sizes: N blocks, L_q kept queries per head. */
void or_sizes(const or_geom* g, double r, int* N, int* Lq) {
  *N = or_num_blocks(g);
  int s = 0;
  for (int b = 0; b < *N; ++b) s += block_kept(g, r, b);
  *Lq = s;
}

/* Partition (a1): block_off[N+1], block_tok[L], block_ext[3N], kept_off[N+1]. */
void or_partition(const or_geom* g, double r, int* block_off, int* block_tok, int* block_ext, int* kept_off) {
  int N = or_num_blocks(g);
  block_off[0] = 0;
  kept_off[0] = 0;
  for (int b = 0; b < N; ++b) {
    int o[3], e[3];
    block_box(g, b, o, e);
    block_ext[3 * b] = e[0]; block_ext[3 * b + 1] = e[1]; block_ext[3 * b + 2] = e[2];
    int n = block_tokens(g, b, block_tok + block_off[b]);
    block_off[b + 1] = block_off[b] + n;
    kept_off[b + 1] = kept_off[b] + block_kept(g, r, b);
  }
}

/* Block average pooling (a2, C11): Xc[b] = (1/|b|) sum_{n in b} X[n], summed in
 * ascending n in fp64. X: [BH, L, d]; Xc: [BH, N, d]. */
void or_pool(const or_geom* g, int BH, int d, const double* X, double* Xc) {
  int N = or_num_blocks(g), L = g->T * g->H * g->W;
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int bh = 0; bh < BH; ++bh)
    for (int b = 0; b < N; ++b) {
      int* toks = (int*)malloc(sizeof(int) * g->ct * g->ch * g->cw);
      int n = block_tokens(g, b, toks);
      double* out = Xc + ((size_t)bh * N + b) * d;
      for (int c = 0; c < d; ++c) out[c] = 0.0;
      for (int i = 0; i < n; ++i) {
        const double* x = X + ((size_t)bh * L + toks[i]) * d;
        for (int c = 0; c < d; ++c) out[c] += x[c];
      }
      for (int c = 0; c < d; ++c) out[c] /= (double)n;
      free(toks);
    }
}

/* cos(a, b) = a.b / (|a| |b|); 0 if either norm is 0 (C4). */
static double dotd(const double* a, const double* b, int d) {
  double s = 0.0;
  for (int c = 0; c < d; ++c) s += a[c] * b[c];
  return s;
}
static double cosine(const double* a, const double* b, int d) {
  double na = sqrt(dotd(a, a, d)), nb = sqrt(dotd(b, b, d));
  if (na == 0.0 || nb == 0.0) return 0.0;
  return dotd(a, b, d) / (na * nb);
}

/* Query selection (a3, Eq.2).
 * Per unit: c_i = cos(q_centre, q_i), c_centre := 1 (self-score 0). Order by
 * (c ascending, token ascending) == rank of 1 - cos descending with ties to the lower index (C5, C7);
 * keep the first m_u. Donor of a pruned i: argmax over kept j of cos(q_i, q_j), ties -> lowest j (C9).
 * Outputs per head: kept_tok[Lq] (block-major, ascending inside a block), donor[L] (self if kept).
 * Optional margins (for the near-tie protocol C24): unit_margin[L] = c_(m) - c_(m-1) gap of the
 * token's unit at the keep cut (DBL_MAX if nothing pruned); donor_margin[L] = best - second best
 * cosine among kept candidates for a pruned token (DBL_MAX otherwise). */
typedef struct { double c; int tok; } ctok;
static int ctok_cmp(const void* x, const void* y) {
  const ctok* a = (const ctok*)x; const ctok* b = (const ctok*)y;
  if (a->c < b->c) return -1;
  if (a->c > b->c) return 1;
  return (a->tok > b->tok) - (a->tok < b->tok);
}
static int int_cmp(const void* x, const void* y) { return (*(const int*)x > *(const int*)y) - (*(const int*)x < *(const int*)y); }

void or_select_queries(const or_geom* g, double r, int BH, int d, const double* Q, int* kept_tok, int* donor,
                       double* unit_margin, double* donor_margin) {
  int N = or_num_blocks(g), L = g->T * g->H * g->W, Lq;
  int* kept_off = (int*)malloc(sizeof(int) * (N + 1));
  kept_off[0] = 0;
  for (int b = 0; b < N; ++b) kept_off[b + 1] = kept_off[b] + block_kept(g, r, b);
  Lq = kept_off[N];
  int maxb = g->ct * g->ch * g->cw;
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int bh = 0; bh < BH; ++bh)
    for (int b = 0; b < N; ++b) {
      const double* Qh = Q + (size_t)bh * L * d;
      int o[3], e[3];
      block_box(g, b, o, e);
      int nu = unit_count(g, e);
      int* toks = (int*)malloc(sizeof(int) * maxb);
      int* kept = (int*)malloc(sizeof(int) * maxb);
      ctok* cs = (ctok*)malloc(sizeof(ctok) * maxb);
      int nk_block = 0;
      int* bkept = kept_tok + (size_t)bh * Lq + kept_off[b];
      for (int u = 0; u < nu; ++u) {
        int centre, n = unit_tokens(g, o, e, u, toks, &centre);
        int m = or_keep_count(r, n);
        for (int i = 0; i < n; ++i) {
          cs[i].tok = toks[i];
          cs[i].c = (toks[i] == centre) ? 1.0 : cosine(Qh + (size_t)centre * d, Qh + (size_t)toks[i] * d, d);
        }
        qsort(cs, n, sizeof(ctok), ctok_cmp);
        double gap = (m < n) ? cs[m].c - cs[m - 1].c : DBL_MAX;
        for (int i = 0; i < m; ++i) kept[i] = cs[i].tok;
        qsort(kept, m, sizeof(int), int_cmp);
        for (int i = 0; i < n; ++i) {
          int t = toks[i];
          if (unit_margin) unit_margin[(size_t)bh * L + t] = gap;
        }
        for (int i = 0; i < m; ++i) {
          donor[(size_t)bh * L + kept[i]] = kept[i];
          if (donor_margin) donor_margin[(size_t)bh * L + kept[i]] = DBL_MAX;
          bkept[nk_block++] = kept[i];
        }
        for (int i = m; i < n; ++i) {
          int t = cs[i].tok;
          double best = -DBL_MAX, second = -DBL_MAX;
          int arg = -1;
          for (int j = 0; j < m; ++j) { /* kept[] ascending: strict > keeps the lowest j on ties */
            double c = cosine(Qh + (size_t)t * d, Qh + (size_t)kept[j] * d, d);
            if (c > best) { second = best; best = c; arg = kept[j]; }
            else if (c > second) second = c;
          }
          donor[(size_t)bh * L + t] = arg;
          if (donor_margin) donor_margin[(size_t)bh * L + t] = (m > 1) ? best - second : DBL_MAX;
        }
      }
      /* block-major, ascending inside the block (units may interleave in raster order) */
      qsort(bkept, nk_block, sizeof(int), int_cmp);
      free(toks); free(kept); free(cs);
    }
  free(kept_off);
}

/* Standard normal quantile Phi^-1(u) (Eq.3's U, C14) by bisection on the lower tail
 * Phi(z) = erfc(-z/sqrt2)/2 until the bracket stops shrinking. For u > 1/2 the symmetric lower
 * tail q = 1 - u (exact in fp64 by Sterbenz) is solved and negated, so both tails keep full
 * relative precision. */
static double lower_tail_quantile(double q) { /* q in (0, 1/2] -> z <= 0 */
  double lo = -40.0, hi = 0.0;
  for (int it = 0; it < 2000; ++it) {
    double mid = 0.5 * (lo + hi);
    if (mid == lo || mid == hi) break;
    double p = 0.5 * erfc(-mid / sqrt(2.0));
    if (p < q) lo = mid; else hi = mid;
  }
  return 0.5 * (lo + hi);
}
double or_normal_quantile(double u) {
  if (u == 0.5) return 0.0;
  if (u < 0.5) return lower_tail_quantile(u);
  return -lower_tail_quantile(1.0 - u);
}

/* KV selection (a4-a6) for every (bh, query-block row i):
 *   s_j = Qc[i].Kc[j] / sqrt(d)                                   (C12)
 *   mu = mean_j s_j, sigma = sqrt(mean_j (s_j - mu)^2)            (Eq.3, C13 population)
 *   k == N: C = all (C15); else z = Phi^-1(clamp(1 - k/N, 1/(2N), 1 - 1/(2N))), p = mu + sigma z,
 *   C = {j : s_j >= p}, empty -> {argmax, lowest j} (C16)
 *   order C by (s desc, j asc); m = max s; e_j = exp(s_j - m); E = sum_C e (in that order);
 *   tau >= 1: S = C; else the shortest prefix with cumulative e >= tau E (Eq.4, C17, C18)
 *   q2k_idx[row] = S ascending, padded with -1; q2k_num[row] = |S|.
 * Optional outputs: thresh[row] = p (or -inf when k == N), scores[BH,N,N],
 *   thr_margin[row] = min_j |s_j - p| / max(|s_j|, |p|, sigma)      (C24 logit rule; DBL_MAX if k == N)
 *   mass_margin[row] = min over the cut of |cum - tau E| / E          (C24 mass rule; DBL_MAX if tau >= 1)
 *   order_margin[row] = (s_(l-1) - s_(l)) / max(sigma, |s|) at the admission cut (DBL_MAX if none). */
typedef struct { double s; int j; } sj;
static int sj_cmp(const void* x, const void* y) {
  const sj* a = (const sj*)x; const sj* b = (const sj*)y;
  if (a->s > b->s) return -1;
  if (a->s < b->s) return 1;
  return (a->j > b->j) - (a->j < b->j);
}

void or_select_kv(int N, int BH, int d, const double* Qc, const double* Kc, int k, double tau, int* q2k_num,
                  int* q2k_idx, double* thresh, double* scores, double* thr_margin, double* mass_margin,
                  double* order_margin) {
  double z = 0.0;
  if (k < N) {
    double u = 1.0 - (double)k / (double)N;
    double lo = 1.0 / (2.0 * N), hi = 1.0 - 1.0 / (2.0 * N);
    if (u < lo) u = lo;
    if (u > hi) u = hi;
    z = or_normal_quantile(u);
  }
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int bh = 0; bh < BH; ++bh)
    for (int i = 0; i < N; ++i) {
      size_t row = (size_t)bh * N + i;
      double* s = (double*)malloc(sizeof(double) * N);
      sj* C = (sj*)malloc(sizeof(sj) * N);
      const double* q = Qc + row * d;
      for (int j = 0; j < N; ++j) s[j] = dotd(q, Kc + ((size_t)bh * N + j) * d, d) / sqrt((double)d);
      if (scores) memcpy(scores + row * N, s, sizeof(double) * N);
      double mu = 0.0;
      for (int j = 0; j < N; ++j) mu += s[j];
      mu /= (double)N;
      double var = 0.0;
      for (int j = 0; j < N; ++j) var += (s[j] - mu) * (s[j] - mu);
      double sigma = sqrt(var / (double)N);
      int nc = 0;
      double tm = DBL_MAX;
      if (k >= N) {
        for (int j = 0; j < N; ++j) { C[nc].s = s[j]; C[nc].j = j; ++nc; }
        if (thresh) thresh[row] = -INFINITY;
      } else {
        double p = mu + sigma * z;
        if (thresh) thresh[row] = p;
        for (int j = 0; j < N; ++j) {
          double den = fmax(fmax(fabs(s[j]), fabs(p)), sigma);
          double mgn = den > 0 ? fabs(s[j] - p) / den : DBL_MAX;
          if (mgn < tm) tm = mgn;
          if (s[j] >= p) { C[nc].s = s[j]; C[nc].j = j; ++nc; }
        }
        if (nc == 0) {
          int arg = 0;
          for (int j = 1; j < N; ++j) if (s[j] > s[arg]) arg = j;
          C[0].s = s[arg]; C[0].j = arg; nc = 1;
        }
      }
      if (thr_margin) thr_margin[row] = tm;
      qsort(C, nc, sizeof(sj), sj_cmp);
      int ell = nc;
      double mm = DBL_MAX, om = DBL_MAX;
      if (tau < 1.0) {
        double m = C[0].s, E = 0.0;
        for (int t = 0; t < nc; ++t) E += exp(C[t].s - m);
        double cum = 0.0;
        ell = nc;
        for (int t = 0; t < nc; ++t) {
          double prev = cum;
          cum += exp(C[t].s - m);
          if (cum >= tau * E) {
            ell = t + 1;
            mm = fmin(fabs(cum - tau * E), fabs(prev - tau * E)) / E;
            if (t == 0) mm = fabs(cum - tau * E) / E;
            break;
          }
        }
      }
      if (ell < nc) {
        double den = fmax(sigma, fabs(C[ell].s));
        om = den > 0 ? (C[ell - 1].s - C[ell].s) / den : DBL_MAX;
      }
      if (mass_margin) mass_margin[row] = mm;
      if (order_margin) order_margin[row] = om;
      int* out = q2k_idx + row * N;
      for (int t = 0; t < ell; ++t) out[t] = C[t].j;
      qsort(out, ell, sizeof(int), int_cmp);
      for (int t = ell; t < N; ++t) out[t] = -1;
      q2k_num[row] = ell;
      free(s); free(C);
    }
}

/* KV selection, SPEC's unified_prob reading of Eq.3/Eq.4 (the variant the north_star's
 * "selection variants" row compares against, C28) for every (bh, row i):
 *   s_j = Qc[i].Kc[j] / sqrt(d); m = max s; e_j = exp(s_j - m); E = sum_j e_j (ascending j);
 *   prob_j = e_j / E; mu = mean_j prob_j, sigma = sqrt(mean_j (prob_j - mu)^2)           (Eq.3 on the
 *   softmax-normalised row); z = Phi^-1(clamp(1 - k/N, 1/(2N), 1 - 1/(2N))) (no k = N bypass here);
 *   p = mu + sigma z clamped to (0, 1] (p_floor = the smallest positive double);
 *   order all j by (s desc, j asc); p >= 1: S = all; else the shortest prefix with cumulative
 *   e >= p E (Eq.4 with p as the mass target, at least one block).
 * thresh[row] = p; mass_margin[row] as in or_select_kv. */
void or_select_kv_unified(int N, int BH, int d, const double* Qc, const double* Kc, int k, int* q2k_num,
                          int* q2k_idx, double* thresh, double* mass_margin) {
  double u = 1.0 - (double)k / (double)N;
  double lo = 1.0 / (2.0 * N), hi = 1.0 - 1.0 / (2.0 * N);
  if (u < lo) u = lo;
  if (u > hi) u = hi;
  const double z = or_normal_quantile(u);
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int bh = 0; bh < BH; ++bh)
    for (int i = 0; i < N; ++i) {
      size_t row = (size_t)bh * N + i;
      double* s = (double*)malloc(sizeof(double) * N);
      sj* C = (sj*)malloc(sizeof(sj) * N);
      const double* q = Qc + row * d;
      for (int j = 0; j < N; ++j) s[j] = dotd(q, Kc + ((size_t)bh * N + j) * d, d) / sqrt((double)d);
      double m = s[0];
      for (int j = 1; j < N; ++j) if (s[j] > m) m = s[j];
      double E = 0.0;
      for (int j = 0; j < N; ++j) E += exp(s[j] - m);
      double mu = 0.0;
      for (int j = 0; j < N; ++j) mu += exp(s[j] - m) / E;
      mu /= (double)N;
      double var = 0.0;
      for (int j = 0; j < N; ++j) {
        double dp = exp(s[j] - m) / E - mu;
        var += dp * dp;
      }
      double sigma = sqrt(var / (double)N);
      double p = mu + sigma * z;
      if (p > 1.0) p = 1.0;
      if (p <= 0.0) p = DBL_MIN;
      if (thresh) thresh[row] = p;
      for (int j = 0; j < N; ++j) { C[j].s = s[j]; C[j].j = j; }
      qsort(C, N, sizeof(sj), sj_cmp);
      int ell = N;
      double mm = DBL_MAX;
      if (p < 1.0) {
        double cum = 0.0;
        for (int t = 0; t < N; ++t) {
          double prev = cum;
          cum += exp(C[t].s - m);
          if (cum >= p * E) {
            ell = t + 1;
            mm = t == 0 ? fabs(cum - p * E) / E : fmin(fabs(cum - p * E), fabs(prev - p * E)) / E;
            break;
          }
        }
      }
      if (mass_margin) mass_margin[row] = mm;
      int* out = q2k_idx + row * N;
      for (int t = 0; t < ell; ++t) out[t] = C[t].j;
      qsort(out, ell, sizeof(int), int_cmp);
      for (int t = ell; t < N; ++t) out[t] = -1;
      q2k_num[row] = ell;
      free(s); free(C);
    }
}

/* Sparse attention forward (a7, Eq.5, C19, C20, C23) for every kept query q of block i:
 * keys = tokens of the blocks in S_i (ascending block id, ascending token), l = scale * q.k,
 * O^s[q] = softmax(l) V, LSE[q] = max l + log sum exp(l - max l); then the fill (C9):
 * O[kept] = O^s, O[pruned t] = O^s[donor(t)].  O: [BH, L, d]; lse: [BH, Lq] (packed order). */
static void attn_row(const or_geom* g, int d, const double* Qh, const double* Kh, const double* Vh, int qtok,
                     const int* blocks, int nblocks, double scale, double* o, double* lse, double* lbuf,
                     int* kbuf) {
  int nk = 0;
  for (int a = 0; a < nblocks; ++a) nk += block_tokens(g, blocks[a], kbuf + nk);
  const double* q = Qh + (size_t)qtok * d;
  double mx = -INFINITY;
  for (int t = 0; t < nk; ++t) {
    lbuf[t] = scale * dotd(q, Kh + (size_t)kbuf[t] * d, d);
    if (lbuf[t] > mx) mx = lbuf[t];
  }
  double sum = 0.0;
  for (int t = 0; t < nk; ++t) { lbuf[t] = exp(lbuf[t] - mx); sum += lbuf[t]; }
  for (int c = 0; c < d; ++c) o[c] = 0.0;
  for (int t = 0; t < nk; ++t) {
    const double* v = Vh + (size_t)kbuf[t] * d;
    double p = lbuf[t] / sum;
    for (int c = 0; c < d; ++c) o[c] += p * v[c];
  }
  *lse = mx + log(sum);
}

/* Query-block range [qb0, qb1) restricts the work to a sample of query blocks (bench cpu_baseline);
 * or_attn_fwd / or_attn_bwd below are the full range. */
static int token_block(const or_geom* g, int t) {
  int tt = t / (g->H * g->W), h = (t / g->W) % g->H, w = t % g->W;
  return ((tt / g->ct) * cdiv(g->H, g->ch) + h / g->ch) * cdiv(g->W, g->cw) + w / g->cw;
}

void or_attn_fwd_range(const or_geom* g, double r, int BH, int d, const double* Q, const double* K,
                       const double* V, const int* kept_tok, const int* donor, const int* q2k_num,
                       const int* q2k_idx, double scale, double* O, double* lse, int qb0, int qb1) {
  int N = or_num_blocks(g), L = g->T * g->H * g->W, Lq;
  int* kept_off = (int*)malloc(sizeof(int) * (N + 1));
  kept_off[0] = 0;
  for (int b = 0; b < N; ++b) kept_off[b + 1] = kept_off[b] + block_kept(g, r, b);
  Lq = kept_off[N];
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int bh = 0; bh < BH; ++bh)
    for (int i = qb0; i < qb1; ++i) {
      double* lbuf = (double*)malloc(sizeof(double) * L);
      int* kbuf = (int*)malloc(sizeof(int) * L);
      size_t row = (size_t)bh * N + i;
      for (int q = kept_off[i]; q < kept_off[i + 1]; ++q) {
        int tok = kept_tok[(size_t)bh * Lq + q];
        attn_row(g, d, Q + (size_t)bh * L * d, K + (size_t)bh * L * d, V + (size_t)bh * L * d, tok,
                 q2k_idx + row * N, q2k_num[row], scale, O + ((size_t)bh * L + tok) * d, lse + (size_t)bh * Lq + q,
                 lbuf, kbuf);
      }
      free(lbuf); free(kbuf);
    }
  /* fill pruned rows from their donors (C9) */
#pragma omp parallel for collapse(2)
  for (int bh = 0; bh < BH; ++bh)
    for (int t = 0; t < L; ++t) {
      int dn = donor[(size_t)bh * L + t];
      int b = token_block(g, t);
      if (dn != t && b >= qb0 && b < qb1)
        memcpy(O + ((size_t)bh * L + t) * d, O + ((size_t)bh * L + dn) * d, sizeof(double) * d);
    }
  free(kept_off);
}

void or_attn_fwd(const or_geom* g, double r, int BH, int d, const double* Q, const double* K, const double* V,
                 const int* kept_tok, const int* donor, const int* q2k_num, const int* q2k_idx, double scale,
                 double* O, double* lse) {
  or_attn_fwd_range(g, r, BH, d, Q, K, V, kept_tok, donor, q2k_num, q2k_idx, scale, O, lse, 0, or_num_blocks(g));
}

/* Forward for a sample of kept rows only (parity at full size): rows[n] = bh * Lq + packed index.
 * Writes O^s rows to Os[n*d] and lse[n]. */
void or_attn_fwd_rows(const or_geom* g, double r, int BH, int d, const double* Q, const double* K,
                      const double* V, const int* kept_tok, const int* q2k_num, const int* q2k_idx,
                      double scale, int nrows, const int* rows, double* Os, double* lse) {
  int N = or_num_blocks(g), L = g->T * g->H * g->W, Lq;
  int* kept_off = (int*)malloc(sizeof(int) * (N + 1));
  kept_off[0] = 0;
  for (int b = 0; b < N; ++b) kept_off[b + 1] = kept_off[b] + block_kept(g, r, b);
  Lq = kept_off[N];
  (void)BH;
#pragma omp parallel for schedule(dynamic)
  for (int n = 0; n < nrows; ++n) {
    int bh = rows[n] / Lq, q = rows[n] % Lq, i = 0;
    while (kept_off[i + 1] <= q) ++i;
    double* lbuf = (double*)malloc(sizeof(double) * L);
    int* kbuf = (int*)malloc(sizeof(int) * L);
    size_t row = (size_t)bh * N + i;
    attn_row(g, d, Q + (size_t)bh * L * d, K + (size_t)bh * L * d, V + (size_t)bh * L * d,
             kept_tok[(size_t)bh * Lq + q], q2k_idx + row * N, q2k_num[row], scale, Os + (size_t)n * d, lse + n,
             lbuf, kbuf);
    free(lbuf); free(kbuf);
  }
  free(kept_off);
}

/* Sparse attention backward (a8; semantics derived, C10: selection is piecewise constant).
 *   dO^s[q] = dO[q] + sum_{t : donor(t) = q, t != q} dO[t]       (gradient of the fill)
 *   D[q]    = sum_c dO^s[q][c] O^s[q][c]
 *   P_qk    = exp(scale q.k - LSE[q])
 *   dV[k]  += P_qk dO^s[q];  dP_qk = dO^s[q].v_k;  dS_qk = P_qk (dP_qk - D[q])
 *   dQ[q]   = scale sum_k dS_qk k      (kept q; pruned rows of dQ are 0)
 *   dK[k]  += scale dS_qk q            (keys never admitted get 0)
 * Pass 1 (parallel over query blocks) computes O^s, LSE, D and dQ; pass 2 (parallel over KV blocks
 * j) sums dK_j, dV_j over the admitting query blocks in ascending (block, row) order. */
void or_attn_bwd_range(const or_geom* g, double r, int BH, int d, const double* Q, const double* K,
                       const double* V, const double* dO, const int* kept_tok, const int* donor, const int* q2k_num,
                       const int* q2k_idx, double scale, double* dQ, double* dK, double* dV, int qb0, int qb1) {
  int N = or_num_blocks(g), L = g->T * g->H * g->W, Lq;
  int* kept_off = (int*)malloc(sizeof(int) * (N + 1));
  kept_off[0] = 0;
  for (int b = 0; b < N; ++b) kept_off[b + 1] = kept_off[b] + block_kept(g, r, b);
  Lq = kept_off[N];
  double* dOs = (double*)malloc(sizeof(double) * (size_t)BH * Lq * d);
  double* Dv = (double*)malloc(sizeof(double) * (size_t)BH * Lq);
  double* lse = (double*)malloc(sizeof(double) * (size_t)BH * Lq);
  memset(dQ, 0, sizeof(double) * (size_t)BH * L * d);
  memset(dK, 0, sizeof(double) * (size_t)BH * L * d);
  memset(dV, 0, sizeof(double) * (size_t)BH * L * d);
  /* pass 1: per kept row: O^s, LSE, dO^s, D, dQ */
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int bh = 0; bh < BH; ++bh)
    for (int i = qb0; i < qb1; ++i) {
      const double *Qh = Q + (size_t)bh * L * d, *Kh = K + (size_t)bh * L * d, *Vh = V + (size_t)bh * L * d;
      double* lbuf = (double*)malloc(sizeof(double) * L);
      int* kbuf = (int*)malloc(sizeof(int) * L);
      int* btok = (int*)malloc(sizeof(int) * g->ct * g->ch * g->cw);
      double* os = (double*)malloc(sizeof(double) * d);
      size_t row = (size_t)bh * N + i;
      int nb = block_tokens(g, i, btok);
      for (int q = kept_off[i]; q < kept_off[i + 1]; ++q) {
        int tok = kept_tok[(size_t)bh * Lq + q];
        double* lq = lse + (size_t)bh * Lq + q;
        attn_row(g, d, Qh, Kh, Vh, tok, q2k_idx + row * N, q2k_num[row], scale, os, lq, lbuf, kbuf);
        double* g_ = dOs + ((size_t)bh * Lq + q) * d;
        for (int c = 0; c < d; ++c) g_[c] = dO[((size_t)bh * L + tok) * d + c];
        for (int a = 0; a < nb; ++a) {
          int t = btok[a];
          if (t != tok && donor[(size_t)bh * L + t] == tok)
            for (int c = 0; c < d; ++c) g_[c] += dO[((size_t)bh * L + t) * d + c];
        }
        double Dq = dotd(g_, os, d);
        Dv[(size_t)bh * Lq + q] = Dq;
        /* dQ row */
        int nk = 0;
        for (int a = 0; a < q2k_num[row]; ++a) nk += block_tokens(g, q2k_idx[row * N + a], kbuf + nk);
        double* dq = dQ + ((size_t)bh * L + tok) * d;
        const double* qv = Qh + (size_t)tok * d;
        for (int t = 0; t < nk; ++t) {
          const double* kv = Kh + (size_t)kbuf[t] * d;
          double P = exp(scale * dotd(qv, kv, d) - *lq);
          double dP = dotd(g_, Vh + (size_t)kbuf[t] * d, d);
          double dS = P * (dP - Dq);
          for (int c = 0; c < d; ++c) dq[c] += scale * dS * kv[c];
        }
      }
      free(lbuf); free(kbuf); free(btok); free(os);
    }
  /* pass 2: per KV block j: dK_j, dV_j over admitting query blocks (ascending i, ascending row) */
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int bh = 0; bh < BH; ++bh)
    for (int j = 0; j < N; ++j) {
      const double *Qh = Q + (size_t)bh * L * d, *Kh = K + (size_t)bh * L * d, *Vh = V + (size_t)bh * L * d;
      int* ktok = (int*)malloc(sizeof(int) * g->ct * g->ch * g->cw);
      int nk = block_tokens(g, j, ktok);
      for (int i = qb0; i < qb1; ++i) {
        size_t row = (size_t)bh * N + i;
        int adm = 0;
        for (int a = 0; a < q2k_num[row]; ++a) if (q2k_idx[row * N + a] == j) adm = 1;
        if (!adm) continue;
        for (int q = kept_off[i]; q < kept_off[i + 1]; ++q) {
          int tok = kept_tok[(size_t)bh * Lq + q];
          const double* qv = Qh + (size_t)tok * d;
          const double* g_ = dOs + ((size_t)bh * Lq + q) * d;
          double lq = lse[(size_t)bh * Lq + q], Dq = Dv[(size_t)bh * Lq + q];
          for (int t = 0; t < nk; ++t) {
            const double* kv = Kh + (size_t)ktok[t] * d;
            double P = exp(scale * dotd(qv, kv, d) - lq);
            double dP = dotd(g_, Vh + (size_t)ktok[t] * d, d);
            double dS = P * (dP - Dq);
            double* dv = dV + ((size_t)bh * L + ktok[t]) * d;
            double* dk = dK + ((size_t)bh * L + ktok[t]) * d;
            for (int c = 0; c < d; ++c) { dv[c] += P * g_[c]; dk[c] += scale * dS * qv[c]; }
          }
        }
      }
      free(ktok);
    }
  free(dOs); free(Dv); free(lse); free(kept_off);
}

void or_attn_bwd(const or_geom* g, double r, int BH, int d, const double* Q, const double* K, const double* V,
                 const double* dO, const int* kept_tok, const int* donor, const int* q2k_num, const int* q2k_idx,
                 double scale, double* dQ, double* dK, double* dV) {
  or_attn_bwd_range(g, r, BH, d, Q, K, V, dO, kept_tok, donor, q2k_num, q2k_idx, scale, dQ, dK, dV, 0,
                    or_num_blocks(g));
}

int or_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
void or_set_threads(int n) {
#ifdef _OPENMP
  omp_set_num_threads(n);
#else
  (void)n;
#endif
}
