/*
 * gd_oracle.c -- TEST INFRASTRUCTURE ONLY.  CPU oracle for parity checks.
 *
 * Plain-C restatement of the reference GeoDock-MA pose-search path
 * (/root/reference/proj/include/geodock/, fp64) plus the north-star
 * extension E1-E8 defined in DESIGN.md.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this; the
 * product (paper_1901_06363_b200) never does.
 *
 * Pinning: tests/test_oracle_cpu.py checks this file against the reference
 * KATs (test_geometry.cpp, test_kernel.cpp) and against golden vectors that
 * oracle/_ref (the reference headers compiled here, see oracle/Makefile)
 * produced, committed under tests/golden/.
 *
 * Build flags matter: -O2 -ffp-contract=off, no -march (no FMA), exactly
 * like the reference Release build plus -ffp-contract=off.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "geodock_b200.h"

#define MIN_DIST_SQ 1e-12   /* geometry.hpp:33 */
#define BUMP_SCALE 0.8      /* geometry.hpp:37 */
#define BUMP_GRAPH_DIST 4   /* geometry.hpp:40 */
#define MIN_AXIS_LEN 1e-9   /* geometry.hpp:43 */
#define DIST_CAP 4          /* molecule.hpp:43 */

/* distance_sq (vec3.hpp:44): ((dx*dx + dy*dy) + dz*dz). */
static double dsq(const double* a, const double* b) {
  const double dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
  return dx * dx + dy * dy + dz * dz;
}

/* overlap_score (geometry.hpp:140-155), brute force. */
double gdo_overlap_score(const double* xyz, int n, const double* pocket, int P) {
  double sum = 0.0;
  for (int i = 0; i < n; ++i) {
    double m = INFINITY;
    for (int j = 0; j < P; ++j) {
      const double d = dsq(xyz + 3 * i, pocket + 3 * j);
      if (d < m) m = d; /* std::min(m, d) */
    }
    sum += (MIN_DIST_SQ < m) ? m : MIN_DIST_SQ; /* std::max(kMin, m) */
  }
  return (double)n / sum;
}

/* ---------------------------------------------------------------------------
 * Ligand graph (molecule.hpp:45-301).
 * ------------------------------------------------------------------------- */
typedef struct {
  int n, nfrag, status;
  uint8_t* capped;  /* n*n */
  double* radii;    /* n (borrowed) */
  int *faxis, *fanchor, *fsize;
  double* frel;
  char* member;     /* nfrag*n */
} olig;

typedef struct {
  int lo, hi, bond;
} orot;

static int cmp_rot(const void* a, const void* b) {
  const orot* x = (const orot*)a;
  const orot* y = (const orot*)b;
  if (x->lo != y->lo) return x->lo < y->lo ? -1 : 1;
  if (x->hi != y->hi) return x->hi < y->hi ? -1 : 1;
  return 0;
}

static void olig_free(olig* L) {
  free(L->capped);
  free(L->faxis);
  free(L->fanchor);
  free(L->fsize);
  free(L->frel);
  free(L->member);
  memset(L, 0, sizeof *L);
}

/* Returns 0 or GD_LIG_INVALID.  Adjacency is a dense n*n bond-index table. */
static int olig_build(olig* L, int n, const double* xyz, double* radii, int nb, const int32_t* bonds,
                      const uint8_t* rot) {
  memset(L, 0, sizeof *L);
  L->n = n;
  L->radii = radii;
  if (n < 2) return L->status = GD_LIG_INVALID;
  for (int i = 0; i < n; ++i) {
    if (!(radii[i] > 0.0)) return L->status = GD_LIG_INVALID;
    if (!isfinite(xyz[3 * i]) || !isfinite(xyz[3 * i + 1]) || !isfinite(xyz[3 * i + 2]))
      return L->status = GD_LIG_INVALID;
  }
  int* adj = (int*)malloc(sizeof(int) * n * n);
  for (int i = 0; i < n * n; ++i) adj[i] = -1;
  for (int b = 0; b < nb; ++b) {
    const int a0 = bonds[2 * b], a1 = bonds[2 * b + 1];
    if (a0 == a1 || a0 < 0 || a1 < 0 || a0 >= n || a1 >= n || adj[a0 * n + a1] >= 0) {
      free(adj);
      return L->status = GD_LIG_INVALID;
    }
    adj[a0 * n + a1] = adj[a1 * n + a0] = b;
  }
  /* Full BFS distances (an independent derivation, like bump_oracle,
   * tests/support/oracles.hpp:51-81), then capped. */
  int* q = (int*)malloc(sizeof(int) * n);
  int* dist = (int*)malloc(sizeof(int) * n);
  L->capped = (uint8_t*)malloc((size_t)n * n);
  for (int src = 0; src < n; ++src) {
    for (int i = 0; i < n; ++i) dist[i] = -1;
    int h = 0, t = 0;
    q[t++] = src;
    dist[src] = 0;
    while (h < t) {
      const int at = q[h++];
      for (int nb2 = 0; nb2 < n; ++nb2)
        if (adj[at * n + nb2] >= 0 && dist[nb2] < 0) {
          dist[nb2] = dist[at] + 1;
          q[t++] = nb2;
        }
    }
    if (src == 0 && t != n) { /* disconnected */
      free(adj), free(q), free(dist);
      return L->status = GD_LIG_INVALID;
    }
    for (int j = 0; j < n; ++j) L->capped[src * n + j] = (uint8_t)(dist[j] > DIST_CAP ? DIST_CAP : dist[j]);
  }
  /* Rotamers: rotatable bonds whose removal disconnects the graph. */
  orot* rots = (orot*)malloc(sizeof(orot) * (nb > 0 ? nb : 1));
  int nr = 0;
  char* seen = (char*)malloc(n);
  for (int b = 0; b < nb; ++b) {
    if (!rot[b]) continue;
    const int a0 = bonds[2 * b], a1 = bonds[2 * b + 1];
    memset(seen, 0, n);
    int h = 0, t = 0;
    q[t++] = a0;
    seen[a0] = 1;
    while (h < t) {
      const int at = q[h++];
      for (int nb2 = 0; nb2 < n; ++nb2) {
        const int bb = adj[at * n + nb2];
        if (bb < 0 || bb == b || seen[nb2]) continue;
        seen[nb2] = 1;
        q[t++] = nb2;
      }
    }
    if (!seen[a1]) {
      rots[nr].lo = a0 < a1 ? a0 : a1;
      rots[nr].hi = a0 < a1 ? a1 : a0;
      rots[nr].bond = b;
      ++nr;
    }
  }
  qsort(rots, nr, sizeof(orot), cmp_rot);
  L->nfrag = 2 * nr;
  L->faxis = (int*)malloc(sizeof(int) * (L->nfrag + 1));
  L->fanchor = (int*)malloc(sizeof(int) * (L->nfrag + 1));
  L->fsize = (int*)malloc(sizeof(int) * (L->nfrag + 1));
  L->frel = (double*)malloc(sizeof(double) * (L->nfrag + 1));
  L->member = (char*)malloc((size_t)(L->nfrag + 1) * n);
  for (int r = 0; r < nr; ++r) {
    char* left = L->member + (size_t)(2 * r) * n;
    char* right = L->member + (size_t)(2 * r + 1) * n;
    memset(left, 0, n);
    int h = 0, t = 0;
    q[t++] = rots[r].lo;
    left[rots[r].lo] = 1;
    while (h < t) {
      const int at = q[h++];
      for (int nb2 = 0; nb2 < n; ++nb2) {
        const int bb = adj[at * n + nb2];
        if (bb < 0 || bb == rots[r].bond || left[nb2]) continue;
        left[nb2] = 1;
        q[t++] = nb2;
      }
    }
    int ls = 0;
    for (int i = 0; i < n; ++i) {
      right[i] = !left[i];
      ls += left[i];
    }
    L->fsize[2 * r] = ls;
    L->fsize[2 * r + 1] = n - ls;
    L->frel[2 * r] = (double)ls / n;
    L->frel[2 * r + 1] = (double)(n - ls) / n;
    L->faxis[2 * r] = rots[r].lo;
    L->fanchor[2 * r] = rots[r].hi;
    L->faxis[2 * r + 1] = rots[r].hi;
    L->fanchor[2 * r + 1] = rots[r].lo;
  }
  free(rots), free(seen), free(adj), free(q), free(dist);
  return L->status = 0;
}

/* ---------------------------------------------------------------------------
 * Geometry (geometry.hpp:161-213).
 * ------------------------------------------------------------------------- */
/* rotate_fragment_into; returns 0, or GD_LIG_DEGENERATE. */
static int rotate_into(const olig* L, const double* pose, int f, double angle_deg, double* out) {
  const int n = L->n;
  const double* o = pose + 3 * L->faxis[f];
  const double* an = pose + 3 * L->fanchor[f];
  const double ax = an[0] - o[0], ay = an[1] - o[1], az = an[2] - o[2];
  const double len = sqrt(ax * ax + ay * ay + az * az);
  if (len < MIN_AXIS_LEN) return GD_LIG_DEGENERATE;
  const double kx = ax / len, ky = ay / len, kz = az / len;
  memcpy(out, pose, sizeof(double) * 3 * n);
  if (angle_deg == 0.0) return 0;
  const double theta = angle_deg * (M_PI / 180.0);
  const double c = cos(theta);
  const double s = sin(theta);
  const char* mem = L->member + (size_t)f * n;
  for (int i = 0; i < n; ++i) {
    if (!mem[i]) continue;
    const double vx = pose[3 * i] - o[0], vy = pose[3 * i + 1] - o[1], vz = pose[3 * i + 2] - o[2];
    const double crx = ky * vz - kz * vy, cry = kz * vx - kx * vz, crz = kx * vy - ky * vx;
    const double w = (kx * vx + ky * vy + kz * vz) * (1.0 - c);
    out[3 * i] = o[0] + vx * c + crx * s + kx * w;
    out[3 * i + 1] = o[1] + vy * c + cry * s + ky * w;
    out[3 * i + 2] = o[2] + vz * c + crz * s + kz * w;
  }
  return 0;
}

/* check_bumps: 1 = feasible. */
static int bumps_ok(const olig* L, const double* pose, int f) {
  const int n = L->n;
  const char* mem = L->member + (size_t)f * n;
  for (int i = 0; i < n; ++i) {
    if (!mem[i]) continue;
    for (int j = 0; j < n; ++j) {
      if (mem[j] || L->capped[i * n + j] < BUMP_GRAPH_DIST) continue;
      const double cut = BUMP_SCALE * (L->radii[i] + L->radii[j]);
      if (dsq(pose + 3 * i, pose + 3 * j) < cut * cut) return 0;
    }
  }
  return 1;
}

/* ---------------------------------------------------------------------------
 * Search (kernel.hpp:62-248).
 * ------------------------------------------------------------------------- */
int gdo_optimal_tile_size(int step) {
  long best = -1;
  int tile = 0;
  for (int x = 360; x >= 1; --x) { /* tile_size_oracle, oracles.hpp:86-98 */
    if (360 % x) continue;
    const long v = (long)step * (360 / x) + x;
    if (best < 0 || v <= best) {
      best = v;
      tile = x;
    }
  }
  return tile;
}

typedef struct {
  const olig* L;
  const double* pocket;
  int P;
  double* scratch;
  long long evals, checks;
  int err;
  int last_angle; /* committed angle of the last flat/refined search */
} osearch;

/* CandidateEvaluator::evaluate; returns 0 if infeasible (score untouched). */
static int evaluate(osearch* S, const double* entry, int f, int angle, double* score) {
  ++S->checks;
  const double* cand = entry;
  if (angle != 0) {
    const int rc = rotate_into(S->L, entry, f, (double)angle, S->scratch);
    if (rc) {
      S->err = rc;
      return 0;
    }
    if (!bumps_ok(S->L, S->scratch, f)) return 0;
    cand = S->scratch;
  }
  ++S->evals;
  *score = gdo_overlap_score(cand, S->L->n, S->pocket, S->P);
  return 1;
}

static void commit(osearch* S, double* pose, int f, int angle) {
  if (angle == 0) return;
  const int rc = rotate_into(S->L, pose, f, (double)angle, S->scratch);
  if (rc) S->err = rc;
  else memcpy(pose, S->scratch, sizeof(double) * 3 * S->L->n);
}

static double flat(osearch* S, double* pose, int f, int step) {
  int best_a = 0, have = 0;
  double best = 0.0, sc;
  for (int a = 0; a < 360; a += step) {
    if (!evaluate(S, pose, f, a, &sc)) {
      if (S->err) return 0.0;
      continue;
    }
    if (!have || sc > best) {
      best = sc;
      best_a = a;
      have = 1;
    }
  }
  S->last_angle = best_a;
  commit(S, pose, f, best_a);
  return best;
}

static double refined(osearch* S, double* pose, int f, int hp, double entry_score) {
  const int T = gdo_optimal_tile_size(hp), tc = 360 / T;
  int have = 0, best_a = 0, wt = -1;
  double best = 0.0, ws = 0.0, sc;
  for (int t = 0; t < tc; ++t) {
    const int a = t * T + T / 2;
    if (!evaluate(S, pose, f, a, &sc)) {
      if (S->err) return 0.0;
      continue;
    }
    if (!have || sc > best) {
      best = sc;
      best_a = a;
      have = 1;
    }
    if (wt < 0 || sc > ws) {
      wt = t;
      ws = sc;
    }
  }
  if (wt >= 0) {
    const int start = wt * T;
    for (int k = 0; (k + 1) * hp <= T; ++k) {
      const int a = start + k * hp;
      if (!evaluate(S, pose, f, a, &sc)) {
        if (S->err) return 0.0;
        continue;
      }
      if (!have || sc > best) {
        best = sc;
        best_a = a;
        have = 1;
      }
    }
  }
  ++S->checks;
  if (!have || entry_score > best) {
    best = entry_score;
    best_a = 0;
  }
  S->last_angle = best_a;
  commit(S, pose, f, best_a);
  return best;
}

/* match_probes_shape (kernel.hpp:205-248); pose in/out.  Returns 0 or a
 * GD_LIG_* error. */
static int mps(const olig* L, const double* pocket, int P, const gd_knobs* k, double* pose,
               double* score, long long* evals, long long* checks) {
  osearch S = {L, pocket, P, (double*)malloc(sizeof(double) * 3 * L->n), 1, 1, 0, 0};
  double cur = gdo_overlap_score(pose, L->n, pocket, P);
  for (int rep = 0; rep < k->repetitions && !S.err; ++rep)
    for (int f = 0; f < L->nfrag && !S.err; ++f) {
      if (L->frel[f] <= k->threshold) cur = flat(&S, pose, f, k->low_precision_step);
      else if (k->enable_refinement) cur = refined(&S, pose, f, k->high_precision_step, cur);
      else cur = flat(&S, pose, f, k->high_precision_step);
    }
  free(S.scratch);
  *score = cur;
  *evals = S.evals;
  *checks = S.checks;
  return S.err;
}

/* ---------------------------------------------------------------------------
 * Extension E1..E8 (no reference implementation exists).
 * ------------------------------------------------------------------------- */
typedef struct {
  long long key[9];
  int idx;
} okey;

static int cmp_key(const void* a, const void* b) {
  const okey* x = (const okey*)a;
  const okey* y = (const okey*)b;
  for (int e = 0; e < 9; ++e)
    if (x->key[e] != y->key[e]) return x->key[e] < y->key[e] ? -1 : 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

static int cmp_int(const void* a, const void* b) {
  const int x = *(const int*)a, y = *(const int*)b;
  return x < y ? -1 : (x > y);
}

/* E2: distinct orientations; returns the count (idx, R malloc-ed). */
int gdo_orientations(int step, int** idx_out, double** R_out) {
  double cs[360], sn[360];
  for (int a = 0; a < 360; ++a) {
    const double th = (double)a * (M_PI / 180.0);
    cs[a] = cos(th);
    sn[a] = sin(th);
  }
  const int m = 360 / step, total = m * m * m;
  double* all = (double*)malloc(sizeof(double) * 9 * total);
  okey* keys = (okey*)malloc(sizeof(okey) * total);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j)
      for (int k = 0; k < m; ++k) {
        const int idx = (i * m + j) * m + k;
        const double ca = cs[i * step], sa = sn[i * step], cb = cs[j * step], sb = sn[j * step],
                     cg = cs[k * step], sg = sn[k * step];
        double* r = all + 9 * idx;
        r[0] = cg * cb;
        r[1] = cg * sb * sa - sg * ca;
        r[2] = cg * sb * ca + sg * sa;
        r[3] = sg * cb;
        r[4] = sg * sb * sa + cg * ca;
        r[5] = sg * sb * ca - cg * sa;
        r[6] = -sb;
        r[7] = cb * sa;
        r[8] = cb * ca;
        for (int e = 0; e < 9; ++e) keys[idx].key[e] = llround(r[e] * 1e6);
        keys[idx].idx = idx;
      }
  qsort(keys, total, sizeof(okey), cmp_key);
  int* idx = (int*)malloc(sizeof(int) * total);
  int cnt = 0;
  for (int t = 0; t < total; ++t)
    if (t == 0 || memcmp(keys[t].key, keys[t - 1].key, sizeof keys[t].key) != 0) idx[cnt++] = keys[t].idx;
  qsort(idx, cnt, sizeof(int), cmp_int);
  double* R = (double*)malloc(sizeof(double) * 9 * cnt);
  for (int t = 0; t < cnt; ++t) memcpy(R + 9 * t, all + 9 * idx[t], 9 * sizeof(double));
  free(all), free(keys);
  *idx_out = idx;
  *R_out = R;
  return cnt;
}

void gdo_free(void* p) { free(p); }

/* E1: pocket centre, index-order sum. */
void gdo_pocket_centre(const double* pocket, int P, double c[3]) {
  double sx = 0.0, sy = 0.0, sz = 0.0;
  for (int j = 0; j < P; ++j) {
    sx += pocket[3 * j];
    sy += pocket[3 * j + 1];
    sz += pocket[3 * j + 2];
  }
  c[0] = sx / P;
  c[1] = sy / P;
  c[2] = sz / P;
}

/* E3: p' = c + R (p - c). */
static void rigid_pose(const double* xyz, int n, const double* R, const double* c, double* out) {
  for (int i = 0; i < n; ++i) {
    const double vx = xyz[3 * i] - c[0], vy = xyz[3 * i + 1] - c[1], vz = xyz[3 * i + 2] - c[2];
    out[3 * i] = c[0] + (R[0] * vx + R[1] * vy + R[2] * vz);
    out[3 * i + 1] = c[1] + (R[3] * vx + R[4] * vy + R[5] * vz);
    out[3 * i + 2] = c[2] + (R[6] * vx + R[7] * vy + R[8] * vz);
  }
}

typedef struct {
  double s;
  int i;
} oent;

/* (score desc, index asc) */
static int cmp_ent(const void* a, const void* b) {
  const oent* x = (const oent*)a;
  const oent* y = (const oent*)b;
  if (x->s != y->s) return x->s > y->s ? -1 : 1;
  return x->i < y->i ? -1 : (x->i > y->i);
}

typedef struct {
  const gd_ligand_batch* b;
  const double* pocket;
  int P;
  double centre[3];
  const gd_knobs* k;
  int n_orient;
  const int* oidx;
  const double* oR;
  gd_result* r;
  int K;
  int next;
  pthread_mutex_t mu;
} ojob;

static void dock_one(ojob* J, int l) {
  const gd_ligand_batch* b = J->b;
  const int a0 = b->atom_offsets[l], n = b->atom_offsets[l + 1] - a0;
  const int b0 = b->bond_offsets[l], nb = b->bond_offsets[l + 1] - b0;
  const int K = J->K;
  gd_result* r = J->r;
  for (int e = 0; e < K; ++e) {
    const size_t d = (size_t)l * K + e;
    if (r->orientation) r->orientation[d] = -2;
    if (r->seed_rank) r->seed_rank[d] = 0;
    if (r->rigid_score) r->rigid_score[d] = 0.0;
    if (r->final_score) r->final_score[d] = 0.0;
    if (r->evaluations) r->evaluations[d] = 0;
    if (r->feasibility_checks) r->feasibility_checks[d] = 0;
    if (r->final_pose && n > 0) memset(r->final_pose + 3 * ((size_t)K * a0 + (size_t)e * n), 0, sizeof(double) * 3 * n);
  }
  if (r->k_eff) r->k_eff[l] = 0;
  if (r->poses_scored) r->poses_scored[l] = 0;
  olig L;
  double* radii = (double*)malloc(sizeof(double) * (n > 0 ? n : 1));
  if (n > 0) memcpy(radii, b->radii + a0, sizeof(double) * n);
  if (olig_build(&L, n, b->xyz + 3 * a0, radii, nb, b->bonds + 2 * b0, b->bond_rotatable + b0)) {
    if (r->status) r->status[l] = GD_LIG_INVALID;
    olig_free(&L);
    free(radii);
    return;
  }
  const int rigid = J->k->rigid_step > 0;
  int k_eff = 1;
  oent* seeds;
  double* pose = (double*)malloc(sizeof(double) * 3 * n);
  if (rigid) {
    oent* all = (oent*)malloc(sizeof(oent) * J->n_orient);
    for (int o = 0; o < J->n_orient; ++o) {
      rigid_pose(b->xyz + 3 * a0, n, J->oR + 9 * o, J->centre, pose);
      all[o].s = gdo_overlap_score(pose, n, J->pocket, J->P);
      all[o].i = o;
    }
    qsort(all, J->n_orient, sizeof(oent), cmp_ent); /* E5 */
    k_eff = K < J->n_orient ? K : J->n_orient;
    seeds = all;
  } else {
    seeds = (oent*)malloc(sizeof(oent));
    seeds[0].s = gdo_overlap_score(b->xyz + 3 * a0, n, J->pocket, J->P);
    seeds[0].i = -1;
  }
  /* E6: one match_probes_shape chain per seed, in rank order. */
  oent* fin = (oent*)malloc(sizeof(oent) * k_eff);
  long long* ev = (long long*)malloc(sizeof(long long) * k_eff);
  long long* ck = (long long*)malloc(sizeof(long long) * k_eff);
  double* poses = (double*)malloc(sizeof(double) * 3 * n * k_eff);
  long long scored = rigid ? J->n_orient : 0;
  int err = 0;
  for (int s = 0; s < k_eff && !err; ++s) {
    double* ps = poses + 3 * (size_t)n * s;
    if (rigid) rigid_pose(b->xyz + 3 * a0, n, J->oR + 9 * seeds[s].i, J->centre, ps);
    else memcpy(ps, b->xyz + 3 * a0, sizeof(double) * 3 * n);
    err = mps(&L, J->pocket, J->P, J->k, ps, &fin[s].s, &ev[s], &ck[s]);
    fin[s].i = s;
    scored += ev[s];
  }
  if (err) {
    if (r->status) r->status[l] = err;
  } else {
    qsort(fin, k_eff, sizeof(oent), cmp_ent); /* E7 */
    for (int e = 0; e < k_eff; ++e) {
      const int s = fin[e].i;
      const size_t d = (size_t)l * K + e;
      if (r->orientation) r->orientation[d] = rigid ? J->oidx[seeds[s].i] : -1;
      if (r->seed_rank) r->seed_rank[d] = s;
      if (r->rigid_score) r->rigid_score[d] = seeds[s].s;
      if (r->final_score) r->final_score[d] = fin[e].s;
      if (r->evaluations) r->evaluations[d] = ev[s];
      if (r->feasibility_checks) r->feasibility_checks[d] = ck[s];
      if (r->final_pose)
        memcpy(r->final_pose + 3 * ((size_t)K * a0 + (size_t)e * n), poses + 3 * (size_t)n * s,
               sizeof(double) * 3 * n);
    }
    if (r->k_eff) r->k_eff[l] = k_eff;
    if (r->poses_scored) r->poses_scored[l] = scored;
    if (r->status) r->status[l] = 0;
  }
  free(fin), free(ev), free(ck), free(poses), free(pose), free(seeds), free(radii);
  olig_free(&L);
}

static void* worker(void* arg) {
  ojob* J = (ojob*)arg;
  for (;;) {
    pthread_mutex_lock(&J->mu);
    const int l = J->next++;
    pthread_mutex_unlock(&J->mu);
    if (l >= J->b->n_ligands) return NULL;
    dock_one(J, l);
  }
}

/* The whole E1-E8 path over a batch, same layout as gd_dock_batch. */
int gdo_dock_batch(const gd_ligand_batch* b, const double* pocket, int P, const gd_knobs* k,
                   int threads, gd_result* r) {
  ojob J;
  memset(&J, 0, sizeof J);
  J.b = b;
  J.pocket = pocket;
  J.P = P;
  J.k = k;
  J.r = r;
  J.K = k->rigid_step > 0 ? k->top_k : 1;
  gdo_pocket_centre(pocket, P, J.centre);
  int* oidx = NULL;
  double* oR = NULL;
  if (k->rigid_step > 0) J.n_orient = gdo_orientations(k->rigid_step, &oidx, &oR);
  J.oidx = oidx;
  J.oR = oR;
  pthread_mutex_init(&J.mu, NULL);
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, worker, &J);
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  pthread_mutex_destroy(&J.mu);
  free(oidx), free(oR);
  return 0;
}

/* Single-chain entry points for fine-grained parity tests. */
int gdo_match_probes_shape(int n, const double* xyz, const double* radii, int nb, const int32_t* bonds,
                           const uint8_t* rot, const double* pocket, int P, const gd_knobs* k,
                           double* pose_out, double* score, long long* evals, long long* checks) {
  olig L;
  double* rad = (double*)malloc(sizeof(double) * (n > 0 ? n : 1));
  if (n > 0) memcpy(rad, radii, sizeof(double) * n);
  int rc = olig_build(&L, n, xyz, rad, nb, bonds, rot);
  if (rc == 0) {
    memcpy(pose_out, xyz, sizeof(double) * 3 * n);
    rc = mps(&L, pocket, P, k, pose_out, score, evals, checks);
  }
  olig_free(&L);
  free(rad);
  return rc;
}

/* optimize_fragment_flat (mode 0) / optimize_fragment_refined (mode 1) on
 * fragment f of the given pose (kernel.hpp:125-198); entry_score < 0 means
 * "not known" (the refined search then scores the entry pose itself). */
int gdo_optimize_fragment(int n, const double* xyz, const double* radii, int nb, const int32_t* bonds,
                          const uint8_t* rot, const double* pocket, int P, const double* pose, int f,
                          int mode, int step, double entry_score, double* pose_out, int* best_angle,
                          double* best_score, long long* evals, long long* checks) {
  olig L;
  double* rad = (double*)malloc(sizeof(double) * (n > 0 ? n : 1));
  if (n > 0) memcpy(rad, radii, sizeof(double) * n);
  int rc = olig_build(&L, n, xyz, rad, nb, bonds, rot);
  if (rc == 0 && (f < 0 || f >= L.nfrag || step < 1 || 360 % step)) rc = GD_LIG_INVALID;
  if (rc == 0) {
    osearch S = {&L, pocket, P, (double*)malloc(sizeof(double) * 3 * n), 0, 0, 0, 0};
    memcpy(pose_out, pose, sizeof(double) * 3 * n);
    const double entry = entry_score >= 0.0 ? entry_score : gdo_overlap_score(pose, n, pocket, P);
    *best_score = mode == 0 ? flat(&S, pose_out, f, step) : refined(&S, pose_out, f, step, entry);
    *best_angle = S.last_angle;
    *evals = S.evals;
    *checks = S.checks;
    rc = S.err;
    free(S.scratch);
  }
  olig_free(&L);
  free(rad);
  return rc;
}

/* Rotate fragment f (reference order) of a ligand by angle_deg. */
int gdo_rotate_fragment(int n, const double* xyz, const double* radii, int nb, const int32_t* bonds,
                        const uint8_t* rot, const double* pose, int f, double angle_deg, double* out,
                        int* feasible) {
  olig L;
  double* rad = (double*)malloc(sizeof(double) * (n > 0 ? n : 1));
  if (n > 0) memcpy(rad, radii, sizeof(double) * n);
  int rc = olig_build(&L, n, xyz, rad, nb, bonds, rot);
  if (rc == 0 && (f < 0 || f >= L.nfrag)) rc = GD_LIG_INVALID;
  if (rc == 0) rc = rotate_into(&L, pose, f, angle_deg, out);
  if (rc == 0 && feasible) *feasible = bumps_ok(&L, out, f);
  olig_free(&L);
  free(rad);
  return rc;
}

/* rotation_profile (analysis.hpp:37-56) of every fragment of one ligand,
 * from the pose `xyz` (reference fragment order): for angle a, valid =
 * check_bumps of the pose with the fragment rotated by a degrees (angle 0 =
 * the pose itself) and score = overlap_score where valid, 0 elsewhere.
 * Writes *nfrag; returns 0, GD_LIG_INVALID, GD_LIG_DEGENERATE (that
 * fragment's profile left all-invalid), or -1 when cap < *nfrag. */
int gdo_rotation_profiles(int n, const double* xyz, const double* radii, int nb,
                          const int32_t* bonds, const uint8_t* rot, const double* pocket, int P,
                          double* scores, uint8_t* valid, double* rel, int cap, int* nfrag) {
  olig L;
  double* rad = (double*)malloc(sizeof(double) * (n > 0 ? n : 1));
  if (n > 0) memcpy(rad, radii, sizeof(double) * n);
  int rc = olig_build(&L, n, xyz, rad, nb, bonds, rot);
  *nfrag = rc == 0 ? L.nfrag : 0;
  if (rc == 0 && L.nfrag > cap) rc = -1;
  double* cand = (double*)malloc(sizeof(double) * 3 * (n > 0 ? n : 1));
  for (int f = 0; rc >= 0 && f < *nfrag; ++f) {
    rel[f] = L.frel[f];
    for (int a = 0; a < 360; ++a) {
      double* sc = scores + 360 * f + a;
      uint8_t* ok = valid + 360 * f + a;
      *sc = 0.0;
      *ok = 0;
      if (rotate_into(&L, xyz, f, (double)a, cand)) {
        rc = GD_LIG_DEGENERATE;
        memset(valid + 360 * f, 0, 360);
        for (int b = 0; b < 360; ++b) scores[360 * f + b] = 0.0;
        break;
      }
      if (!bumps_ok(&L, cand, f)) continue;
      *ok = 1;
      *sc = gdo_overlap_score(cand, n, pocket, P);
    }
  }
  free(cand);
  olig_free(&L);
  free(rad);
  return rc;
}
