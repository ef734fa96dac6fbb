/*
 * semblance_oracle.c — CPU restatement of the reference semblance scan.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path links, loads or
 * calls this file: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg use it, and only as the checker.
 *
 * It restates, in plain C with the reference's fp32/fp64 evaluation order
 * (built with -ffp-contract=off like proj/CMakeLists.txt:15-20), the
 * functions on the hot path of /root/reference/proj/include/velan:
 *
 *   halfpoint h2            traveltime.hpp:16-27   vo_halfpoint
 *   midpoint_of             types.hpp:57-62        vo_midpoint
 *   crs_traveltime          traveltime.hpp:53-56   vo_traveltime_q
 *   hit_for                 traveltime.hpp:66-80   vo_hit_for
 *   interpolate             kernel.hpp:39          vo_interpolate
 *   TraceSweep order        kernel.hpp:61-113      vo_build_sweep
 *   scan_pair_baseline      kernel.hpp:244-270     vo_scan_pair (mode 0)
 *   finalize                kernel.hpp:43-56       vo_finalize
 *   scan_sweep argmax/stack scan.hpp:167-179       vo_run_cells
 *   neighbors_of            crs_pipeline.hpp:162-180 vo_build_sweep
 *   semblance_reference     oracle.hpp:39-113      vo_scan_pair (mode 1)
 *   scan_tile_blocked       kernel.hpp:276-316     vo_worker_blocked (mode 2:
 *                           trace-outer over a tile of (cell, candidate)
 *                           pairs, per-pair order of mode 0, bitwise equal)
 *
 * plus the BASELINE three-parameter CRS operator (vo_traveltime_abc), which
 * has no reference implementation; its evaluation order is fixed in
 * DESIGN.md §3 and shared with the CUDA kernels.  Mode 3 evaluates that
 * operator independently of the fp32 order: the literal BASELINE formula
 * t^2 = (t0 + 2 A dm)^2 + 2 t0 (B dm^2 + C h^2), C = 2 / (t0 v^2), entirely in
 * fp64 (geometry, traveltime, hit, interpolation and sums), the pin of the
 * restated fp32 order.
 *
 * Parity is pinned two ways: against the reference compiled from its own
 * headers (oracle/_ref, built by oracle/Makefile) and against golden
 * fixtures generated from it (tests/golden/make_golden.py).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define VO_OP_NMO 0
#define VO_OP_CRS_D2 1
#define VO_OP_CRS_ABC 2

typedef struct {
  int k1;
  float x;
  int valid;
} vo_hit;

/* traveltime.hpp:16-27: h2 = (dx*dx + dy*dy) * 0.25f, fp32 */
float vo_halfpoint(float sx, float sy, float gx, float gy) {
  const float dx = gx - sx;
  const float dy = gy - sy;
  return (dx * dx + dy * dy) * 0.25f;
}

/* types.hpp:57-62: mean of the first trace's source and receiver */
void vo_midpoint(const float* c4, float* mx, float* my) {
  *mx = (c4[0] + c4[2]) * 0.5f;
  *my = (c4[1] + c4[3]) * 0.5f;
}

/* traveltime.hpp:53-56: sqrt(t0*t0 + (4*h2 + d2) / (v*v)), fp32 */
float vo_traveltime_q(float t0, float h2, float d2, float v) {
  return sqrtf(t0 * t0 + (4.0f * h2 + d2) / (v * v));
}

/* BASELINE CRS operator, DESIGN.md §3.3 (no reference implementation):
 *   qa = (2*A)*dm ; qb = B*(dm*dm) ; qc = (4*h2)/(v*v)
 *   (t0 + qa)^2 + 2 t0 qb + qc = t0^2 + 2 t0 beta + gamma with the per
 *   (trace, candidate) terms beta = qa + qb, gamma = fma(qa, qa, qc):
 *   t = sqrt(t0*t0 + fma(2*t0, beta, gamma))
 * (fmaf is correctly rounded, the GPU's FFMA; everything else is compiled
 * with -ffp-contract=off).  dm = 0 reduces to vo_traveltime_q(t0, h2, 0, v)
 * bit for bit (beta = 0, gamma = qc). */
float vo_traveltime_abc(float t0, float h2, float dm, float A, float B,
                        float v) {
  const float qa = (2.0f * A) * dm;
  const float qb = B * (dm * dm);
  const float qc = (4.0f * h2) / (v * v);
  const float beta = qa + qb;
  const float gamma = fmaf(qa, qa, qc);
  const float t2 = t0 * t0 + fmaf(2.0f * t0, beta, gamma);
  return sqrtf(t2);
}

/* traveltime.hpp:66-80 */
vo_hit vo_hit_for(float t, double dt_s, int ns, int w) {
  vo_hit h;
  const double s = (double)t / dt_s;
  const double base = floor(s);
  /* static_cast<int>(base): x86 cvttsd2si gives INT_MIN when out of range,
   * which the validity test rejects; mirror that explicitly. */
  int ib;
  if (base >= -2147483648.0 && base < 2147483648.0)
    ib = (int)base;
  else
    ib = (int)0x80000000;
  h.k1 = ib - w / 2;
  h.x = (float)(s - base);
  h.valid = h.k1 >= 0 && (long long)h.k1 + w < ns;
  return h;
}

/* kernel.hpp:39 */
float vo_interpolate(float a, float b, float x) { return (b - a) * x + a; }

void vo_finalize(const float* num, int w, float den, float ac, int m_used,
                 float* semblance, float* stack);

/* ------------------------------------------------------------------------ */
/* Sweep construction (TraceSweep, kernel.hpp:61-113; neighbors_of,
 * crs_pipeline.hpp:162-180).                                                */

typedef struct {
  int gather;
  float d2; /* |dm|^2, fp32 (kernel.hpp:88-90)        */
  float dm; /* signed mx offset, ABC operator only     */
  double dmd; /* mode 3: the same offset in fp64          */
  double d2d; /* mode 3: |dm|^2 in fp64                   */
} vo_leg;

typedef struct {
  const float* samples;
  const float* coords;
  const int32_t* ntraces;
  const uint32_t* cdp_id;
  int G, M, ns;
  double dt_s;
  int op, w;
  int n_a, n_b, n_c, ncand;
  const float* a;
  const float* b;
  const float* v;
  double apm;
  int mode; /* 0 = kernel order (scan_pair_baseline), 1 = oracle.hpp sums */
  float* h2;       /* [G][M] */
  float* mx;       /* [G]    */
  float* my;       /* [G]    */
  int* row_gather; /* output row -> input gather */
  double* h2d;     /* mode 3: [G][M] h^2 in fp64 */
  double* mxd;     /* mode 3: [G] midpoint x in fp64 */
  double* myd;
} vo_problem;

static int cmp_cdp_ctx_sort(const void* pa, const void* pb, void* ctx) {
  const uint32_t* id = (const uint32_t*)ctx;
  const int a = *(const int*)pa, b = *(const int*)pb;
  if (id[a] != id[b]) return id[a] < id[b] ? -1 : 1;
  return a < b ? -1 : (a > b ? 1 : 0);
}

/* Simple insertion sort keyed by (cdp_id, index): neighbourhoods are small. */
static void sort_by_cdp(int* idx, int n, const uint32_t* id) {
  for (int i = 1; i < n; ++i) {
    const int key = idx[i];
    int j = i - 1;
    while (j >= 0 && cmp_cdp_ctx_sort(&idx[j], &key, (void*)id) > 0) {
      idx[j + 1] = idx[j];
      --j;
    }
    idx[j + 1] = key;
  }
}

/* Legs of the sweep of output gather g: central first (d2 = 0), then for CRS
 * every non-empty gather in the closed ball |dm| <= apm (double compare),
 * excluding the central one, in cdp_id order.  Returns the leg count. */
static int vo_build_sweep(const vo_problem* p, int g, vo_leg* legs,
                          int* scratch) {
  int n = 0;
  legs[n].gather = g;
  legs[n].d2 = 0.0f;
  legs[n].dm = 0.0f;
  legs[n].dmd = 0.0;
  legs[n].d2d = 0.0;
  ++n;
  if (p->op == VO_OP_NMO) return n;
  int cnt = 0;
  for (int o = 0; o < p->G; ++o) {
    if (o == g || p->ntraces[o] <= 0) continue;
    /* crs_pipeline.hpp:172-173: the difference is taken in fp32, then
     * widened; the ball test itself is double */
    const double dx = (double)(p->mx[o] - p->mx[g]);
    const double dy = (double)(p->my[o] - p->my[g]);
    if (dx * dx + dy * dy <= p->apm * p->apm) scratch[cnt++] = o;
  }
  sort_by_cdp(scratch, cnt, p->cdp_id);
  for (int i = 0; i < cnt; ++i) {
    const int o = scratch[i];
    const float dx = p->mx[o] - p->mx[g];
    const float dy = p->my[o] - p->my[g];
    legs[n].gather = o;
    legs[n].d2 = dx * dx + dy * dy;
    legs[n].dm = dx;
    legs[n].dmd = p->mxd ? p->mxd[o] - p->mxd[g] : (double)dx;
    legs[n].d2d = p->mxd ? legs[n].dmd * legs[n].dmd +
                               (p->myd[o] - p->myd[g]) * (p->myd[o] - p->myd[g])
                         : (double)legs[n].d2;
    ++n;
  }
  return n;
}

/* ------------------------------------------------------------------------ */

typedef struct {
  float semblance;
  float stack;
  int m_used;
} vo_result;

static float vo_moveout(const vo_problem* p, const vo_leg* leg, float t0,
                        float h2, int cand) {
  const int ic = cand % p->n_c;
  const int r = cand / p->n_c;
  const int ib = r % p->n_b;
  const int ia = r / p->n_b;
  if (p->op == VO_OP_CRS_ABC)
    return vo_traveltime_abc(t0, h2, leg->dm, p->a[ia], p->b[ib], p->v[ic]);
  return vo_traveltime_q(t0, h2, leg->d2, p->v[ic]);
}

/* Mode 0: scan_pair_baseline (kernel.hpp:244-270) + finalize
 * (kernel.hpp:43-56), fp32, reference order.  Mode 1: semblance_reference
 * (oracle.hpp:64-113): fp32 windows and column sums, double num_sq/den/
 * linear. */
static vo_result vo_scan_pair(const vo_problem* p, const vo_leg* legs,
                              int nlegs, float t0, int cand, float* num,
                              float* win) {
  const int w = p->w;
  vo_result r = {0.0f, 0.0f, 0};
  float den = 0.0f, ac = 0.0f;
  int m_used = 0;
  double dden = 0.0, dlin = 0.0;
  for (int j = 0; j < w; ++j) num[j] = 0.0f;
  for (int l = 0; l < nlegs; ++l) {
    const int g = legs[l].gather;
    const int M = p->ntraces[g];
    for (int m = 0; m < M; ++m) {
      const float h2 = p->h2[(size_t)g * p->M + m];
      const float t = vo_moveout(p, &legs[l], t0, h2, cand);
      const vo_hit hit = vo_hit_for(t, p->dt_s, p->ns, w);
      if (!hit.valid) continue;
      const float* s =
          p->samples + ((size_t)g * p->M + m) * (size_t)p->ns + hit.k1;
      for (int j = 0; j < w; ++j) {
        const float v = vo_interpolate(s[j], s[j + 1], hit.x);
        if (p->mode == 0) {
          num[j] += v;
          den += v * v;
          ac += v;
        } else {
          win[j] = v;
        }
      }
      if (p->mode == 1) {
        /* column sums in trace order (fp32), squares/linear in double */
        for (int j = 0; j < w; ++j) {
          num[j] += win[j];
          dden += (double)win[j] * win[j];
          dlin += win[j];
        }
      }
      ++m_used;
    }
  }
  r.m_used = m_used;
  if (p->mode == 0) {
    if (den > 0.0f) {
      float sum_sq = 0.0f;
      for (int j = 0; j < w; ++j) sum_sq += num[j] * num[j];
      r.semblance = sum_sq / den;
    }
    if (m_used > 0) r.stack = ac / ((float)m_used * (float)w);
  } else {
    if (m_used == 0) return r;
    double num_sq = 0.0;
    for (int j = 0; j < w; ++j) num_sq += (double)num[j] * num[j];
    if (dden > 0.0) r.semblance = (float)(num_sq / dden);
    r.stack = (float)(dlin / ((double)m_used * w));
  }
  return r;
}

/* Mode 3: the BASELINE CRS operator written literally, all in fp64 — an
 * evaluation independent of the restated fp32 order:
 *   t^2 = (t0 + 2 A dm)^2 + 2 t0 (B dm^2 + C h^2),  C = 2 / (t0 v^2)
 * (t0 = 0: the C h^2 term's limit 2 t0 C h^2 = 4 h^2 / v^2), h^2 and dm from
 * the coordinates in fp64, t0 = k dt, the hit rule of traveltime.hpp:66-80 on
 * the fp64 traveltime, fp64 interpolation (kernel.hpp:39) and fp64 sums
 * (finalize, kernel.hpp:43-56).  NMO and d2 legs use the same fp64 path with
 * t^2 = t0^2 + (4 h^2 + dm^2) / v^2. */
static vo_result vo_scan_pair_f64(const vo_problem* p, const vo_leg* legs,
                                  int nlegs, double t0, int cand, double* num) {
  const int w = p->w;
  vo_result r = {0.0f, 0.0f, 0};
  const int ic = cand % p->n_c;
  const int rr = cand / p->n_c;
  const double v = p->v[ic];
  const double A = p->op == VO_OP_CRS_ABC ? p->a[rr / p->n_b] : 0.0;
  const double B = p->op == VO_OP_CRS_ABC ? p->b[rr % p->n_b] : 0.0;
  double den = 0.0, ac = 0.0;
  int m_used = 0;
  for (int j = 0; j < w; ++j) num[j] = 0.0;
  for (int l = 0; l < nlegs; ++l) {
    const int g = legs[l].gather;
    const double dm = legs[l].dmd;
    const int M = p->ntraces[g];
    for (int m = 0; m < M; ++m) {
      const double hh = p->h2d[(size_t)g * p->M + m];
      double t2;
      if (p->op == VO_OP_CRS_ABC) {
        const double u = t0 + 2.0 * A * dm;
        const double c_h2 = t0 > 0.0 ? 2.0 * t0 * ((2.0 / (t0 * v * v)) * hh)
                                     : 4.0 * hh / (v * v);
        t2 = u * u + 2.0 * t0 * (B * dm * dm) + c_h2;
      } else {
        t2 = t0 * t0 + (4.0 * hh + legs[l].d2d) / (v * v);
      }
      if (!(t2 >= 0.0)) continue; /* NaN traveltime: hit_for rejects it */
      const double s = sqrt(t2) / p->dt_s;
      const double base = floor(s);
      if (!(base >= -2147483648.0 && base < 2147483648.0)) continue;
      const long long k1 = (long long)base - w / 2;
      if (!(k1 >= 0 && k1 + w < p->ns)) continue;
      const double x = s - base;
      const float* tr = p->samples + ((size_t)g * p->M + m) * (size_t)p->ns + k1;
      for (int j = 0; j < w; ++j) {
        const double a0 = tr[j], a1 = tr[j + 1];
        const double val = (a1 - a0) * x + a0;
        num[j] += val;
        den += val * val;
        ac += val;
      }
      ++m_used;
    }
  }
  r.m_used = m_used;
  if (den > 0.0) {
    double sq = 0.0;
    for (int j = 0; j < w; ++j) sq += num[j] * num[j];
    r.semblance = (float)(sq / den);
  }
  if (m_used > 0) r.stack = (float)(ac / ((double)m_used * w));
  return r;
}

/* ------------------------------------------------------------------------ */

typedef struct {
  const vo_problem* p;
  const int32_t* cell_row;
  const int32_t* cell_k;
  int n_cells;
  int32_t* best_idx;
  float* best_s;
  float* best_stack;
  float* matrix;       /* [n_cells][ncand] or NULL */
  float* stack_matrix; /* [n_cells][ncand] or NULL */
  uint64_t valid;
  int next;
  pthread_mutex_t* lock;
} vo_job;

static void* vo_worker(void* arg) {
  vo_job* job = (vo_job*)arg;
  const vo_problem* p = job->p;
  vo_leg* legs = (vo_leg*)malloc(sizeof(vo_leg) * (size_t)(p->G + 1));
  int* scratch = (int*)malloc(sizeof(int) * (size_t)(p->G + 1));
  float* num = (float*)malloc(sizeof(float) * (size_t)p->w);
  float* win = (float*)malloc(sizeof(float) * (size_t)p->w);
  double* numd = (double*)malloc(sizeof(double) * (size_t)p->w);
  uint64_t valid = 0;
  int cached_row = -1, nlegs = 0;
  for (;;) {
    pthread_mutex_lock(job->lock);
    const int i = job->next;
    job->next += 16;
    pthread_mutex_unlock(job->lock);
    if (i >= job->n_cells) break;
    const int iend = i + 16 < job->n_cells ? i + 16 : job->n_cells;
    for (int c = i; c < iend; ++c) {
      const int row = job->cell_row[c];
      const int g = p->row_gather[row];
      if (row != cached_row) {
        nlegs = vo_build_sweep(p, g, legs, scratch);
        cached_row = row;
      }
      const int k = job->cell_k[c];
      const float t0 = (float)(k * p->dt_s); /* scan.hpp:133 */
      int best_c = 0;
      float best = 0.0f, best_st = 0.0f;
      for (int cand = 0; cand < p->ncand; ++cand) {
        const vo_result r =
            p->mode == 3 ? vo_scan_pair_f64(p, legs, nlegs, (double)k * p->dt_s, cand, numd)
                         : vo_scan_pair(p, legs, nlegs, t0, cand, num, win);
        valid += (uint64_t)r.m_used;
        if (job->matrix) job->matrix[(size_t)c * p->ncand + cand] = r.semblance;
        if (job->stack_matrix)
          job->stack_matrix[(size_t)c * p->ncand + cand] = r.stack;
        /* scan.hpp:167-179 / oracle.hpp:141: strict '>', lowest index wins */
        if (cand == 0 || r.semblance > best) {
          best = r.semblance;
          best_c = cand;
          best_st = r.stack;
        }
      }
      job->best_idx[c] = best_c;
      job->best_s[c] = best;
      job->best_stack[c] = best_st;
    }
  }
  pthread_mutex_lock(job->lock);
  job->valid += valid;
  pthread_mutex_unlock(job->lock);
  free(legs);
  free(scratch);
  free(num);
  free(win);
  free(numd);
  return NULL;
}

/* ------------------------------------------------------------------------ */
/* Mode 2: the blocked, trace-outer form (the structure of scan_tile_blocked,
 * kernel.hpp:276-316, applied to any operator): a work item is one output
 * row, a block of up to VO_KB of its requested cells (t0 samples) and a
 * chunk of up to VO_CB candidates; the row's sweep is walked once per item,
 * trace-outer, each trace's moveout terms hoisted over the item's t0 block,
 * and every (cell, candidate) pair accumulates in sweep order exactly as
 * vo_scan_pair mode 0 (scan_pair_baseline) does — so the results are
 * bitwise those of mode 0, only the loop nest (cache locality) differs.
 * Semblance and stack land in a per-(cell, candidate) panel; the argmax
 * runs per cell afterwards with scan.hpp:167-179's rule.                   */

#define VO_KB 16
#define VO_CB 64

/* One trace of a blocked work item: the hits of every (candidate, t0) pair
 * of the item (branch-free over the t0 block, so the compiler vectorises the
 * sqrt / double division / floor), then the windows of the valid ones in
 * scan_pair_baseline's order (kernel.hpp:244-270).  Compiled twice: generic
 * x86-64 and, chosen at run time when the CPU has them, AVX2 + FMA (fmaf is
 * the correctly rounded FMA either way; -ffp-contract=off keeps every other
 * operation unfused). */
#define VO_BLK_TRACE_BODY                                                       \
  const int w = p->w;                                                          \
  const int W2 = w + 2;                                                        \
  const int abc = p->op == VO_OP_CRS_ABC;                                      \
  const double dt = p->dt_s;                                                   \
  const int half = w / 2, ns = p->ns;                                          \
  int k1v[VO_KB];                                                              \
  float xv[VO_KB];                                                             \
  for (int c = 0; c < nc; ++c) {                                               \
    for (int i = 0; i < nk; ++i) {                                             \
      const float t = abc ? sqrtf(t0sq[i] + fmaf(two_t0[i], q0[c], q1[c]))     \
                          : sqrtf(t0sq[i] + q0[c]);                            \
      const double sv = (double)t / dt;                                        \
      double base = floor(sv);                                                 \
      /* out of int range (inf/NaN/huge): invalid, as the INT_MIN cast is */   \
      const int inr = base >= -2147483648.0 && base < 2147483648.0;            \
      const long long kk = inr ? (long long)base - half : -1;                  \
      k1v[i] = (kk >= 0 && kk + w < ns) ? (int)kk : -1;                        \
      xv[i] = (float)(sv - base);                                              \
    }                                                                          \
    for (int i = 0; i < nk; ++i) {                                             \
      if (k1v[i] < 0) continue;                                                \
      const float* sp = tr + k1v[i];                                           \
      float* a = acc + ((size_t)i * VO_CB + c) * W2;                           \
      float den = a[w], ac = a[w + 1];                                         \
      const float x = xv[i];                                                   \
      for (int j = 0; j < w; ++j) {                                            \
        const float v = (sp[j + 1] - sp[j]) * x + sp[j];                       \
        a[j] += v;                                                             \
        den += v * v;                                                          \
        ac += v;                                                               \
      }                                                                        \
      a[w] = den;                                                              \
      a[w + 1] = ac;                                                           \
      ++mu[i * VO_CB + c];                                                     \
    }                                                                          \
  }

#define VO_BLK_TRACE_ARGS                                                      \
  const vo_problem *p, const float *tr, int nc, int nk, const float *q0,     \
      const float *q1, const float *t0sq, const float *two_t0, float *acc,     \
      int *mu

static void vo_blk_trace_generic(VO_BLK_TRACE_ARGS) { VO_BLK_TRACE_BODY }
__attribute__((target("avx2,fma"))) static void vo_blk_trace_fma(VO_BLK_TRACE_ARGS) {
  VO_BLK_TRACE_BODY
}
static int g_have_fma = 0;

typedef struct {
  const vo_problem* p;
  const int32_t* order;     /* cells sorted by (row, k)            */
  const int32_t* item_cell; /* first position in order per item    */
  const int32_t* item_n;    /* cells per item                      */
  const int32_t* item_c0;   /* first candidate per item            */
  int n_items;
  const int32_t* cell_k;
  const int32_t* cell_row;
  float* sem;   /* [n_cells][ncand] */
  float* stk;   /* [n_cells][ncand] */
  uint64_t valid;
  int next;
  pthread_mutex_t* lock;
} vo_bjob;

static void* vo_worker_blocked(void* arg) {
  vo_bjob* job = (vo_bjob*)arg;
  const vo_problem* p = job->p;
  const int w = p->w;
  const int W2 = w + 2; /* num[w], den, ac */
  vo_leg* legs = (vo_leg*)malloc(sizeof(vo_leg) * (size_t)(p->G + 1));
  int* scratch = (int*)malloc(sizeof(int) * (size_t)(p->G + 1));
  float* acc = (float*)malloc(sizeof(float) * (size_t)VO_KB * VO_CB * W2);
  int* mu = (int*)malloc(sizeof(int) * (size_t)VO_KB * VO_CB);
  float q0[VO_CB], q1[VO_CB];
  float t0sq[VO_KB], two_t0[VO_KB];
  uint64_t valid = 0;
  int cached_row = -1, nlegs = 0;
  for (;;) {
    pthread_mutex_lock(job->lock);
    const int it = job->next++;
    pthread_mutex_unlock(job->lock);
    if (it >= job->n_items) break;
    const int32_t* cells = job->order + job->item_cell[it];
    const int nk = job->item_n[it];
    const int c0 = job->item_c0[it];
    const int nc = p->ncand - c0 < VO_CB ? p->ncand - c0 : VO_CB;
    const int row = job->cell_row[cells[0]];
    if (row != cached_row) {
      nlegs = vo_build_sweep(p, p->row_gather[row], legs, scratch);
      cached_row = row;
    }
    for (int i = 0; i < nk; ++i) {
      const float t0 = (float)(job->cell_k[cells[i]] * p->dt_s); /* scan.hpp:133 */
      t0sq[i] = t0 * t0;
      two_t0[i] = 2.0f * t0;
    }
    memset(acc, 0, sizeof(float) * (size_t)nk * VO_CB * W2);
    memset(mu, 0, sizeof(int) * (size_t)nk * VO_CB);
    for (int l = 0; l < nlegs; ++l) {
      const int g = legs[l].gather;
      const int M = p->ntraces[g];
      const float d2 = legs[l].d2, dm = legs[l].dm;
      for (int m = 0; m < M; ++m) {
        const float h2 = p->h2[(size_t)g * p->M + m];
        const float* tr = p->samples + ((size_t)g * p->M + m) * (size_t)p->ns;
        /* per (trace, candidate) moveout terms, independent of t0 */
        for (int c = 0; c < nc; ++c) {
          const int cand = c0 + c;
          const int ic = cand % p->n_c;
          if (p->op == VO_OP_CRS_ABC) {
            const int r = cand / p->n_c;
            const float A = p->a[r / p->n_b], B = p->b[r % p->n_b], v = p->v[ic];
            const float qa = (2.0f * A) * dm;
            const float qb = B * (dm * dm);
            const float qc = (4.0f * h2) / (v * v);
            q0[c] = qa + qb;            /* beta  */
            q1[c] = fmaf(qa, qa, qc);   /* gamma */
          } else {
            const float v = p->v[ic];
            q0[c] = (4.0f * h2 + d2) / (v * v);
          }
        }
        if (g_have_fma)
          vo_blk_trace_fma(p, tr, nc, nk, q0, q1, t0sq, two_t0, acc, mu);
        else
          vo_blk_trace_generic(p, tr, nc, nk, q0, q1, t0sq, two_t0, acc, mu);
      }
    }
    for (int i = 0; i < nk; ++i)
      for (int c = 0; c < nc; ++c) {
        const float* a = acc + ((size_t)i * VO_CB + c) * W2;
        float sem, st;
        vo_finalize(a, w, a[w], a[w + 1], mu[i * VO_CB + c], &sem, &st);
        valid += (uint64_t)mu[i * VO_CB + c];
        const size_t o = (size_t)cells[i] * p->ncand + c0 + c;
        job->sem[o] = sem;
        job->stk[o] = st;
      }
  }
  pthread_mutex_lock(job->lock);
  job->valid += valid;
  pthread_mutex_unlock(job->lock);
  free(legs);
  free(scratch);
  free(acc);
  free(mu);
  return NULL;
}

static const int32_t* g_sort_row;
static const int32_t* g_sort_k;
static int cmp_cell(const void* pa, const void* pb) {
  const int a = *(const int*)pa, b = *(const int*)pb;
  if (g_sort_row[a] != g_sort_row[b]) return g_sort_row[a] < g_sort_row[b] ? -1 : 1;
  if (g_sort_k[a] != g_sort_k[b]) return g_sort_k[a] < g_sort_k[b] ? -1 : 1;
  return a < b ? -1 : (a > b);
}

static void vo_run_blocked(vo_problem* p, const int32_t* cell_row,
                           const int32_t* cell_k, int n_cells, int n_threads,
                           int32_t* best_idx, float* best_s, float* best_stack,
                           float* matrix, float* stack_matrix, uint64_t* valid_out) {
  __builtin_cpu_init();
  g_have_fma = __builtin_cpu_supports("avx2") && __builtin_cpu_supports("fma");
  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_cells + 1));
  for (int i = 0; i < n_cells; ++i) order[i] = i;
  g_sort_row = cell_row; /* single caller at a time (test infrastructure) */
  g_sort_k = cell_k;
  qsort(order, (size_t)n_cells, sizeof(int32_t), cmp_cell);
  const int nchunks = (p->ncand + VO_CB - 1) / VO_CB;
  /* items: runs of <= VO_KB cells of one row x candidate chunks */
  int cap = 16, n_items = 0;
  int32_t* ic = (int32_t*)malloc(sizeof(int32_t) * cap);
  int32_t* in = (int32_t*)malloc(sizeof(int32_t) * cap);
  int32_t* i0 = (int32_t*)malloc(sizeof(int32_t) * cap);
  for (int i = 0; i < n_cells;) {
    int e = i + 1;
    while (e < n_cells && e - i < VO_KB && cell_row[order[e]] == cell_row[order[i]]) ++e;
    for (int ch = 0; ch < nchunks; ++ch) {
      if (n_items == cap) {
        cap *= 2;
        ic = (int32_t*)realloc(ic, sizeof(int32_t) * cap);
        in = (int32_t*)realloc(in, sizeof(int32_t) * cap);
        i0 = (int32_t*)realloc(i0, sizeof(int32_t) * cap);
      }
      ic[n_items] = i;
      in[n_items] = e - i;
      i0[n_items] = ch * VO_CB;
      ++n_items;
    }
    i = e;
  }
  float* sem = matrix ? matrix : (float*)malloc(sizeof(float) * (size_t)n_cells * p->ncand + 1);
  float* stk = stack_matrix ? stack_matrix
                            : (float*)malloc(sizeof(float) * (size_t)n_cells * p->ncand + 1);
  pthread_mutex_t lock;
  pthread_mutex_init(&lock, NULL);
  vo_bjob job;
  memset(&job, 0, sizeof job);
  job.p = p;
  job.order = order;
  job.item_cell = ic;
  job.item_n = in;
  job.item_c0 = i0;
  job.n_items = n_items;
  job.cell_k = cell_k;
  job.cell_row = cell_row;
  job.sem = sem;
  job.stk = stk;
  job.lock = &lock;
  if (n_threads < 1) n_threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n_threads);
  for (int i = 0; i < n_threads; ++i) pthread_create(&th[i], NULL, vo_worker_blocked, &job);
  for (int i = 0; i < n_threads; ++i) pthread_join(th[i], NULL);
  free(th);
  pthread_mutex_destroy(&lock);
  /* scan.hpp:167-179: strict '>', candidate 0 first, lowest index wins */
  for (int c = 0; c < n_cells; ++c) {
    const float* sr = sem + (size_t)c * p->ncand;
    int bc = 0;
    float bs = sr[0];
    for (int k = 1; k < p->ncand; ++k)
      if (sr[k] > bs) {
        bs = sr[k];
        bc = k;
      }
    best_idx[c] = bc;
    best_s[c] = bs;
    best_stack[c] = stk[(size_t)c * p->ncand + bc];
  }
  if (valid_out) *valid_out = job.valid;
  if (!matrix) free(sem);
  if (!stack_matrix) free(stk);
  free(order);
  free(ic);
  free(in);
  free(i0);
}

/* Output row order: CMP = input order; CRS = cdp_id order, ties by input
 * index (run_crs, crs_pipeline.hpp:449-459). */
void vo_row_order(const uint32_t* cdp_id, int G, int op, int32_t* rows) {
  for (int i = 0; i < G; ++i) rows[i] = i;
  if (op != VO_OP_NMO) sort_by_cdp((int*)rows, G, cdp_id);
}

/*
 * Evaluate a list of output cells (row, t0 index k).  Returns 0 on success,
 * 1 on an invalid configuration (w < 1, ns <= w + 1, empty central gather,
 * v <= 0), mirroring the reference's checks.
 */
int vo_run_cells(const float* samples, const float* coords,
                 const int32_t* ntraces, const uint32_t* cdp_id, int G,
                 int M, int ns, uint32_t dt_us, int op, int w, int n_a,
                 int n_b, int n_c, const float* a, const float* b,
                 const float* v, double apm, int mode,
                 const int32_t* cell_row, const int32_t* cell_k, int n_cells,
                 int n_threads, int32_t* best_idx, float* best_s,
                 float* best_stack, float* matrix, float* stack_matrix,
                 uint64_t* valid_out) {
  if (w < 1 || ns <= w + 1 || n_c < 1 || n_a < 1 || n_b < 1) return 1;
  for (int c = 0; c < n_c; ++c)
    if (!(v[c] > 0.0f)) return 1;
  vo_problem p;
  memset(&p, 0, sizeof p);
  p.samples = samples;
  p.coords = coords;
  p.ntraces = ntraces;
  p.cdp_id = cdp_id;
  p.G = G;
  p.M = M;
  p.ns = ns;
  p.dt_s = (double)dt_us * 1e-6; /* types.hpp:35 */
  p.op = op;
  p.w = w;
  p.n_a = op == VO_OP_CRS_ABC ? n_a : 1;
  p.n_b = op == VO_OP_CRS_ABC ? n_b : 1;
  p.n_c = n_c;
  p.ncand = p.n_a * p.n_b * p.n_c;
  p.a = a;
  p.b = b;
  p.v = v;
  p.apm = apm;
  p.mode = mode;
  p.h2 = (float*)malloc(sizeof(float) * (size_t)G * M + 1);
  p.mx = (float*)malloc(sizeof(float) * (size_t)G + 1);
  p.my = (float*)malloc(sizeof(float) * (size_t)G + 1);
  p.row_gather = (int*)malloc(sizeof(int) * (size_t)G + 1);
  for (int g = 0; g < G; ++g) {
    for (int m = 0; m < ntraces[g]; ++m) {
      const float* c4 = coords + ((size_t)g * M + m) * 4;
      p.h2[(size_t)g * M + m] = vo_halfpoint(c4[0], c4[1], c4[2], c4[3]);
    }
    if (ntraces[g] > 0)
      vo_midpoint(coords + (size_t)g * M * 4, &p.mx[g], &p.my[g]);
    else
      p.mx[g] = p.my[g] = 0.0f;
  }
  vo_row_order(cdp_id, G, op, p.row_gather);
  if (mode == 3) {
    /* fp64 geometry for the literal-formula mode */
    p.h2d = (double*)malloc(sizeof(double) * (size_t)G * M + 1);
    p.mxd = (double*)malloc(sizeof(double) * (size_t)G + 1);
    p.myd = (double*)malloc(sizeof(double) * (size_t)G + 1);
    for (int g = 0; g < G; ++g) {
      for (int m = 0; m < ntraces[g]; ++m) {
        const float* c4 = coords + ((size_t)g * M + m) * 4;
        const double dx = (double)c4[2] - c4[0], dy = (double)c4[3] - c4[1];
        p.h2d[(size_t)g * M + m] = (dx * dx + dy * dy) * 0.25;
      }
      const float* c0 = coords + (size_t)g * M * 4;
      p.mxd[g] = ntraces[g] > 0 ? 0.5 * ((double)c0[0] + c0[2]) : 0.0;
      p.myd[g] = ntraces[g] > 0 ? 0.5 * ((double)c0[1] + c0[3]) : 0.0;
    }
  }
  for (int c = 0; c < n_cells; ++c)
    if (cell_row[c] < 0 || cell_row[c] >= G || cell_k[c] < 0 || cell_k[c] >= ns ||
        ntraces[p.row_gather[cell_row[c]]] <= 0) {
      free(p.h2);
      free(p.mx);
      free(p.my);
      free(p.row_gather);
      return 1;
    }

  if (mode == 2) {
    vo_run_blocked(&p, cell_row, cell_k, n_cells, n_threads, best_idx, best_s,
                   best_stack, matrix, stack_matrix, valid_out);
    free(p.h2);
    free(p.mx);
    free(p.my);
    free(p.row_gather);
    return 0;
  }
  pthread_mutex_t lock;
  pthread_mutex_init(&lock, NULL);
  vo_job job;
  memset(&job, 0, sizeof job);
  job.p = &p;
  job.cell_row = cell_row;
  job.cell_k = cell_k;
  job.n_cells = n_cells;
  job.best_idx = best_idx;
  job.best_s = best_s;
  job.best_stack = best_stack;
  job.matrix = matrix;
  job.stack_matrix = stack_matrix;
  job.lock = &lock;
  if (n_threads < 1) n_threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n_threads);
  for (int i = 0; i < n_threads; ++i)
    pthread_create(&th[i], NULL, vo_worker, &job);
  for (int i = 0; i < n_threads; ++i) pthread_join(th[i], NULL);
  free(th);
  pthread_mutex_destroy(&lock);
  if (valid_out) *valid_out = job.valid;
  free(p.h2);
  free(p.mx);
  free(p.my);
  free(p.row_gather);
  free(p.h2d);
  free(p.mxd);
  free(p.myd);
  return 0;
}

/* NMO-corrected gathers (the GPU's velan_gpu_nmo_correct):
 * out[r][m][k] = interpolate(a[k1], a[k1+1], x) at hit_for(t, dt, ns, 1) of
 * t = crs_traveltime(t0_k, h2_m, 0, v[pick % n_c]) (traveltime.hpp:53-80,
 * kernel.hpp:39); 0 outside the trace and for traces past ntraces.  Rows in
 * output order (vo_row_order for op). */
void vo_nmo_correct(const float* samples, const float* coords, const int32_t* ntraces,
                    const uint32_t* cdp_id, int G, int M, int ns, uint32_t dt_us, int op,
                    const float* v, int n_c, const int32_t* picks, float* out) {
  const double dt = (double)dt_us * 1e-6;
  int32_t* rows = (int32_t*)malloc(sizeof(int32_t) * (size_t)(G + 1));
  vo_row_order(cdp_id, G, op, rows);
  for (int r = 0; r < G; ++r) {
    const int g = rows[r];
    for (int m = 0; m < M; ++m) {
      float* o = out + ((size_t)r * M + m) * (size_t)ns;
      if (m >= ntraces[g]) {
        for (int k = 0; k < ns; ++k) o[k] = 0.0f;
        continue;
      }
      const float* c4 = coords + ((size_t)g * M + m) * 4;
      const float h2 = vo_halfpoint(c4[0], c4[1], c4[2], c4[3]);
      const float* a = samples + ((size_t)g * M + m) * (size_t)ns;
      for (int k = 0; k < ns; ++k) {
        const int c = picks[(size_t)r * ns + k];
        const float t0 = (float)(k * dt);
        const float t = vo_traveltime_q(t0, h2, 0.0f, v[((c % n_c) + n_c) % n_c]);
        const vo_hit hit = vo_hit_for(t, dt, ns, 1);
        o[k] = hit.valid ? vo_interpolate(a[hit.k1], a[hit.k1 + 1], hit.x) : 0.0f;
      }
    }
  }
  free(rows);
}

/* Batch helpers for the golden / known-answer tests. */
void vo_hit_batch(const float* t, int n, double dt_s, int ns, int w,
                  int32_t* k1, float* x, uint8_t* valid) {
  for (int i = 0; i < n; ++i) {
    const vo_hit h = vo_hit_for(t[i], dt_s, ns, w);
    k1[i] = h.k1;
    x[i] = h.x;
    valid[i] = (uint8_t)h.valid;
  }
}

void vo_traveltime_batch(int op, const float* t0, const float* h2,
                         const float* dm, const float* A, const float* B,
                         const float* v, int n, float* out) {
  for (int i = 0; i < n; ++i) {
    if (op == VO_OP_CRS_ABC)
      out[i] = vo_traveltime_abc(t0[i], h2[i], dm[i], A[i], B[i], v[i]);
    else
      out[i] = vo_traveltime_q(t0[i], h2[i], dm[i] * dm[i], v[i]);
  }
}

/* finalize (kernel.hpp:43-56) on explicit accumulators. */
void vo_finalize(const float* num, int w, float den, float ac, int m_used,
                 float* semblance, float* stack) {
  float s = 0.0f, st = 0.0f;
  if (den > 0.0f) {
    float sum_sq = 0.0f;
    for (int j = 0; j < w; ++j) sum_sq += num[j] * num[j];
    s = sum_sq / den;
  }
  if (m_used > 0) st = ac / ((float)m_used * (float)w);
  *semblance = s;
  *stack = st;
}
