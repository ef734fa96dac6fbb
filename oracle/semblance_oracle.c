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
 *
 * plus the BASELINE three-parameter CRS operator (vo_traveltime_abc), which
 * has no reference implementation; its evaluation order is fixed in
 * DESIGN.md §3 and shared with the CUDA kernels.
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

/* ------------------------------------------------------------------------ */
/* Sweep construction (TraceSweep, kernel.hpp:61-113; neighbors_of,
 * crs_pipeline.hpp:162-180).                                                */

typedef struct {
  int gather;
  float d2; /* |dm|^2, fp32 (kernel.hpp:88-90)        */
  float dm; /* signed mx offset, ABC operator only     */
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
        const vo_result r = vo_scan_pair(p, legs, nlegs, t0, cand, num, win);
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
  return NULL;
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
  for (int c = 0; c < n_cells; ++c)
    if (ntraces[p.row_gather[cell_row[c]]] <= 0) {
      free(p.h2);
      free(p.mx);
      free(p.my);
      free(p.row_gather);
      return 1;
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
  return 0;
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
