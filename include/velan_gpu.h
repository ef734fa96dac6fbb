/*
 * velan_gpu.h — C-ABI of the B200-native semblance parameter search.
 *
 * This is the drop-in boundary for the hot path of the reference library
 * "velan" (/root/reference/proj/include/velan, header-only C++20).  The
 * reference has no FFI; its replacement seam is the pipeline layer:
 *
 *   velan::run_cmp(const Dataset&, const ScanConfig&, int workers,
 *                  CacheStats*)                       cmp_pipeline.hpp:94-106
 *   velan::run_crs(const Dataset&, const ScanConfig&, GridDims, double apm,
 *                  const CrsOptions&, CrsRunInfo*, CacheStats*)
 *                                                     crs_pipeline.hpp:283-460
 *   velan::scan_cdp(gather, cfg)                       cmp_pipeline.hpp:17-27
 *   velan::scan_central_cdp(central, neighbors, cfg)   crs_pipeline.hpp:184-197
 *
 * Every entry point below replaces one of those (cited per function).  The
 * signatures are plain C: host pointers and sizes, no torch or velan types,
 * no exceptions.  Errors are status codes that map 1:1 onto the reference's
 * exception hierarchy (error.hpp:9-40); the message of the last failure on
 * the calling thread is available from velan_gpu_last_error().
 *
 * Data layout (mirrors velan::Dataset, types.hpp:14-54, flattened):
 *   samples  fp32 [n_gathers][max_traces][ns]  (trace-contiguous, as
 *                                               Trace::samples)
 *   coords   fp32 [n_gathers][max_traces][4]   (sx, sy, gx, gy)
 *   ntraces  i32  [n_gathers]                  (traces actually present)
 *   cdp_id   u32  [n_gathers]
 * Half-offsets (compute_halfpoints, traveltime.hpp:16-27) and midpoints
 * (midpoint_of, types.hpp:57-62) are derived from coords on the host with the
 * reference's fp32 expressions, so results are bit-comparable.
 */
#ifndef VELAN_GPU_H_
#define VELAN_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VELAN_GPU_ABI_VERSION 2

/* Status codes.  0 = success.  Config and parameter errors are raised before
 * any device work, like ScanConfig::validate (scan.hpp:61-78). */
enum {
  VELAN_GPU_OK = 0,
  VELAN_GPU_ECONFIG = 1,  /* velan::config_error    (error.hpp:19-22) */
  VELAN_GPU_EPARAM = 2,   /* velan::parameter_error (error.hpp:14-17) */
  VELAN_GPU_ERUNTIME = 3, /* velan::error: worker/device failure       */
  VELAN_GPU_ENODEV = 4    /* no usable sm_100 device                    */
};

/* Moveout operator evaluated per (pair, trace).
 *  NMO     t = sqrt(t0^2 + 4 h2 / v^2)                traveltime.hpp:59-61
 *  CRS_D2  t = sqrt(t0^2 + (4 h2 + d2) / v^2)         traveltime.hpp:53-56
 *          (the reference's neighbourhood operator, d2 = |dm|^2)
 *  CRS_ABC t = sqrt((t0 + 2 A dm)^2 + 2 t0 B dm^2 + 4 h2 / v^2)
 *          (BASELINE.json's three-parameter operator; C = 2/(t0 v^2) is
 *          scanned through v.  No reference implementation exists, see
 *          DESIGN.md §3 for the exact fp32 evaluation order.) */
typedef enum {
  VELAN_OP_NMO = 0,
  VELAN_OP_CRS_D2 = 1,
  VELAN_OP_CRS_ABC = 2
} velan_operator;

/* Kernel variant, the GPU analogue of velan::KernelVariant (scan.hpp:14-23).
 *  EXACT  every fp32 operation in the reference order and rounding: the
 *         semblance matrix, picks and stack are bitwise identical to
 *         velan::scan_tile_blocked + scan_sweep (kernel.hpp:276-316,
 *         scan.hpp:108-181).
 *  FAST   restructured accumulation (the production variant): picks and hit
 *         indices identical, semblance/stack within 1e-4 relative. */
typedef enum { VELAN_VARIANT_EXACT = 0, VELAN_VARIANT_FAST = 1 } velan_variant;

typedef enum { VELAN_MEM_HOST = 0, VELAN_MEM_DEVICE = 1 } velan_mem;

typedef struct velan_gpu_dataset {
  int32_t n_gathers;
  int32_t max_traces; /* stride of the trace axis (Dataset::fold)          */
  int32_t ns;         /* CdpGather::ns, shared by every gather            */
  uint32_t dt_us;     /* CdpGather::dt_us                                  */
  const uint32_t* cdp_id;  /* host [n_gathers]                             */
  const int32_t* ntraces;  /* host [n_gathers]                             */
  const float* coords;     /* host [n_gathers][max_traces][4]              */
  const float* samples;    /* [n_gathers][max_traces][ns], see samples_mem */
  int32_t samples_mem;     /* velan_mem                                    */
  int32_t samples_device;  /* CUDA ordinal when samples_mem == DEVICE      */
} velan_gpu_dataset;

typedef struct velan_gpu_scan {
  int32_t op;      /* velan_operator                                      */
  int32_t variant; /* velan_variant                                       */
  int32_t w;       /* ScanConfig::w, window length in samples (1..32)     */
  /* Candidate axes.  Flat candidate index = (ia * n_b + ib) * n_c + ic;
   * NMO / CRS_D2 use n_a = n_b = 1.  Lowest flat index wins exact ties,
   * like scan_sweep's strict '>' (scan.hpp:167-179). */
  int32_t n_a, n_b, n_c;
  const float* a; /* host [n_a]  A, s/m          (CRS_ABC only)           */
  const float* b; /* host [n_b]  B, s/m^2        (CRS_ABC only)           */
  const float* v; /* host [n_c]  velocity, m/s   (all operators)          */
  double apm;     /* CRS: closed-ball radius in m (neighbors_of,
                     crs_pipeline.hpp:162-180); ignored for NMO           */
  /* Output rows [row_first, row_first + row_count) of the row order below
   * (row_count 0 = all).  A shard of a longer line passes its own gathers
   * plus the +-aperture halo and restricts the outputs to its block: the
   * halo gathers then only feed neighbourhoods (run_crs's strips,
   * crs_pipeline.hpp:341-347, as a replicated 1-D halo). */
  int32_t row_first, row_count;
} velan_gpu_scan;

typedef struct velan_gpu_result {
  /* Caller-allocated outputs, row r = output midpoint r.  CMP rows follow
   * input order (run_cmp); CRS rows follow cdp_id order, ties by input index
   * (run_crs, crs_pipeline.hpp:449-459). */
  int32_t out_mem;        /* velan_mem of the four arrays               */
  int32_t* best_idx;      /* [rows][ns] flat candidate index            */
  float* best_semblance;  /* [rows][ns]  BestPick::semblance            */
  float* best_stack;      /* [rows][ns]  SemblanceMatrix::stack_trace   */
  float* matrix;          /* optional [rows][ns][n_cand] (values),
                             NULL = not emitted                         */
  int32_t* row_gather;    /* optional [rows]: input gather index per row */
  /* Filled by the call. */
  uint64_t valid_intersections;   /* CacheStats::naive_fetches          */
  uint64_t nominal_intersections; /* rows * ns * n_cand * traces/sweep  */
  double kernel_ms;  /* device time of the scan kernels, max over devices */
  double total_ms;   /* wall time of the whole call                       */
  /* Optional per-sample top-k (QC of the semblance panel
   * without the ns x n_cand matrix): the k best candidates of every output
   * sample, best first (ties: lower flat index first, so entry 0 is the
   * pick); entries past n_cand hold index -1.  topk 0 = off, max 8.  Same
   * memory kind as the other outputs (out_mem). */
  int32_t topk;
  int32_t* topk_idx;      /* [rows][ns][topk] flat candidate index      */
  float* topk_semblance;  /* [rows][ns][topk]                           */
} velan_gpu_result;

typedef struct velan_gpu_ctx velan_gpu_ctx;
typedef struct velan_gpu_plan velan_gpu_plan;

/* ABI version and the message of the last failure on this thread. */
int velan_gpu_abi_version(void);
const char* velan_gpu_last_error(void);
/* Struct layout check for foreign bindings: writes sizeof and the offset of
 * the last member of velan_gpu_dataset, _scan, _result, _synth (8 values). */
int velan_gpu_abi_layout(int32_t* out8);
/* Number of visible sm_100 devices (0 on a host without GPU). */
int velan_gpu_device_count(void);

/* Context: owns per-device streams, events and cached device buffers.
 * device_ids may be NULL (then devices 0..n_devices-1).  Replaces the
 * std::thread worker pool of parallel_for_indexed (cmp_pipeline.hpp:34-88):
 * midpoints are split into contiguous blocks, one host thread per device. */
int velan_gpu_create(const int32_t* device_ids, int32_t n_devices,
                     velan_gpu_ctx** out);
void velan_gpu_destroy(velan_gpu_ctx* ctx);

/* Validate a scan without touching a device; mirrors ScanConfig::validate
 * (scan.hpp:61-78) and scan_sweep's ns > w + 1 check (scan.hpp:113-114). */
int velan_gpu_validate(const velan_gpu_dataset* ds, const velan_gpu_scan* sc);

/* Host-side sweep description, no device needed: the output row order
 * (row_gather[rows]), traces per sweep (sweep_traces[rows]), the legs of
 * every sweep in TraceSweep order (kernel.hpp:61-113) as CSR (leg_off[rows+1],
 * leg_gather[n_legs], filled when leg_capacity >= n_legs) and the nominal
 * intersection count.  Any output pointer may be NULL. */
int velan_gpu_describe(const velan_gpu_dataset* ds, const velan_gpu_scan* sc,
                       int32_t* row_gather, int32_t* sweep_traces,
                       int32_t* leg_off, int32_t* leg_gather,
                       int64_t leg_capacity, int64_t* n_legs,
                       uint64_t* nominal);

/* One-shot scans over host buffers (host->device, kernels, device->host).
 *  velan_gpu_cmp  replaces run_cmp   (cmp_pipeline.hpp:94-106); op NMO.
 *  velan_gpu_crs  replaces run_crs   (crs_pipeline.hpp:283-460) on a 1-D
 *                 contiguous shard layout; op CRS_D2 or CRS_ABC.
 * Both are synchronous, deterministic and bitwise independent of the number
 * of devices (the reference's worker-count invariance,
 * test_cmp_pipeline.cpp:122-140). */
int velan_gpu_cmp(velan_gpu_ctx* ctx, const velan_gpu_dataset* ds,
                  const velan_gpu_scan* sc, velan_gpu_result* res);
int velan_gpu_crs(velan_gpu_ctx* ctx, const velan_gpu_dataset* ds,
                  const velan_gpu_scan* sc, velan_gpu_result* res);

/* Resident plans (single device): tables and samples stay in HBM across
 * executions.  samples may already be device memory (samples_mem DEVICE).
 * execute runs on `stream` (a cudaStream_t, NULL = the plan's own stream)
 * and leaves outputs where res->out_mem says. */
int velan_gpu_plan_create(velan_gpu_ctx* ctx, const velan_gpu_dataset* ds,
                          const velan_gpu_scan* sc, velan_gpu_plan** out);
int velan_gpu_plan_execute(velan_gpu_plan* plan, velan_gpu_result* res,
                           void* stream);
/* Kernel launches the last execute issued (scan waves, FAST table passes,
 * top-k; for launch accounting); before the first execute, the scan waves. */
int velan_gpu_plan_launches(const velan_gpu_plan* plan);
void velan_gpu_plan_destroy(velan_gpu_plan* plan);

/* NMO-corrected output gathers: every trace m of output
 * row r flattened with the row's picks — out[r][m][k] = interpolate(a[k1],
 * a[k1 + 1], x) (kernel.hpp:39) at hit_for(t, dt, ns, 1) (traveltime.hpp:
 * 66-80: k1 = floor(t / dt), x its fraction, 0 outside the trace) of the
 * central gather's traveltime t = crs_traveltime(t0_k, h2_m, 0, v)
 * (traveltime.hpp:53-56) for the pick's velocity v = v[picks[r][k] % n_c]
 * (for CRS_ABC at dm = 0 the operator is that same NMO expression bit for
 * bit).  Rows are the scan's output rows (row order and row_first /
 * row_count as for the scan); picks [rows][ns] host, out [rows][max_traces]
 * [ns] host, traces past a gather's count zero.  The stacked, corrected
 * trace is the mean over m.  Single device (the context's first). */
int velan_gpu_nmo_correct(velan_gpu_ctx* ctx, const velan_gpu_dataset* ds,
                          const velan_gpu_scan* sc, const int32_t* picks, float* out);

/* hit_for (traveltime.hpp:66-80) evaluated by the device code path of the
 * given variant, for n traveltimes t (host arrays).  Test hook for the
 * index arithmetic: k1 and valid must match the reference bit for bit. */
int velan_gpu_hit_batch(const float* t, int32_t n, double dt_s, int32_t ns,
                        int32_t w, int32_t variant, int32_t* k1, float* x,
                        uint8_t* valid);

/* Seeded synthetic inputs of the BASELINE.json configs, generated on the
 * host with per-gather counter-based streams (order-free, reproducible for
 * any thread count).  kind: 0 = CMP (hyperbolic events), 1 = CRS line
 * (dipping curved reflectors).  Fills caller buffers shaped like
 * velan_gpu_dataset (samples [G][M][ns], coords [G][M][4], ntraces,
 * cdp_id).  See DESIGN.md §6 for the event model. */
/* FP32 FMA throughput of `device` in TFLOP/s (best of 5 probes): the
 * measured denominator of the FP32 roofline fraction (bench.py). */
int velan_gpu_measure_fp32_peak(int32_t device, double* tflops);

typedef struct velan_gpu_synth {
  int32_t kind;
  int32_t n_gathers, n_traces, ns;
  uint32_t dt_us;
  double spacing;           /* midpoint spacing, m                     */
  double h0, dh;            /* half-offset of trace m = h0 + m * dh    */
  int32_t n_events;
  double t0_lo, t0_hi;      /* event zero-offset time range, s         */
  double v_lo, v_hi;        /* event velocity range (CMP-small, CRS)   */
  int32_t v_profile;        /* CMP: 0 = uniform v, 1 = v(t0) trend     */
  double v_trend_0, v_trend_slope, v_perturb; /* v = (v0 + s t0)(1+eps) */
  double amp_lo, amp_hi;
  double freq;              /* Ricker peak frequency, Hz               */
  double sigma;             /* Gaussian noise sigma                    */
  double a_abs, b_max;      /* CRS: A ~ U[-a_abs, a_abs], B ~ U[0,b_max] */
  uint64_t seed;
  int32_t gather_first;     /* generate gathers [first, first+n) of the
                               full line (for sharded generation)      */
  int32_t n_line;           /* gathers in the full line (0 = n_gathers);
                               CRS reflector positions span it         */
  int32_t n_threads;        /* 0 = hardware concurrency                */
} velan_gpu_synth;

int velan_gpu_synth_generate(const velan_gpu_synth* p, float* samples,
                             float* coords, int32_t* ntraces,
                             uint32_t* cdp_id);
/* The same generator on the device: fills device memory
 * d_samples [n_gathers][n_traces][ns] on `stream` (a cudaStream_t, NULL =
 * default) with the host generator's streams and model (geometry via
 * velan_gpu_synth_generate with samples = NULL).  Synchronous. */
int velan_gpu_synth_generate_device(const velan_gpu_synth* p, float* d_samples,
                                    void* stream);
/* The CRS line's reflectors, 6 doubles per event (t0, v, amp, x, A, B). */
int velan_gpu_synth_line_events(const velan_gpu_synth* p, double* out6);

/* ---------------------------------------------------------------------
 * Files.  SSF1 trace files (read_dataset / write_dataset,
 * io.hpp:88-166) and SMB1 pick files (write_picks, io.hpp:168-194), byte-
 * compatible with the reference, read and written without materialising a
 * Dataset of per-trace vectors.  Errors: ECONFIG = velan::format_error
 * (message carries the byte offset), ERUNTIME = I/O failure, EPARAM = bad
 * arguments.
 * --------------------------------------------------------------------- */
typedef struct velan_ssf1_info {
  uint32_t n_gathers;      /* ncdps                                       */
  uint32_t fold;           /* Dataset::fold (the layout's trace stride)    */
  uint32_t ns, dt_us;      /* of the first gather                          */
  int32_t uniform;         /* 1: every gather has the same ns and dt_us    */
  uint64_t metadata_bytes; /* optional JSON tail                           */
  uint64_t file_bytes;
} velan_ssf1_info;

typedef struct velan_ssf1 velan_ssf1;
typedef struct velan_smb1_writer velan_smb1_writer;

/* Index an SSF1 file: header words of every gather, validated like
 * read_dataset (magic, version, trace count <= fold, dt != 0, metadata tail,
 * no trailing bytes); samples are not read. */
int velan_ssf1_open(const char* path, velan_ssf1** out, velan_ssf1_info* info);
void velan_ssf1_close(velan_ssf1* f);
/* Per-gather header arrays [n_gathers] (any pointer may be NULL). */
int velan_ssf1_gathers(const velan_ssf1* f, uint32_t* cdp_id, int32_t* ntraces,
                       uint32_t* ns, uint32_t* dt_us);
int velan_ssf1_metadata(const velan_ssf1* f, char* buf, uint64_t cap);
/* Gathers [first, first + count) into the flattened layout of
 * velan_gpu_dataset: samples [count][max_traces][ns], coords
 * [count][max_traces][4], zero beyond each gather's trace count.  One pread
 * per gather, n_threads readers (0 = hardware concurrency); pass pinned
 * buffers to feed asynchronous host->device copies. */
int velan_ssf1_read(const velan_ssf1* f, int32_t first, int32_t count, int32_t max_traces,
                    float* samples, float* coords, int32_t n_threads);
/* The same for an arbitrary list of gather indices (a CRS block with its
 * halo): gathers[i] lands at position i of the layout. */
int velan_ssf1_read_list(const velan_ssf1* f, const int32_t* gathers, int32_t count,
                         int32_t max_traces, float* samples, float* coords,
                         int32_t n_threads);
/* midpoint_of (types.hpp:57-62) of every gather [n_gathers], from the first
 * trace's coordinates only (16 bytes per gather read; EPARAM on an empty
 * gather, as midpoint_of throws) — what a halo-aware block reader needs
 * before any samples. */
int velan_ssf1_midpoints(const velan_ssf1* f, float* mx, float* my);
/* write_dataset (io.hpp:95-122), byte-identical; samples must be host. */
int velan_ssf1_write(const char* path, const velan_gpu_dataset* ds, const char* metadata,
                     uint64_t metadata_bytes);

/* write_picks (io.hpp:170-194) as a stream: the header declares n_cdps,
 * records are appended block by block (per CDP: cdp_id, ns, nc, ns x
 * (velocity, semblance), then the ns x nc matrix when with_matrix), and
 * _end checks that every declared record was written. */
int velan_smb1_begin(const char* path, uint32_t n_cdps, int32_t ns, int32_t nc,
                     int32_t with_matrix, velan_smb1_writer** out);
int velan_smb1_append(velan_smb1_writer* w, int32_t n, const uint32_t* cdp_id,
                      const float* pick_velocity, const float* pick_semblance,
                      const float* matrix);
int velan_smb1_end(velan_smb1_writer* w);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* VELAN_GPU_H_ */
