/*
 * csrk.h -- C-ABI of libcsrk_cuda.so, the B200-native CSR-k SpMV.
 *
 * The reference (arxiv 2203.05096's `csrk` package, /root/reference/pkg) is
 * pure Python; its "FFI" for this path is the Python call surface listed in
 * SURVEY.md §8(b).  Every entry point below names the reference function it
 * replaces (file:line under pkg/src/csrk/).  The Python package
 * `paper_2203_05096_b200` binds these through ctypes.
 *
 * Conventions
 *   - plain pointers and sizes only; no torch or CUDA types in signatures
 *     (streams are passed as `void*` holding a cudaStream_t, NULL = default);
 *   - indices are uint32 (reference format.py:32 INDEX_DTYPE), values f64
 *     (format.py:33 VALUE_DTYPE), permutations int64 (format.py:130);
 *   - every function returns CSRK_OK (0) or an error code; the message of
 *     the last failure on the calling thread is csrk_last_error();
 *   - CSRK_EINVAL messages reuse the reference's ValueError wording.
 *
 * Threading
 *   - a matrix handle is bound to one device; calls on distinct handles are
 *     independent;
 *   - every entry point that plans, stages or launches on a handle holds
 *     that handle's lock, so concurrent calls on ONE handle serialise (the
 *     reference's kernels are reentrant -- spmv_csr2/3 under a caller's
 *     executor, kernels.py:158-182 -- and so are these);
 *   - the stream-ordered SpMV entry points return once the work is queued:
 *     a caller that launches on several streams orders its own x / y
 *     buffers; the long-row kernel runs on a side stream private to each
 *     caller stream (forked from and joined back to it), so launches on
 *     different streams, or on one stream under CUDA-graph capture, share
 *     no fork / join state;
 *   - the host-buffer entry points (csrk_spmv_host, construction) block
 *     until their results are in host memory.
 */
#ifndef CSRK_H
#define CSRK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CSRK_ABI_VERSION 1

#define CSRK_OK 0
#define CSRK_EINVAL 1 /* maps to ValueError */
#define CSRK_ECUDA 2  /* maps to RuntimeError */
#define CSRK_ENOMEM 3 /* maps to MemoryError */
#define CSRK_ENCCL 4  /* maps to RuntimeError (multi-GPU entry points) */

/* value storage types for csrk_matrix_upload(value_types) bitmask and for
 * the `value_type` argument of the SpMV entry points */
#define CSRK_F64 1
#define CSRK_F32 2

/* summation order of a row (bitwise contract):
 *   SERIAL  -- strict left-to-right sum, no FMA: kernels.py:117-147 and
 *              kernels.py:224-228 (spmv_csr_ref / spmv_csr2 / spmv_csr3 /
 *              emulate_gpu_spmv3 all share it)
 *   STRIDED -- nonzero p of a row goes to lane p mod nx, lanes summed
 *              serially, then a zero-padded halving tree:
 *              kernels.py:264-324 (emulate_gpu_spmv35) */
#define CSRK_SERIAL 0
#define CSRK_STRIDED 1

typedef struct csrk_matrix csrk_matrix;

int csrk_abi_version(void);
const char *csrk_last_error(void);
int csrk_device_count(int *count);

/* ---- raw device buffers (for callers without another CUDA allocator) ---- */
int csrk_buffer_alloc(int device, int64_t bytes, void **out);
int csrk_buffer_free(int device, void *p);
/* kind: 0 host->device, 1 device->host, 2 device->device; stream may be
 * NULL (legacy default stream); the copy is complete on return when stream
 * is NULL, otherwise stream-ordered */
int csrk_memcpy(void *dst, const void *src, int64_t bytes, int kind,
                void *stream);
int csrk_memset(void *dst, int value, int64_t bytes, void *stream);
int csrk_stream_sync(void *stream);
int csrk_device_sync(int device);

/* ---- device matrix handle ------------------------------------------------
 * Replaces the host-resident CsrMatrix / CsrKMatrix (format.py:45-230) on the
 * device.  k = 1 is plain CSR (group pointers ignored), k = 2 uses sr_ptr
 * (n_sr + 1 entries), k = 3 uses sr_ptr and ssr_ptr (n_ssr + 1 entries).
 * Host arrays are only read during the call.  value_types: CSRK_F64 and/or
 * CSRK_F32 storage to keep resident. */
int csrk_matrix_upload(int device, int64_t n_rows, int64_t n_cols, int64_t nnz,
                       const uint32_t *row_ptr, const uint32_t *col_idx,
                       const double *vals, int k, int64_t n_sr,
                       const uint32_t *sr_ptr, int64_t n_ssr,
                       const uint32_t *ssr_ptr, int value_types,
                       csrk_matrix **out);
int csrk_matrix_free(csrk_matrix *m);
/* out[0..6] = n_rows, n_cols, nnz, k, n_sr, n_ssr, device */
int csrk_matrix_shape(const csrk_matrix *m, int64_t out[7]);
/* copy the device arrays back; any output pointer may be NULL */
int csrk_matrix_download(const csrk_matrix *m, uint32_t *row_ptr,
                         uint32_t *col_idx, double *vals, uint32_t *sr_ptr,
                         uint32_t *ssr_ptr);
/* add an f32 copy of the values (for CSRK_F32 SpMV) if not present */
int csrk_matrix_add_f32(csrk_matrix *m);
/* Tile plan of the streaming kernel: contiguous row ranges balanced by
 * cost = nonzeros + rows (tile_cost per tile), cut only on group boundaries
 * (SSRs for k=3, SRs for k=2) when every group costs at most tile_cost / 8;
 * cap = stage capacity in nonzeros (larger tiles run in direct mode);
 * stages = TMA ring depth per CTA.  0 = defaults. */
int csrk_matrix_set_plan(csrk_matrix *m, int64_t tile_cost, int64_t cap,
                         int64_t stages);
/* out = tile_cost, cap, rcap, stages, n_tiles, group_aligned, gather mode,
 *       ctas_per_sm (the f64 value when auto), cut mode, n_long (rows
 *       longer than 128 nonzeros, summed by the long-row kernel) */
int csrk_matrix_plan(const csrk_matrix *m, int64_t out[10]);
/* CTAs per SM a launch with this value type uses (out[7] of
 * csrk_matrix_plan is the f64 figure; fp32 runs 4 per SM on regular rows). */
int csrk_matrix_plan_ctas(const csrk_matrix *m, int value_type, int64_t *ctas);
/* Schedule of the streaming kernel (B200 tuning knobs with no reference
 * counterpart; results are bitwise identical under every setting).
 * gather: 0 = inline (each row gathers its x while summing), 1 = gather-first
 * (f64 only: a tile's x gathers are issued together, the products staged in
 * shared memory, then summed in the row's order), 2 = auto (default:
 * gather-first for the serial order when rows average > 16 nonzeros).
 * ctas_per_sm: resident CTAs per SM (1..8; 0 = auto: 2 for irregular rows
 * -- variance > 10 --, else 3 in f64 and 4 in f32); the shared-memory
 * carveout is set to exactly what they need, and the rest of the 256 KB
 * stays L1 for the x gathers. */
int csrk_matrix_set_schedule(csrk_matrix *m, int gather, int ctas_per_sm);
/* Where tile cuts may fall: 0 = auto (on group boundaries -- SSRs for
 * k=3, SRs for k=2, the paper's block <-> super-super-row mapping of
 * Listing 3 -- when every group costs at most tile_cost / 8, else on rows),
 * 1 = always on rows, 2 = always on group boundaries (pitch shrunk by the
 * largest group so a tile still fits its stage).  Results are bitwise the
 * same; this is the A/B knob of DESIGN.md §7. */
int csrk_matrix_set_cut_mode(csrk_matrix *m, int mode);
/* Build (or rebuild) the tile plan a launch with this value type / order /
 * nx would use, without launching: csrk_spmv_tiles and
 * csrk_matrix_tile_rows then index exactly that plan. */
int csrk_matrix_prepare(csrk_matrix *m, int value_type, int variant, int nx);

/* ---- SpMV ------------------------------------------------------------------
 * y = A x on device-resident x / y (already in the permuted index space, as
 * spmv_csr3 expects, kernels.py:209-221).  Replaces spmv_csr_ref
 * (kernels.py:97-114, k=1), spmv_csr2 (kernels.py:185-206, k=2),
 * spmv_csr3 (kernels.py:209-221, k=3) with variant CSRK_SERIAL, and the
 * arithmetic of emulate_gpu_spmv35 (kernels.py:284-324) with CSRK_STRIDED
 * and nx = dims.x (1..32).  value_type selects f64 x/y/vals or f32
 * x/y/vals (f32: batches of up to 8 products summed with fp32 FMAs, each
 * batch folded into an f64 row accumulator, rounded to f32 once).
 * Asynchronous on `stream`, launched with programmatic dependent launch
 * (CSRK_PDL=0 disables it): the launch may begin streaming the handle's
 * matrix arrays while the previous kernel on `stream` still runs, and it
 * reads x and writes y only after that kernel has completed -- ordinary
 * stream order for x and y; the matrix arrays must not be modified by
 * kernels on `stream` between launches. */
int csrk_spmv(const csrk_matrix *m, int value_type, int variant, int nx,
              const void *x, void *y, void *stream);
/* Same, from host x to host y (H2D, kernel, D2H on an internal stream;
 * returns when y is written).  The drop-in call shape of spmv_csr3(m, x). */
int csrk_spmv_host(csrk_matrix *m, int value_type, int variant, int nx,
                   const void *x_host, void *y_host);
/* csrk_spmv over the tiles [t0, t1) of the handle's plan only (rows
 * tile_rows[t0] .. tile_rows[t1]); the multi-GPU step computes the interior
 * tiles while the x halo is in flight, then the boundary tiles. */
int csrk_spmv_tiles(const csrk_matrix *m, int value_type, int variant, int nx,
                    const void *x, void *y, int64_t t0, int64_t t1, void *stream);
/* the plan's tile row bounds (n_tiles + 1 entries, see csrk_matrix_plan) */
int csrk_matrix_tile_rows(const csrk_matrix *m, uint32_t *out);
/* CUDA-event device time of the last csrk_spmv_host kernel, milliseconds */
int csrk_last_kernel_ms(const csrk_matrix *m, float *ms);

/* Literal paper mappings, with the reference's per-row lane trace
 * (EmulationTrace, kernels.py:55-87; 7 int64 columns of n_rows entries:
 * row, block, z_lane, y_lane, x_first, x_count, reduction_depth; may be
 * NULL).  listing3 = emulate_gpu_spmv3 (kernels.py:231-261, PAPER Listing
 * 3); listing4 = emulate_gpu_spmv35 (kernels.py:284-324, PAPER Listing 4).
 * Require k = 3, f64. */
int csrk_spmv_listing3(const csrk_matrix *m, int dx, int dy, const double *x,
                       double *y, int64_t *trace, void *stream);
int csrk_spmv_listing4(const csrk_matrix *m, int dx, int dy, int dz,
                       const double *x, double *y, int64_t *trace,
                       void *stream);

/* Diagnostic (no reference counterpart; SURVEY.md 8(d) "a gather-only kernel
 * variant to isolate x"): walks col_idx in the streaming kernel's chunk
 * distribution; mode 0 reads col_idx only, mode 1 also gathers
 * x[col_idx[p]] (f64).  The difference of the two launches' ncu sector
 * counters is the x gathers' own L2 / L1 hit rate.  out: 1 double (written
 * only to keep the loads alive). */
int csrk_probe_gather(const csrk_matrix *m, int mode, const double *x, double *out,
                      void *stream);

/* ---- construction on device ------------------------------------------------
 * csrk_pack: replaces pack_csrk (format.py:347-393) + _permute_symmetric
 * (format.py:318-344).  Uploads A (original order) and the permutation,
 * builds P.A.P^T with per-row column sort and the group pointer arrays
 * (prefix sums of sizes1 / sizes2) on the device, and returns the packed
 * handle.  n_levels = 1 (k=2) or 2 (k=3); sizes2 may be NULL for k=2.
 * Validation (square, sizes positive and summing to the level below) uses
 * the reference's messages ("level N ..."). */
int csrk_pack(int device, int64_t n, int64_t nnz, const uint32_t *row_ptr,
              const uint32_t *col_idx, const double *vals, const int64_t *fwd,
              const int64_t *inv, int n_levels, int64_t n_sizes1,
              const int64_t *sizes1, int64_t n_sizes2, const int64_t *sizes2,
              csrk_matrix **out);
/* permute_vector / unpermute_vector (format.py:396-409) on device:
 * out[i] = in[idx[i]] with idx = perm.inv (permute) or perm.fwd (unpermute);
 * f64, device pointers, asynchronous. */
int csrk_gather_f64(int64_t n, const double *in, const int64_t *idx,
                    double *out, void *stream);
/* compute_stats (tuning.py:108-134) integer parts on the device:
 * out[0] = sum(row_nnz), out[1] = sum(row_nnz^2), out[2] = max row_nnz,
 * out[3] = off-diagonal count, out[4] = off-diagonal entries whose
 * transpose is present.  Works on any handle (uses its current arrays). */
int csrk_stats(const csrk_matrix *m, int64_t out[5]);
/* float(np.var(row_nnz)) bit for bit (tuning.py:130): numpy's pairwise
 * summation of (row_nnz - mean)^2 divided by n_rows; `mean` must be
 * float(nnz) / n_rows as numpy computes it. */
int csrk_row_variance(const csrk_matrix *m, double mean, double *out);

/* Stable LSD radix sort of n (uint64 key, uint32 value) pairs in device
 * memory by key bits [begin_bit, end_bit) (multiples of 8) -- the sorting
 * primitive of device-side construction. */
int csrk_sort_pairs(int device, int64_t n, uint64_t *keys, uint32_t *vals,
                    int begin_bit, int end_bit, void *stream);

/* Device graphs (first stage of device-side Band-k): the graph of A + A^T
 * without the diagonal (build_graph, reorder.py:115-135), relabelling by a
 * permutation (_relabel_graph, reorder.py:192-196) and contraction by a
 * fine-to-coarse map (_contract, reorder.py:176-184), built on the device by
 * composite-key radix sorts; arrays identical to the host restatement. */
typedef struct csrk_dgraph csrk_dgraph;
typedef struct csrk_bandk_result csrk_bandk_result;
int csrk_dgraph_build(const csrk_matrix *a, csrk_dgraph **out);
int csrk_dgraph_relabel(const csrk_dgraph *g, const int64_t *fwd_host,
                        csrk_dgraph **out);
int csrk_dgraph_contract(const csrk_dgraph *g, const int64_t *f2c_host,
                         int64_t m, csrk_dgraph **out);
/* out = n, number of directed adjacency entries */
int csrk_dgraph_sizes(const csrk_dgraph *g, int64_t out[2]);
int csrk_dgraph_download(const csrk_dgraph *g, int64_t *ptr, int64_t *idx,
                         int64_t *ew, int64_t *nw);
int csrk_dgraph_free(csrk_dgraph *g);
/* weighted_bandwidth_order (reorder.py:281-336) of a device graph, bit-exact:
 * level-synchronous Cuthill-McKee with min-position parent claims, all
 * components at once; fwd[n] written to host memory. */
int csrk_dgraph_wbo(const csrk_dgraph *g, int64_t *fwd_host);
/* heavy_edge_matching (reorder.py:138-173) on the device (Jacobi fixed
 * point over visit ranks); match[n] to host memory, sweeps in *iters. */
int csrk_dgraph_match(const csrk_dgraph *g, int64_t *match_host, int *iters);
/* coarsen (reorder.py:199-237) on the device: new coarse graph + f2c[n]. */
int csrk_dgraph_coarsen(const csrk_dgraph *g, double target, int64_t *f2c_host,
                        csrk_dgraph **out);
/* band_k (reorder.py:415-469) entirely on the device, bit-exact with
 * csrk_band_k; the matrix handle supplies the pattern (any k). */
int csrk_band_k_device(const csrk_matrix *a, int k, const double *targets,
                       csrk_bandk_result **out);

/* Canonical CSR from coordinate triplets on the device; replaces the body of
 * csr_from_arrays (format.py:233-284) after its range checks: a stable sort
 * by (row, col) and duplicates summed in input order exactly as
 * np.add.reduceat does (first value + numpy's pairwise sum of the rest), so
 * row_ptr / col_idx / vals are bit-identical.  Indices must already be in
 * range (the caller validates, with the reference's messages).  k = 1
 * handle, natural order. */
int csrk_coo_to_csr(int device, int64_t n_rows, int64_t n_cols, int64_t count,
                    const int64_t *rows, const int64_t *cols, const double *vals,
                    csrk_matrix **out);

/* Entry lines of a coordinate Matrix Market body (everything after the size
 * line), parsed on all host cores: rows / cols 0-based, vals (1.0 for
 * pattern files).  The loop of read_matrix_market (io.py:96-206) for large
 * files; strict -- a line outside the plain grammar, an out-of-range index,
 * a skew-symmetric diagonal or a count other than n_entries returns
 * CSRK_EINVAL, and the caller re-reads the body with the reference's loop
 * for the exact error. */
int csrk_mm_parse(const char *buf, int64_t len, int64_t n_entries, int with_value,
                  int64_t n_rows, int64_t n_cols, int skew, int64_t *rows, int64_t *cols,
                  double *vals);

/* Synthetic stencil generator writing canonical CSR on the device
 * (SURVEY.md §8(d)); shape = {nz, ny, nx} (nz = 1 for 2D), points = 5, 7, 27.
 * Produces a k = 1 handle (natural order). */
int csrk_stencil(int device, int64_t nz, int64_t ny, int64_t nx, int points,
                 csrk_matrix **out);
/* One rank's slab of a 3D stencil (7 or 27 points) for the row-block
 * partition (no reference counterpart -- the reference is
 * single-node): rows of planes [z0, z1), columns numbered from plane
 * max(z0 - 1, 0), so the handle's x is [lower halo plane | own planes |
 * upper halo plane] (halo planes only where the grid has them). */
int csrk_stencil_slab(int device, int64_t nz, int64_t ny, int64_t nx, int points,
                      int64_t z0, int64_t z1, csrk_matrix **out);

/* Give a handle uniform groups (k = 3): srs rows per super-row, ssrs
 * super-rows per super-super-row, the last of each shorter -- the
 * identity-permutation CSR-k of a generated stencil. */
int csrk_matrix_group_uniform(csrk_matrix *m, int64_t srs, int64_t ssrs);

/* ---- solvers around the SpMV -------------------
 * csrk_cg: `iters` conjugate-gradient iterations for A x = b from the x
 * given (device vectors of n_rows entries: b, x in/out, and scratch r, p,
 * ap), every SpMV the streaming kernel (variant / nx as csrk_spmv);
 * reductions in float64 with a fixed order (deterministic).  No host
 * synchronisation unless `scalars` is non-NULL (then out = r.r, alpha, beta,
 * p.Ap of the last iteration), so the call can be captured in a CUDA graph.
 * csrk_power: `iters` repeated SpMVs x <- A x / max|A x| (y is scratch). */
int csrk_cg(const csrk_matrix *m, int value_type, int variant, int nx,
            const void *b, void *x, void *r, void *p, void *ap, int iters,
            double *scalars, void *stream);
int csrk_power(const csrk_matrix *m, int value_type, int variant, int nx,
               void *x, void *y, int iters, void *stream);

/* Step kernels of the distributed CG (paper_2203_05096_b200.dist.DistCG;
 * no reference counterpart -- the C4 caller of spmv_csr3 at N GPUs).  Each
 * finishes its reduction on the device (the last block folds the per-block
 * partials in a fixed order: deterministic, one launch) into a caller-owned
 * device array `scalars` = {rr, pAp, rr_new, alpha, beta}, which the
 * caller's all-reduce updates in place between the calls:
 *   csrk_vec_dot(p, Ap -> &scalars[1])          then all-reduce scalars[1]
 *   csrk_cg_update(x += a p; r -= a Ap; rr_new)  then all-reduce scalars[2]
 *   csrk_cg_direction(p = r + b p; rr = rr_new)
 * `partials` holds >= 592 doubles, `counter` one zeroed unsigned (re-armed
 * by every call).  Stream-ordered, no host synchronisation. */
int csrk_vec_dot(int value_type, int64_t n, const void *a, const void *b, double *partials,
                 unsigned *counter, double *out, void *stream);
int csrk_cg_update(int value_type, int64_t n, void *x, void *r, const void *p,
                   const void *ap, double *scalars, double *partials, unsigned *counter,
                   void *stream);
int csrk_cg_direction(int value_type, int64_t n, void *p, const void *r, double *scalars,
                      unsigned *counter, void *stream);

/* ---- Band-k reordering (native) -------------------------------------------
 * Bit-exact native restatement of reorder.py (band_k 415-469 and its
 * helpers).  Results are held in an opaque object and read back with
 * csrk_bandk_result_get. */
int csrk_band_k(int64_t n, const uint32_t *row_ptr, const uint32_t *col_idx,
                int k, const double *targets, csrk_bandk_result **out);
/* sizes: out[0] = n, out[1] = len(level 1 sizes), out[2] = len(level 2) */
int csrk_bandk_result_sizes(const csrk_bandk_result *r, int64_t out[3]);
int csrk_bandk_result_get(const csrk_bandk_result *r, int64_t *fwd,
                          int64_t *sizes1, int64_t *sizes2);
int csrk_bandk_result_free(csrk_bandk_result *r);

/* Graph-level pieces of reorder.py on the reference's AdjacencyGraph arrays
 * (int64 CSR adjacency, reorder.py:35-58). */
/* heavy_edge_matching (reorder.py:138-173): match[n] */
int csrk_heavy_edge_matching(int64_t n, const int64_t *adj_ptr,
                             const int64_t *adj_idx,
                             const int64_t *edge_weight, int64_t *match);
/* weighted_bandwidth_order (reorder.py:281-336): fwd[n] */
int csrk_weighted_bandwidth_order(int64_t n, const int64_t *adj_ptr,
                                  const int64_t *adj_idx,
                                  const int64_t *node_weight, int64_t *fwd);
/* build_graph (reorder.py:115-135) and coarsen (reorder.py:199-237) return
 * an opaque graph (plus the fine-to-coarse map for coarsen) read back with
 * csrk_graph_sizes (out = n, adjacency length, f2c length) / csrk_graph_get. */
typedef struct csrk_graph csrk_graph;
int csrk_build_graph(int64_t n, const uint32_t *row_ptr,
                     const uint32_t *col_idx, csrk_graph **out);
int csrk_coarsen(int64_t n, const int64_t *adj_ptr, const int64_t *adj_idx,
                 const int64_t *edge_weight, const int64_t *node_weight,
                 double target, csrk_graph **out);
int csrk_graph_sizes(const csrk_graph *g, int64_t out[3]);
int csrk_graph_get(const csrk_graph *g, int64_t *adj_ptr, int64_t *adj_idx,
                   int64_t *edge_weight, int64_t *node_weight, int64_t *f2c);
int csrk_graph_free(csrk_graph *g);

/* ---- multi-GPU row blocks (SURVEY.md 8(b) csrk_mg_*, 8(e)) -----------------
 * The reference has no multi-GPU path; these generalise its static chunks
 * (kernels.py:150-155, _static_chunks: contiguous group ranges per worker)
 * from equal group counts to equal nonzeros, across one process per GPU.
 *
 * Host planning (no GPU; mirrors paper_2203_05096_b200.dist):
 *   csrk_mg_partition  -- cuts (parts + 1 global rows) on super-super-row
 *                         boundaries balancing nonzeros: part g starts at the
 *                         first SSR whose first nonzero offset reaches
 *                         ceil(g * nnz / parts) (dist.partition_by_nnz);
 *   csrk_mg_footprints -- per part the column window [lo, hi) its rows read
 *                         (fps: parts x 2; lo = hi = first row if empty);
 *   csrk_mg_plan       -- the transfers (src, dst, lo, hi), dst needing
 *                         x[lo, hi) owned by src (dist.halo_plan); out holds
 *                         cap x 4 entries, *count the full number.
 * Exchange + SpMV (NCCL loaded at run time from libnccl.so.2):
 *   csrk_mg_unique_id  -- rank 0 creates the communicator id (128 bytes) and
 *                         passes it to the other ranks by its own means;
 *   csrk_mg_create     -- rank `rank` of `world`: `block` is its rows
 *                         [cuts[rank], cuts[rank+1]) as a k = 3 csrk_matrix
 *                         (local rows / groups) whose columns are local to
 *                         x_local = x[x0, x0 + block->n_cols) (borrowed; it
 *                         must outlive the handle; NULL for a rank without
 *                         rows); mode CSRK_MG_HALO or CSRK_MG_ALLGATHER;
 *                         id NULL: no communicator -- the caller fills the
 *                         halo of x_local itself before csrk_mg_spmv;
 *   csrk_mg_spmv       -- y_own = A[r0:r1, :] x on `stream`: the exchange of
 *                         x_local's halo on an internal stream (NCCL send /
 *                         recv of exactly the windows each rank reads, or the
 *                         north-star all-gather), the interior tiles meanwhile,
 *                         the boundary tiles after it; x_local's owned slice
 *                         must be written (stream-ordered) before the call;
 *                         y_own is bitwise the single-GPU y;
 *   csrk_mg_info       -- out[9] = interior rows a, b, interior tiles t_lo,
 *                         t_hi, n_tiles, elements sent / received per step,
 *                         number of sends / receives. */
#define CSRK_MG_HALO 0
#define CSRK_MG_ALLGATHER 1
#define CSRK_MG_ID_BYTES 128
typedef struct csrk_mg csrk_mg;
int csrk_mg_partition(const uint32_t *row_ptr, const uint32_t *sr_ptr,
                      const uint32_t *ssr_ptr, int64_t n_ssr, int parts,
                      int64_t *cuts);
int csrk_mg_footprints(const uint32_t *row_ptr, const uint32_t *col_idx,
                       const int64_t *cuts, int parts, int64_t *fps);
int csrk_mg_plan(int world, const int64_t *cuts, const int64_t *fps,
                 int64_t *out, int64_t cap, int64_t *count);
int csrk_mg_unique_id(unsigned char *id);
int csrk_mg_create(int rank, int world, const unsigned char *id,
                   const int64_t *cuts, const int64_t *fps, csrk_matrix *block,
                   int64_t x0, int mode, csrk_mg **out);
int csrk_mg_spmv(csrk_mg *h, int value_type, int variant, int nx, void *x_local,
                 void *y_own, void *stream);
int csrk_mg_info(const csrk_mg *h, int64_t *out);
int csrk_mg_destroy(csrk_mg *h);

#ifdef __cplusplus
}
#endif
#endif /* CSRK_H */
