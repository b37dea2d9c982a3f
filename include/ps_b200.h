/*
 * ps_b200.h -- C ABI of libps_b200.so, the B200-native (sm_100a) FastPoint
 * sampling path.
 *
 * Every entry point replaces one operator of the reference package's kernel
 * layer, /root/reference/pkg/src/pointsample/_kernels.py (cited as
 * _kernels.py:L), or one SPEC-level operation that the reference specifies
 * but does not ship (SPEC.md:L).  The reference binds its kernels as numba
 * functions over numpy arrays; INTEGRATION.md shows the ctypes stub that a
 * maintainer adds to bind these instead.
 *
 * Conventions
 *   - All array arguments are DEVICE pointers (cudaMalloc / torch CUDA
 *     tensors).  `stream` is a cudaStream_t passed as void* (NULL = legacy
 *     default stream).  Calls are stream-ordered and never synchronise the
 *     host unless stated.
 *   - A batch of B clouds with N points each is stored as xyz4 =
 *     float[B][N][4] (x, y, z, unused): coordinates are float32, exactly as
 *     the reference's PointCloud stores them (core.py:176-191); every
 *     index-deciding distance is evaluated in float64 without FMA,
 *     ((dx*dx + dy*dy) + dz*dz), the operand order of _kernels.py:55-58.
 *   - Exclusion lists are per-cloud CSR: indptr int64[B][N+1] (offsets
 *     relative to the cloud's slice), nbr int32[B][cap_entries],
 *     d2 float64[B][cap_entries], rows ordered by (d2, index), self included;
 *     level counts int32[B][L][N] = #row entries with d2 < r2_level.
 *   - Return value: PS_OK (0) or a negative PS_ERR_* code; ps_last_error()
 *     gives the message.  Callers map PS_ERR_INVALID to ValueError and the
 *     rest to RuntimeError (the reference raises ValueError for argument
 *     errors, core.py:88, 141, 184-189).  Kernels never abort the process.
 */
#ifndef PS_B200_H
#define PS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define PS_API __attribute__((visibility("default")))
#else
#define PS_API
#endif

#define PS_OK 0
#define PS_ERR_INVALID (-1)
#define PS_ERR_CUDA (-2)
#define PS_ERR_UNSUPPORTED (-3)

/* ABI version (bumped on any signature change). */
PS_API int ps_version(void);
/* Message for the last failing call on this host thread. */
PS_API const char* ps_last_error(void);
/* Number of kernel launches issued through this library since load. */
PS_API int64_t ps_launch_count(void);

/* ---- K1: exact FPS -------------------------------------------------------
 * ps_fps_loop replaces fps_loop (_kernels.py:35-74): runs iterations
 * k_start..n_total-1 in place for every cloud.  md, taken, out_idx, curve
 * carry the caller's state exactly as in the reference (md squared float64
 * min-distances, taken u8, out_idx[k_start-1] = last sample).  k_start_dev
 * (int64[B], nullable) overrides k_start per cloud; clouds whose k_start is
 * >= n_total only write md/taken back.  out_idx / curve have row stride
 * ld_out.  Duplicate fallback of _kernels.py:65-70 included. */
PS_API int ps_fps_loop(const float* xyz4, int64_t B, int64_t N, double* md, uint8_t* taken,
                int64_t* out_idx, double* curve, int64_t ld_out, int64_t k_start,
                const int64_t* k_start_dev, int64_t n_total, void* stream);

/* Fresh exact FPS (SPEC.md:124-132 baselines.fps; SPEC.md:238-246
 * curve.extract_prefix when k_stop < n_total): initialises md = +inf,
 * taken = {seed}, out_idx[0] = seed, curve[0] = +inf and runs iterations
 * 1..k_stop-1.  seed_dev (int64[B], nullable) overrides `seed`. */
PS_API int ps_fps(const float* xyz4, int64_t B, int64_t N, double* md, uint8_t* taken,
           int64_t* out_idx, double* curve, int64_t ld_out, int64_t k_stop, int64_t seed,
           const int64_t* seed_dev, void* stream);

/* ---- K1 point-split: one cloud split over G ranks --
 * Rank g owns the original indices [g*ceil(N/G), (g+1)*ceil(N/G)) of each of
 * the B clouds; every iteration each rank reduces its shard in one
 * thread-block cluster, publishes the shard record (md, index, taken, xyz)
 * into every rank's mailbox (peer memory over NVLink, 32 bytes, sequence
 * tagged) and reduces the G records with the rule of the chunked merge in
 * fps_update_chunk / first_untaken (_kernels.py:77-100; max md, lowest
 * index; duplicate fallback = lowest untaken index) -- bit-identical to
 * fps_loop for any G.  A launch runs Gl ranks starting at g_base: Gl == G
 * puts all ranks on this GPU ("virtual ranks"), Gl == 1 is one rank per GPU.
 * mbox_dev: device array of G device pointers, mailbox g of
 * ps_fps_mailbox_bytes(B, G) bytes, filled with 0xff before first use;
 * seq_base + k_stop must stay below 2^32 - 1 and grow by >= k_stop + 1
 * between launches sharing the mailboxes.  all_write: every rank writes
 * out_idx / curve (one process per GPU), else rank 0 only.  Fresh FPS as
 * ps_fps; md / taken are written for each rank's own shard. */
PS_API int64_t ps_fps_mailbox_bytes(int64_t B, int32_t G);
PS_API int ps_fps_split_plan(int64_t N, int64_t B, int32_t G, int32_t Gl, int32_t* C_out, int32_t* P_out);
PS_API int ps_fps_split(const float* xyz4, int64_t B, int64_t N, double* md, uint8_t* taken, int64_t* out_idx,
                        double* curve, int64_t ld_out, int64_t k_stop, int64_t seed, int32_t G, int32_t g_base,
                        int32_t Gl, void* const* mbox_dev, uint32_t seq_base, int32_t all_write, void* stream);
/* Throughput hint for the exact-FPS dispatch (ps_fps / ps_fps_loop): the
 * number of clouds the caller keeps in flight across concurrent streams
 * (0 = latency mode, the default).  Above the launch's own batch, the
 * cluster width is chosen to cover the most SMs with that many clouds
 * instead of minimising one cloud's latency; results are identical.
 * Returns the previous value; process-wide, read at launch (and baked into
 * a captured graph). */
PS_API int64_t ps_set_fps_inflight(int64_t clouds);

/* fps_loop (_kernels.py:35-74) resumed from a partial state over the same
 * point split: iterations [k_start, n_total) (k_start_dev: per-cloud int64
 * device values, e.g. the sampler's reached counts) continue from md/taken
 * (valid on the launching ranks' shards) and out_idx/curve[0 .. k_start)
 * (replicated); the early-termination tail of FastPoint at C5.  Tags as
 * ps_fps_split: seq_base + iteration, unique per mailbox use. */
PS_API int ps_fps_split_loop(const float* xyz4, int64_t B, int64_t N, double* md, uint8_t* taken,
                             int64_t* out_idx, double* curve, int64_t ld_out, int64_t k_start,
                             const int64_t* k_start_dev, int64_t n_total, int32_t G, int32_t g_base, int32_t Gl,
                             void* const* mbox_dev, uint32_t seq_base, int32_t all_write, void* stream);
/* CUDA IPC for the mailboxes of one-process-per-GPU ranks: 64-byte handle of
 * a device allocation, opened in a peer process (peer access enabled).  The
 * handle describes a whole cudaMalloc allocation and opens at its base, so
 * mailboxes are allocated with ps_device_alloc (plain cudaMalloc, optionally
 * filled with fill_byte), not carved out of a caching allocator. */
PS_API int ps_device_alloc(int64_t bytes, int32_t fill_byte, void** dev_ptr_out);
PS_API int ps_device_free(void* dev_ptr);
PS_API int ps_ipc_handle(const void* dev_ptr, void* handle_out);
PS_API int ps_ipc_open(const void* handle, void** dev_ptr_out);
PS_API int ps_ipc_close(void* dev_ptr);

/* fps_update_chunk (_kernels.py:77-92) for one cloud: folds (px,py,pz) into
 * md[lo:hi] and writes the slice argmax (best float64, index int64; lowest
 * index on ties) to best_out[0], arg_out[0]. */
PS_API int ps_fps_update_chunk(const float* xyz4, int64_t N, double px, double py, double pz,
                        double* md, int64_t lo, int64_t hi, double* best_out,
                        int64_t* arg_out, void* stream);

/* Set-abstraction stage input: out4[b][t] = xyz4[b][idx[b][t]]
 * (float[B][n][4], w = 0) for t < n; idx int64 with row stride idx_ld. */
PS_API int ps_gather_xyz4(const float* xyz4, const int64_t* idx, int64_t idx_ld, int64_t B, int64_t N, int64_t n,
                          float* out4, void* stream);

/* first_untaken (_kernels.py:95-100): lowest j with taken[j] == 0, else -1. */
PS_API int ps_first_untaken(const uint8_t* taken, int64_t N, int64_t* out, void* stream);

/* ---- K3a/K3b: exclusion lists -------------------------------------------
 * Replaces excl_collect + csr_fill + csr_sort_rows + csr_level_counts
 * (_kernels.py:111-234; SPEC.md:394-402 build_exclusion_lists).  Every
 * unordered pair is evaluated once against r2max = max(r2_levels[b][:L]).
 * r2_levels float64[B][levels_ld].  `work` is a device buffer of
 * ps_excl_workspace_bytes(B, N, cap_edges) bytes; cap_edges bounds the
 * undirected edges per cloud and cap_entries the CSR entries per cloud
 * (< 2^31).  status int32[B] receives bit0 = edge overflow, bit1 = entry
 * overflow; an overflowed cloud's CSR is incomplete and must be rebuilt with
 * larger capacities.  method 0 enumerates the i<j triangle (each pair
 * evaluated once, the reference's accounting SPEC.md:438); method 1 enumerates
 * candidates from a uniform grid of cell width >= R_max (cap_edges unused) --
 * the CSR is byte-identical, only the number of evaluations differs.
 * method 2 (the FastPoint hot path) uses the same grid candidates but writes
 * fixed-stride rows: row i starts at indptr[i] = i * ps_excl_row_stride(N,
 * cap_entries), entries bucketed by level (each level's entries are the row
 * prefix of length counts[l][i]); a row longer than the stride takes a run
 * of the spill arena behind the N strided rows (indptr[i] then points
 * there), so only an exhausted arena sets status bit 1.  Consumers that take
 * a status pointer (sampler, rf queries) turn a failed cloud into explicit
 * error outputs instead of reading its incomplete rows. */
PS_API int64_t ps_excl_row_stride(int64_t N, int64_t cap_entries);
PS_API int64_t ps_excl_workspace_bytes(int64_t B, int64_t N, int64_t cap_edges, int32_t method);
/* Byte offset, inside a method-1 workspace, of the uint64[B] count of
 * candidate pairs the grid build evaluated (pair_evals accounting). */
PS_API int64_t ps_excl_grid_evals_offset(int64_t B, int64_t N);
PS_API int ps_excl_build(const float* xyz4, int64_t B, int64_t N, const double* r2_levels, int32_t L,
                  int64_t levels_ld, int64_t* indptr, int32_t* nbr, double* d2, int32_t* counts,
                  int64_t cap_entries, void* work, int64_t cap_edges, int32_t* status,
                  int32_t method, void* stream);

/* One rank's share of the method-2 build for a point split (MDPS
 * at C5): every point is a candidate, but only rows [row_lo, row_hi) are
 * written (their indptr, entries and counts) and rows longer than the
 * stride take spill entries [spill_lo, spill_hi) of the arena (offsets past
 * N * ps_excl_row_stride(N, cap_entries)), so G ranks with disjoint ranges
 * fill one CSR without coordination.  work: ps_excl_workspace_bytes(B, N, 1,
 * 2) bytes per rank; status as ps_excl_build. */
PS_API int ps_excl_build_shard(const float* xyz4, int64_t B, int64_t N, const double* r2_levels, int32_t L,
                               int64_t levels_ld, int64_t row_lo, int64_t row_hi, int64_t spill_lo,
                               int64_t spill_hi, int64_t* indptr, int32_t* nbr, double* d2, int32_t* counts,
                               int64_t cap_entries, void* work, int32_t* status, void* stream);

/* csr_fill (_kernels.py:164-185): scatter the M undirected edges (ei, ej
 * int32, ed float64; excl_collect's emission order) into both rows of a CSR
 * whose indptr (int64[N+1]) counts self + degree per row: row r = r (d2 0),
 * then the other endpoint of every edge touching r in edge order.  out_idx
 * int64[E], out_d2 float64[E].  work: ps_csr_fill_workspace_bytes(M, N)
 * device bytes (stable radix sort of the half-edges by row). */
PS_API int64_t ps_csr_fill_workspace_bytes(int64_t M, int64_t N);
PS_API int ps_csr_fill(const int32_t* ei, const int32_t* ej, const double* ed, int64_t M, const int64_t* indptr,
                       int64_t N, int64_t* out_idx, double* out_d2, void* work, int64_t work_bytes, void* stream);

/* csr_sort_rows (_kernels.py:188-219): order every row by (d2, index) in
 * place.  work: >= 256 + 4*B*N bytes. */
PS_API int ps_csr_sort_rows(int64_t* indptr, int32_t* nbr, double* d2, int64_t cap_entries, int64_t B,
                            int64_t N, void* work, void* stream);

/* csr_level_counts (_kernels.py:222-234) over an existing sorted CSR. */
PS_API int ps_level_counts(const int64_t* indptr, const double* d2, int64_t cap_entries, int64_t B,
                    int64_t N, const double* r2_levels, int32_t L, int64_t levels_ld,
                    int32_t* counts, void* stream);

/* ---- K2: curve estimate -> thresholds -----------------------------------
 * SPEC.md:258-266 estimate_power (mode 0, pow_tab[i] = i**e, float64[n]) or
 * a given estimated curve (mode 1, given_curve float64[B][given_ld]) on top
 * of the measured prefix curve[b][0..k0); SPEC.md:318-326 segment_thresholds
 * at d[s] (host int64[nseg]).  Writes R_out float64[B][nseg] and
 * r2_levels[b] = {max(R_s^2, 5e-324) for s < nseg} ++ extra_r2[0..n_extra). */
PS_API int ps_thresholds(const double* prefix_curve, int64_t curve_ld, int64_t B, int64_t k0,
                  int64_t n, int32_t nseg, const int64_t* d_host, int32_t mode,
                  const double* pow_tab, const double* given_curve, int64_t given_ld,
                  const double* extra_r2_host, int32_t n_extra, double* R_out,
                  double* r2_levels, int64_t levels_ld, void* stream);

/* SPEC.md:298-306 estimate_mlp + segment_thresholds: the measured prefix
 * curve[b][1..k0) resampled to 32 values and divided by curve[b][k0-1], a
 * 32-128-128-64 relu MLP (mlp_weights: device float64 W1[128][32], b1[128],
 * W2[128][128], b2[128], W3[64][128], b3[64], the SPEC.md:357 layer order),
 * outputs times curve[b][k0-1] resampled to the n-k0 tail positions, running
 * minimum from curve[b][k0-1]; then radii / levels as ps_thresholds.  Fixed
 * summation order (input order, bias last): bit-identical to the host
 * curve.estimate_mlp.  k0 >= 3. */
PS_API int ps_thresholds_mlp(const double* prefix_curve, int64_t curve_ld, int64_t B, int64_t k0, int64_t n,
                             int32_t nseg, const int64_t* d_host, const double* mlp_weights,
                             const double* extra_r2_host, int32_t n_extra, double* R_out, double* r2_levels,
                             int64_t levels_ld, void* stream);

/* ---- K3c: predicted-distance bitmap sampler ------------------------------
 * Replaces sample_predicted (_kernels.py:251-353).  out_idx[b][0..k0) holds
 * the FPS prefix on entry; entries [k0, n_total) are written (-1 beyond the
 * count reached).  seg_level_rows_host / boundaries_host are host arrays of
 * nseg entries; boundaries are segment ends and the last must equal n_total
 * (SURVEY 0.4).  state_io (uint64[B], device) is the splitmix64 state in/out.
 * work: ps_sampler_workspace_bytes(B, N, nseg) bytes.  excl_status (int32[B]
 * from ps_excl_build, nullable): a cloud whose build failed gets
 * out_idx[b][k0..n_total) = -1, reached[b] = n_total (nothing left for early
 * termination) and entered[b] = -1 -- an explicit error state that stays
 * visible through CUDA-graph replays. */
PS_API int64_t ps_sampler_workspace_bytes(int64_t B, int64_t N, int32_t nseg);
PS_API int ps_sample_predicted(const int64_t* indptr, const int32_t* nbr, int64_t cap_entries,
                        const int32_t* counts, int32_t L, const int32_t* seg_level_rows_host,
                        const int64_t* boundaries_host, int32_t nseg, int64_t* out_idx,
                        int64_t ld_out, int64_t k0, int64_t n_total, int64_t B, int64_t N,
                        uint64_t* state_io, int32_t pick_lowest, int64_t* reached,
                        int32_t* exhausted, int32_t* entered, void* work, const int32_t* excl_status,
                        void* stream);

/* ---- K3d: early termination ----------------------------------------------
 * earlyterm_scan (_kernels.py:356-367) over points [lo, hi) of every cloud:
 * md[i] = min(md[i], min{d2 of the first lvl1_counts[i] row entries j with
 * taken[j]}).  lvl1_counts int32 with cloud stride counts_stride. */
PS_API int ps_earlyterm_scan(const int64_t* indptr, const int32_t* nbr, const double* d2,
                      int64_t cap_entries, const int32_t* lvl1_counts, int64_t counts_stride,
                      const uint8_t* taken, double* md, int64_t B, int64_t N, int64_t lo,
                      int64_t hi, void* stream);

/* SPEC.md:415-423 early_termination set-up for clouds with reached[b] <
 * n_total: taken = {out_idx[b][0..reached)}, md = +inf, then the scan above.
 * Follow with ps_fps_loop(k_start_dev = reached) to finish the tail. */
PS_API int ps_early_termination_prepare(const int64_t* indptr, const int32_t* nbr, const double* d2,
                                 int64_t cap_entries, const int32_t* lvl1_counts,
                                 int64_t counts_stride, uint8_t* taken, double* md,
                                 const int64_t* out_idx, int64_t ld_out, const int64_t* reached,
                                 int64_t n_total, int64_t B, int64_t N, void* stream);

/* early_termination seeding for one rank of a point split: taken = the
 * first reached[b] samples (all N points), md = +inf and the level-1 row
 * pull of earlyterm_scan (_kernels.py:356-367) for the rank's points
 * [lo, hi) only -- the rows it built.  Continue with ps_fps_split_loop. */
PS_API int ps_early_termination_shard(const int64_t* indptr, const int32_t* nbr, const double* d2,
                                      int64_t cap_entries, const int32_t* lvl1_counts, int64_t counts_stride,
                                      uint8_t* taken, double* md, const int64_t* out_idx, int64_t ld_out,
                                      const int64_t* reached, int64_t n_total, int64_t B, int64_t N, int64_t lo,
                                      int64_t hi, void* stream);

/* ---- K4: grouping ---------------------------------------------------------
 * Outputs idx int32[B][n][k] (-1 padded), dist float64[B][n][k] (sqrt(d2),
 * NaN padded), cnt int32[B][n].  Order (d2, index), strict d2 < r^2. */
/* rf_ball_query: level = the level row the radius was baked
 * into; zero distance evaluations; k <= 128 (PS_ERR_INVALID otherwise).
 * A centroid outside [0, N), or any centroid of a cloud whose excl_status
 * (nullable) is nonzero, gets cnt = -1 and an empty (-1 / NaN) group. */
PS_API int ps_ball_query_rf(const int64_t* indptr, const int32_t* nbr, const double* d2,
                     int64_t cap_entries, const int32_t* counts, int32_t L, int32_t level,
                     const int64_t* centroids, int64_t cent_ld, int64_t B, int64_t N, int64_t n,
                     int32_t k, int32_t* idx_out, double* dist_out, int32_t* cnt_out,
                     const int32_t* excl_status, void* stream);
/* ball_query_naive; k <= 128. */
PS_API int ps_ball_query_naive(const float* xyz4, const int64_t* centroids, int64_t cent_ld, int64_t B,
                        int64_t N, int64_t n, double r2, int32_t k, int32_t* idx_out,
                        double* dist_out, int32_t* cnt_out, void* stream);
/* knn_naive: queries int64[B][q_ld] (NULL = 0..nq-1),
 * pool int64[B][pool_ld]; k <= 16. */
PS_API int ps_knn_naive(const float* xyz4, const int64_t* queries, int64_t q_ld, int64_t nq,
                 const int64_t* pool, int64_t pool_ld, int64_t npool, int64_t B, int64_t N,
                 int32_t k, int32_t* idx_out, double* dist_out, int32_t* cnt_out, void* stream);
/* rf_knn: level-1 rows filtered by sampled (u8[B][N]);
 * brute-force fallback over pool; fallback_count int32[B] is incremented.
 * A cloud whose excl_status (nullable) is nonzero gets cnt = -1 everywhere. */
PS_API int ps_knn_rf(const float* xyz4, const int64_t* indptr, const int32_t* nbr, const double* d2,
              int64_t cap_entries, const int32_t* lvl1_counts, int64_t counts_stride,
              const uint8_t* sampled, const int64_t* queries, int64_t q_ld, int64_t nq,
              const int64_t* pool, int64_t pool_ld, int64_t npool, int64_t B, int64_t N,
              int32_t k, int32_t* idx_out, double* dist_out, int32_t* cnt_out,
              int32_t* fallback_count, const int32_t* excl_status, void* stream);

/* ---- K6: quality -----------------------------------------------------------
 * avg_min_spacing helper: out_d2[b][s] = squared distance
 * from sample s to its nearest other sample. */
PS_API int ps_min_spacing(const float* xyz4, const int64_t* samples, int64_t ld, int64_t n, int64_t B,
                   int64_t N, double* out_d2, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PS_B200_H */
