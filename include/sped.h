/*
 * sped.h — C ABI of the B200-native SPED hot path (libsped.so, sm_100a).
 *
 * Plain pointers and sizes only.  Every array argument is DEVICE memory
 * (cudaMalloc / torch CUDA storage) unless its comment says "host".  Row-major
 * n x k fp32 blocks.  Every entry point is stream-ordered on `stream`
 * (a cudaStream_t passed as void*) and returns an sped_status; on error
 * sped_last_error() describes it.  The Python host layer maps
 * SPED_ERR_ARG / SPED_ERR_ZERO_DEGREE to the reference's ValueError.
 *
 * Reference interfaces replaced (paths relative to
 * /root/reference/pkg/src/specgap/):
 *   sped_canonicalize_edges    Graph.__post_init__               graph.py:64-88
 *   sped_laplacian_build       LaplacianOperator.__post_init__   graph.py:182-199
 *                              (+ Graph.degrees graph.py:118-122)
 *   sped_csr_poly_apply        TransformedOperator.apply         transforms.py:229-262
 *                              (ell x LaplacianOperator.matvec   graph.py:205-211)
 *   sped_edge_batch_poly_apply make_stochastic_oracle identity   solvers.py:166-178
 *                              (+ restated per-term composition)
 *   sped_csr_term_split        one term of the apply on a row shard (own-column
 *                              pass overlapping the halo exchange)
 *   sped_gram_mueg / sped_mueg_coeffs / sped_block_update
 *                              mu_eg_step                        solvers.py:121-144
 *   sped_persistent_mueg / sped_persistent_oja
 *                              run_solver's step loop            solvers.py:227-292
 *                              (whole steps per launch)          solvers.py:114-144
 *   sped_gram / sped_oja_coeffs (+ update)
 *                              oja_step + _orthonormalize        solvers.py:84-118
 *   sped_pcg64_integers        Generator(PCG64).integers(0,m,B)  solvers.py:171
 *   sped_kmeans_*              kmeans_cluster                    metrics.py:143-176
 *   sped_walk_index_build / sped_walk_poly_estimate
 *                              estimate_polynomial_matvec        walks.py:276-341
 *                              (edge incidence walks, Philox)    walks.py:175-273
 *   sped_gather_rows/scatter   (new) halo exchange staging for row-sharded L
 */
#ifndef SPED_H_
#define SPED_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* sped_stream_t;

enum sped_status {
  SPED_OK = 0,
  SPED_ERR_ARG = 1,          /* invalid argument -> ValueError */
  SPED_ERR_CUDA = 2,         /* CUDA runtime error -> RuntimeError */
  SPED_ERR_ZERO_DEGREE = 3,  /* normalized Laplacian with an isolated node (graph.py:187-188) */
  SPED_ERR_UNSUPPORTED = 4
};

const char* sped_last_error(void);
int sped_abi_version(void);

/* ---- graph -> Laplacian CSR (graph.py:182-199) --------------------------
 * u, v, w: canonical edge list (u < v, lexsorted, unique; graph.py:64-88),
 * int64/int64/fp64, m edges.  Outputs (caller-allocated, worst-case sizes):
 *   indptr  int32[n+1]
 *   indices int32[2m+n]      sorted columns, explicit diagonal (scipy layout)
 *   values  fp32[2m+n]       fp32(scipy fp64 value); may be NULL when
 *                            store_values == 0 (unweighted combinatorial:
 *                            kernels synthesise -1 / row_len-1)
 *   degrees fp64[n]          Graph.degrees() bit-exact (bincount order)
 *   epos    int32[2m]        CSR position of edge e's (u,v) entry at [2e] and
 *                            (v,u) entry at [2e+1] (stochastic path)
 * *nnz_out (host) receives nnz.  Synchronises `stream`.  normalized=1 with a
 * zero-degree node returns SPED_ERR_ZERO_DEGREE. */
int sped_laplacian_build(int64_t n, int64_t m, const int64_t* u, const int64_t* v,
                         const double* w, int normalized, int store_values,
                         int32_t* indptr, int32_t* indices, float* values,
                         double* degrees, int32_t* epos, int64_t* nnz_out,
                         sped_stream_t stream);

/* ---- one row shard of the same CSR (replaces slicing the
 * LaplacianOperator of graph.py:182-199 built whole on every rank) --------
 * Rows [row_begin, row_end) of sped_laplacian_build's CSR, bit for bit, from
 * any lexsorted subsequence of the canonical edge list that contains every
 * edge incident to those rows (other edges are ignored).  indices hold
 * GLOBAL column ids.  normalized + store_values needs col_degrees = every
 * node's degree (fp64[n]; the all-gather of the shards' `degrees`).
 *   indptr  int32[nr+1], indices/values capacity 2m+nr, degrees fp64[nr]
 *   (own rows, Graph.degrees order), epos int32[2m] (local CSR position of
 *   each input edge's two entries, -1 where the row is not in the shard).
 * Synchronises `stream`. */
int sped_laplacian_build_rows(int64_t n, int64_t row_begin, int64_t row_end, int64_t m,
                              const int64_t* u, const int64_t* v, const double* w,
                              const double* col_degrees, int normalized, int store_values,
                              int32_t* indptr, int32_t* indices, float* values,
                              double* degrees, int32_t* epos, int64_t* nnz_out,
                              sped_stream_t stream);

/* ---- graph canonicalisation (Graph.__post_init__, graph.py:64-88) -------
 * Drops w == 0 edges, orients u < v and sorts by (u, v) on the device (the
 * reference's lexsort, bit for bit: a radix sort of the unique keys u*n+v).
 * Outputs (device, capacity m) receive the *m_out (host) kept edges.
 * *status_out (host) is a bit set of the reference's ValueErrors: 1 negative
 * weight, 2 self loop, 4 endpoint out of range, 8 duplicate unordered pair;
 * outputs are only written when it is 0.  Synchronises `stream`. */
int sped_canonicalize_edges(int64_t n, int64_t m, const int64_t* u, const int64_t* v,
                            const double* w, int64_t* u_out, int64_t* v_out, double* w_out,
                            int64_t* m_out, int32_t* status_out, sped_stream_t stream);

/* ---- locality ordering for power-law graphs -----------------------------
 * perm (new -> old) lists nodes by descending row length (stable), iperm is
 * its inverse.  sped_relabel_edges maps the canonical edges through iperm and
 * re-canonicalises them (u2 < v2, lexsorted); edge_map[new] = old edge id. */
int sped_degree_order(int64_t n, const int32_t* indptr, int32_t* perm, int32_t* iperm,
                      sped_stream_t stream);
int sped_relabel_edges(int64_t n, int64_t m, const int64_t* u, const int64_t* v,
                       const double* w, const int32_t* iperm, int64_t* u2, int64_t* v2,
                       double* w2, int32_t* edge_map, sped_stream_t stream);

/* ---- long-row split plan for the SpMM ----------------------------------
 * Rows longer than long_threshold nonzeros are cut into chunks of chunk_len
 * processed by separate warps and combined deterministically.  chunk_desc is
 * int32[4*max_chunks] = {row, p_begin, p_end, first_chunk_of_row}.
 * Synchronises `stream` (returns the counts to the host). */
int64_t sped_spmm_plan_max_chunks(int64_t n, int64_t nnz, int32_t long_threshold,
                                  int32_t chunk_len);
int sped_spmm_plan(int64_t n, const int32_t* indptr, int32_t long_threshold,
                   int32_t chunk_len, int32_t* chunk_desc, int64_t max_chunks,
                   int64_t* n_chunks_out, int64_t* n_long_rows_out,
                   sped_stream_t stream);

/* ---- dilation-polynomial apply (transforms.py:229-262) -------------------
 * w_0 = w0_scale * (w_init ? w_init : x);  for t < n_terms:
 *     w_{t+1} = alpha[t]*x + beta[t]*(L w_t) + gamma[t]*w_t
 * out = lam_f*x + s_final*w_{n_terms}.
 * alpha/beta/gamma are HOST arrays of n_terms doubles.  w_a, w_b: n x k
 * scratch (ping-pong; may be NULL when n_terms <= 1 / 2 respectively).
 * long_threshold / chunk_len / chunk_desc / n_chunks: the sped_spmm_plan
 * (rows longer than long_threshold are chunk-processed; n_chunks == 0 means
 * no plan).  partials fp32[n_chunks*k] and tickets int32[n_chunks] (zero on
 * entry, left zero) serve the plan (NULL when n_chunks == 0).
 * segments: HOST int64[3*n_segments] = {row_begin, row_end, sub} row ranges,
 * each launched with rows handled by (k/4)*sub lanes (sub nonzero-parallel
 * lane groups per row); n_segments == 0 means one warp per row.  Gathered rows
 * with index < hot_rows are cached with L2 evict_last, others evict_first.
 * w_init (optional) lets a row shard start from its halo-extended block
 * while x stays its own rows.  x / w_init must not alias out, w_a or w_b.
 * row_scale (optional, fp32[n] = d_i^-1/2): the caller asserts L is the
 * normalized Laplacian of a unit-weight graph without self loops; terms after
 * the first then run on u = D^-1/2 w and skip the values stream (values must
 * still be given: the first term reads them).  Ignored for k not in
 * {4,...,128}, unaligned buffers or w_init. */
int sped_csr_poly_apply(int64_t n, int32_t k, const int32_t* indptr,
                        const int32_t* indices, const float* values,
                        int32_t long_threshold, int32_t chunk_len,
                        const int32_t* chunk_desc, int64_t n_chunks,
                        float* partials, int32_t* tickets,
                        const int64_t* segments, int32_t n_segments, int64_t hot_rows,
                        const float* row_scale,
                        const float* x, const float* w_init, float* w_a, float* w_b, float* out,
                        int32_t n_terms, const double* alpha, const double* beta,
                        const double* gamma, double w0_scale, double lam_f,
                        double s_final, sped_stream_t stream);

/* ---- split shard term (row-sharded L) ------------------------
 * One term of sped_csr_poly_apply's schedule on a row shard whose CSR is
 * split into the entries that read the shard's own rows (L_own) and those
 * that read halo rows (L_halo), so the halo exchange overlaps pass 0:
 *   raw_out = 1 (pass 0): out = L_own w                      (no epilogue)
 *   raw_out = 0 (pass 1): out = lam_f x + s_final (alpha x + beta w0 (L_halo w
 *                          + partial_in) + gamma w0 w)
 * w is the [own | halo] block (own rows first), x / out / partial_in the own
 * rows (n x k); values are required (stored fp32).  Replaces, per term, the
 * ell x LaplacianOperator.matvec of transforms.py:241-262 on one shard. */
int sped_csr_term_split(int64_t n, int32_t k, const int32_t* indptr, const int32_t* indices,
                        const float* values, int32_t long_threshold, int32_t chunk_len,
                        const int32_t* chunk_desc, int64_t n_chunks, float* partials,
                        int32_t* tickets, const int64_t* segments, int32_t n_segments,
                        const float* x, const float* w, const float* partial_in,
                        int32_t raw_out, float* out, double alpha, double beta, double gamma,
                        double w0_scale, double lam_f, double s_final, sped_stream_t stream);

/* General shard term: as sped_csr_term_split, plus
 *   - the scaled-normalized form of sped_csr_poly_apply for unit-weight
 *     normalized Laplacians: scaled_in = 1 means w holds u = D^-1/2 w (own
 *     AND halo rows -- the exchange moves u) and the neighbour sums are
 *     unweighted (values not read); scaled_out = 1 writes u' = D^-1/2 w';
 *     row_scale = d^-1/2 of the own rows (fp32);
 *   - a persisting-L2 window over rows [hot_begin, hot_begin + hot_rows) of
 *     w (the hub rows: the own prefix on the shard that owns the hubs, the
 *     head of the halo elsewhere); hot_rows = 0: none.
 * With raw_out = 1 and partial_in = NULL on a split CSR this is pass 0; an
 * unsplit shard (no halo) runs one pass with partial_in = NULL. */
int sped_csr_term_shard(int64_t n, int32_t k, const int32_t* indptr, const int32_t* indices,
                        const float* values, int32_t long_threshold, int32_t chunk_len,
                        const int32_t* chunk_desc, int64_t n_chunks, float* partials,
                        int32_t* tickets, const int64_t* segments, int32_t n_segments,
                        const float* row_scale, int32_t scaled_in, int32_t scaled_out,
                        int64_t hot_begin, int64_t hot_rows, const float* x, const float* w,
                        const float* partial_in, int32_t raw_out, float* out, double alpha,
                        double beta, double gamma, double w0_scale, double lam_f,
                        double s_final, sped_stream_t stream);

/* ---- edge-minibatch apply (solvers.py:166-178, per term) ----------------
 * Term t replaces L w by (m/B) * sum_{b<B} w_e x_e x_e^T w over the sampled
 * edge ids batch[t*B .. t*B+B) (int32, the numpy rng.integers stream).
 * edge_w fp32[m] (NULL = unit weights) are the RAW graph weights, exactly as
 * the reference's identity oracle uses g.w (also in normalized mode).
 * epos int32[2m] = the CSR positions of each edge's two entries (the entry's
 * CSR column is the neighbour); -1 marks an entry this call does not own.
 * erow int32[2m] (optional) = the row of each entry; NULL derives it from the
 * partner entry's column (whole graph; a row shard must pass it).  workspace
 * >= sped_edge_batch_workspace_bytes(n, B).  w_init (optional) is the term-0
 * input with halo rows appended (row shards), x stays the own rows; neither
 * may alias out / w_a / w_b.  Deterministic (sorted records, no float
 * atomics). */
int64_t sped_edge_batch_workspace_bytes(int64_t n, int64_t B);
/* Workspace for sorting all n_terms terms' records at once (one
 * bandwidth-bound radix sort by (term, row) instead of n_terms small ones;
 * same summation order, bit-identical output).  sped_edge_batch_poly_apply
 * takes that path whenever workspace_bytes is at least this size and the
 * keys fit in int32; otherwise it sorts per term, overlapping term t+1's
 * sort with term t's sweep on a side stream.  SPED_STO_ALLTERMS=0 /
 * SPED_STO_OVERLAP=0 switch either off. */
int64_t sped_edge_batch_workspace_bytes_terms(int64_t n, int64_t B, int32_t n_terms);
int sped_edge_batch_poly_apply(int64_t n, int32_t k, int64_t m, const int32_t* indices,
                               const float* edge_w, const int32_t* epos, const int32_t* erow,
                               const int32_t* batch, int64_t B, void* workspace,
                               int64_t workspace_bytes, const float* x, const float* w_init,
                               float* w_a, float* w_b, float* out, int32_t n_terms,
                               const double* alpha, const double* beta, const double* gamma,
                               double w0_scale, double lam_f, double s_final,
                               sped_stream_t stream);

/* As sped_edge_batch_poly_apply with the estimator scale given explicitly:
 * a row shard passes its COMPACTED batch (only the samples with an endpoint
 * in the shard, in sample order, as indices into its local edge arrays of
 * m local edges) and scale = m_global / B_global, so its rows get the
 * single-GPU arithmetic while sorting O(B / P) records.  B may be 0 (no
 * sampled endpoint in the shard: epilogues only); B > 0 needs n_terms <= 1. */
int sped_edge_batch_poly_apply_scaled(int64_t n, int32_t k, int64_t m, const int32_t* indices,
                                      const float* edge_w, const int32_t* epos,
                                      const int32_t* erow, const int32_t* batch, int64_t B,
                                      double scale, void* workspace, int64_t workspace_bytes,
                                      const float* x, const float* w_init, float* w_a, float* w_b,
                                      float* out, int32_t n_terms, const double* alpha,
                                      const double* beta, const double* gamma, double w0_scale,
                                      double lam_f, double s_final, sped_stream_t stream);

/* ---- solver step pieces (solvers.py:84-144) -----------------------------
 * sped_gram: G fp64[3*k*k] = {S = V^T V, C = V^T M, Q = M^T M} (M may be
 * NULL: only S).  workspace: sped_gram_workspace_bytes(n, k) bytes. */
size_t sped_gram_workspace_bytes(int64_t n, int32_t k);
int sped_gram(int64_t n, int32_t k, const float* V, const float* M, double* G,
              void* workspace, size_t workspace_bytes, sped_stream_t stream);
/* As sped_gram with M required, for mu-EG, which reads S, C and diag(Q)
 * only: at k = 128 the Q block's MMAs are skipped (diag(Q) is summed in fp64
 * from the converted M values; Q's off-diagonal entries come back 0).  Other
 * k: identical to sped_gram.  Replaces the V^T MV / column-norm work of
 * mu_eg_step, solvers.py:121-144. */
int sped_gram_mueg(int64_t n, int32_t k, const float* V, const float* M, double* G,
                   void* workspace, size_t workspace_bytes, sped_stream_t stream);
/* mu-EG k x k algebra: A = I - eta*(triu(C,1) + diag d),
 * scale_i = 1/||W_i||.  flag int32[1]: set to 1 if a column norm < 1e-12
 * (rank collapse, solvers.py:136-143); left unchanged otherwise. */
int sped_mueg_coeffs(int32_t k, const double* G, double eta, float* A, float* scale,
                     int32_t* flag, sped_stream_t stream);
/* Oja/CholQR k x k algebra: with_m=1: Gram of W = V + eta*M from {S,C,Q};
 * with_m=0: Gram = S.  T = R^{-1} for R = chol(Gram)^T (upper), fp32. */
int sped_oja_coeffs(int32_t k, const double* G, double eta, int32_t with_m, float* T,
                    int32_t* flag, sped_stream_t stream);
/* Grid-resident fast path (k <= 32): `steps` whole mu-EG steps in ONE
 * cooperative launch (one CTA per SM; polynomial terms exchange rows through
 * generation-tagged 64-bit words instead of grid barriers, grid barriers only
 * around the Gram; state in HBM/L2).  V (n x k) is updated in place; flag
 * bit 0 is set when a column's norm vanishes (rank collapse,
 * solvers.py:136-143), bit 1 when a tagged wait timed out (a bug, never
 * expected); SPED_ERR_UNSUPPORTED for k > 32 or > 256 terms.  `nnz` =
 * indptr[n] (host copy, sizes the launch); `workspace` of at least
 * sped_persistent_workspace_bytes(n, k) bytes, ZEROED before its first use
 * and kept across launches (two fp32 and two tagged n x k blocks, Gram
 * partials, the tag base). */
int sped_persistent_workspace_bytes(int32_t n, int32_t k, int64_t* bytes);
/* As sped_persistent_mueg, for oja_step (solvers.py:114-118): W = V + eta
 * p(L)V orthonormalised by CholQR2 (two Gram / Cholesky / R^{-1} rounds, the
 * MGS of _orthonormalize, solvers.py:84-102); flag set when a Cholesky pivot
 * is not positive (rank collapse). */
int sped_persistent_oja(int32_t n, int32_t k, int64_t nnz, const int32_t* indptr,
                        const int32_t* indices, const float* values, int32_t n_terms,
                        const double* alpha, const double* beta, const double* gamma,
                        double w0_scale, double lam_f, double s_final, double eta, int32_t steps,
                        float* V, int32_t* flag, void* workspace, int64_t workspace_bytes,
                        sped_stream_t stream);
int sped_persistent_mueg(int32_t n, int32_t k, int64_t nnz, const int32_t* indptr,
                         const int32_t* indices, const float* values, int32_t n_terms, const double* alpha,
                         const double* beta, const double* gamma, double w0_scale,
                         double lam_f, double s_final, double eta, int32_t steps, float* V,
                         int32_t* flag, void* workspace, int64_t workspace_bytes,
                         sped_stream_t stream);
/* ---- walk-based polynomial estimator (walks.py) ---------------------------
 * sped_walk_index_build: from the canonical lexsorted edge list (u < v,
 * int64, device) the incidence index: up_start[n+1] (edges with u == x are
 * ids [up_start[x], up_start[x+1])), lo_start[n+1] and sorted_e[m] (the ids
 * stably sorted by v; node x's v-run is sorted_e[lo_start[x] .. lo_start[x+1])).
 * sped_walk_poly_estimate: for each of the k columns of x (fp64 n x k,
 * row-major) one estimate of sum_i coeffs[i] L^i x_j (mode 0, importance,
 * walks.py:311-341) or of L^ell x_j / (N p_min) with coeffs = e_ell (mode 1,
 * rejection, walks.py:276-308) from `walks` walks of length ell on the edge
 * incidence graph; keys = uint64[k][ceil(walks/8192)][2], the Philox keys of
 * SeedSequence((seed_j, chunk)) (walks.py:196-198).  coeffs is a HOST array of
 * ell+1 doubles; deg_star_inc = 2 * max unweighted degree - 1 (rejection).
 * The walks reproduce numpy's Philox draws bit for bit; out is fp64. */
int64_t sped_walk_index_workspace_bytes(int64_t n, int64_t m);
int sped_walk_index_build(int64_t n, int64_t m, const int64_t* u, const int64_t* v,
                          int32_t* up_start, int32_t* lo_start, int32_t* sorted_e,
                          void* workspace, int64_t workspace_bytes, sped_stream_t stream);
int64_t sped_walk_workspace_bytes(int64_t n, int32_t k, int64_t walks);
int sped_walk_poly_estimate(int64_t n, int64_t m, int32_t k, const int64_t* u, const int64_t* v,
                            const double* w, const int32_t* up_start, const int32_t* lo_start,
                            const int32_t* sorted_e, int32_t ell, const double* coeffs,
                            int32_t mode, int64_t deg_star_inc, int64_t walks,
                            const uint64_t* keys, const double* x, double* out, void* workspace,
                            int64_t workspace_bytes, sped_stream_t stream);

/* out = (P*A + M*B) * diag(scale).  A k x k fp32; M may be NULL; B may be
 * NULL meaning B = eta*I; scale may be NULL (ones).  upper != 0 promises A is
 * upper triangular (mu-EG), letting the SIMT kernels skip the zero half.
 * k = 128 without B runs on the tensor cores (tcgen05 3xTF32, ~1e-6
 * relative; SPED_UPDATE_TC=0 selects the SIMT kernel). */
int sped_block_update(int64_t n, int32_t k, const float* P, const float* A,
                      const float* M, const float* B, double eta, const float* scale,
                      int32_t upper, float* out, sped_stream_t stream);
/* out = a*x + b*y elementwise over count floats (y may be NULL). */
int sped_axpby(int64_t count, double a, const float* x, double b, const float* y,
               float* out, sped_stream_t stream);

/* ---- bit-exact numpy PCG64 + Lemire (solvers.py:171) ---------------------
 * Reproduces Generator(PCG64).integers(0, m, size=count) (m < 2^32) from the
 * bit generator state (host scalars).  out int32[count].  On return
 * *draws32_out (host) = number of 32-bit draws consumed, so the caller can
 * advance its host generator.  workspace: sped_pcg64_workspace_bytes(count). */
size_t sped_pcg64_workspace_bytes(int64_t count);
int sped_pcg64_integers(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                        uint64_t inc_lo, int32_t has_uint32, uint32_t uinteger,
                        uint64_t m, int64_t count, int32_t* out, int64_t* draws32_out,
                        void* workspace, size_t workspace_bytes, sped_stream_t stream);
/* The same draw with the generator state resident in DEVICE memory:
 * state_words[6] = {state_hi, state_lo, inc_hi, inc_lo, has_uint32, uinteger}
 * (numpy's bit_generator.state), advanced in place on the stream; nothing
 * waits on the host, so the call is CUDA-graph capturable.  *status (device,
 * may be NULL) gets bit 0 if the candidate pool ran out (state unchanged).
 * Replaces the per-call rng.integers of solvers.py:171 with the stream kept
 * on the GPU; the host Generator is re-synchronised from the words lazily. */
int sped_pcg64_integers_device(uint64_t* state_words, uint64_t m, int64_t count,
                               int32_t* out, int32_t* status, void* workspace,
                               size_t workspace_bytes, sped_stream_t stream);

/* ---- k-means on the embedding (metrics.py:143-176) ----------------------- */
int sped_kmeans_assign(int64_t n, int32_t d, int32_t c, const float* X,
                       const double* centers, int32_t* labels, double* sums,
                       int64_t* counts, double* min_d2, sped_stream_t stream);
int sped_row_dist2(int64_t n, int32_t d, const float* X, const double* center,
                   double* dist, int32_t accumulate_min, sped_stream_t stream);

/* ---- halo staging for row-sharded L (multi-GPU) ------------------------- */
int sped_gather_rows(int64_t count, int32_t k, const int32_t* rows, const float* src,
                     float* dst, sped_stream_t stream);

/* ---- debug-check builds (-DSPED_DEBUG_CHECKS=1) ----------------------------
 * sped_debug_checks() is 1 in such a build; sped_debug_take() returns and
 * clears the OR of the device-side check bits (gather out of the input
 * block 1, hub-chunk ticket overflow 2, CSR position outside its row 4,
 * stochastic record out of range 8).  Synchronises the device.  Always 0 in
 * release builds. */
int sped_debug_checks(void);
unsigned int sped_debug_take(void);

#ifdef __cplusplus
}
#endif

#endif /* SPED_H_ */
