/*
 * rfxc.h — C ABI of the B200 (sm_100a) RFX proximity library (librfxc.so).
 *
 * The reference has no C ABI: its kernel boundary is Numba flat-array calls
 * on caller-allocated numpy arrays.  Each entry point below
 * replaces one of those calls (or one numpy/scipy step of the same path);
 * the reference site is cited per function (paths relative to
 * /root/reference/pkg/src/rfx/).
 *
 * Conventions
 *   - Every pointer argument named d_* is DEVICE memory owned by the caller
 *     (torch tensors in the Python host layer); the library never frees or
 *     retains caller memory.  h_* pointers are host memory.
 *   - `stream` is a cudaStream_t passed as void*; every call is
 *     stream-ordered and asynchronous unless documented otherwise.
 *   - Return value: RFXC_OK (0) or an error status; rfxc_last_error()
 *     returns a thread-local message.  Python maps RFXC_EDATA -> DataError,
 *     RFXC_EBUDGET -> BudgetError, anything else -> RfxError
 *     (errors.py:4-19).
 *   - Layouts: codes "nb" = (n, B) int32 row-major, exactly
 *     LeafMembership.codes (proximity.py:73, :113-116); codes "tm" =
 *     (B, n) int32 tree-major (device-internal).  Values are the dataset
 *     matrix column-major (n, p), i.e. Dataset.values F-order
 *     (dataset.py:59-71).
 */
#ifndef RFXC_H
#define RFXC_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    RFXC_OK = 0,
    RFXC_EDATA = 1,    /* bad shapes / ranges        -> DataError   */
    RFXC_EBUDGET = 2,  /* device capacity exceeded   -> BudgetError */
    RFXC_ERUNTIME = 3, /* anything else              -> RfxError    */
    RFXC_ECUDA = 4     /* CUDA runtime failure       -> RfxError    */
};

/* Node layouts produced by rfxc_forest_pack. */
enum { RFXC_NODES_F32 = 0, /* 8 B/node, thresholds rounded down to f32 */
       RFXC_NODES_F64 = 1, /* 16 B/node, f64 thresholds             */
       RFXC_NODES_F32_NUMERIC = 2, /* traversal only: F32 records of a forest with
                                      no categorical column (no category test per node) */
       RFXC_NODES_F32_B2 = 3, /* F32 records in 32-byte two-level groups (host packer
                                 only): per tree [root, pad x3], then for every internal
                                 node x at even depth group0 = [L, R, L's children pair]
                                 and, if R is internal, group1 = [R (copy), pad, R's
                                 children pair]; x's record points at group0, bit fb+1
                                 = "R internal".  One 256-bit load per two levels.  The
                                 record count per tree depends on the shape: call
                                 rfxc_forest_pack_host with h_nodes = NULL first (fills
                                 h_node_off / h_leaf_counts only). */
       RFXC_NODES_F32_B2_NUMERIC = 4 /* traversal only: B2 records, no categorical column */ };

/* Output layouts of rfxc_pair_counts. */
enum { RFXC_UPPER_I32 = 0,  /* packed i<j rows [row_lo,row_hi), int32 counts      */
       RFXC_UPPER_F64 = 1,  /* packed i<j rows, count/B in f64 (FullTriangle)    */
       RFXC_BLOCK_I32 = 2   /* (row_hi-row_lo, n) int32, j>i counted, else 0     */ };

/* Bit 31 of a bucketed perm entry marks the first member of its leaf. */
#define RFXC_PERM_FIRST 0x80000000u

/* Quantisation modes (quantize.py:16). */
enum { RFXC_Q_F32 = 0, RFXC_Q_F16 = 1, RFXC_Q_I8 = 2, RFXC_Q_NF4 = 3 };

const char* rfxc_last_error(void);
int rfxc_version(void);
/* Device properties the host layer sizes grids with. */
int rfxc_device_info(int device, int* sm_count, int64_t* l2_bytes,
                     int64_t* smem_per_block_optin);

/* ----------------------------------------------------------------- K0/K1 */
/* Values: f64 column-major (n, p) -> f32 copy; *d_inexact set to 1 if any
 * value is not exactly representable in f32 (then use RFXC_NODES_F64).
 * Replaces nothing in the reference (its traversal reads f64,
 * _kernels.py:339); it is the precondition for the exact f32 compare. */
int rfxc_values_to_f32(const double* d_values, int64_t count, float* d_out,
                       int32_t* d_inexact, void* stream);

/* Flatten concatenated per-tree node arrays (forest.py:67-99 layout; child
 * ids tree-local; tree b owns nodes [node_off[b], node_off[b+1])) into the
 * packed traversal layout and compute leaf_counts (forest.py:91-93) and
 * leaf codes (forest.py:95-99).  Requires right == left + 1 for internal
 * nodes (trained trees satisfy it, _kernels.py:313-317; the host relays out
 * other trees first).  d_nodes: total_nodes * (8 | 16) bytes.  d_leaf_code
 * (nullable): explicit per-node leaf code, used for relaid-out trees whose
 * terminal order differs from the reference node order. */
int rfxc_forest_pack(const int8_t* d_status, const int32_t* d_split_var,
                     const double* d_threshold, const int64_t* d_cat_mask,
                     const int32_t* d_left, const int32_t* d_leaf_code,
                     const int64_t* d_node_off,
                     int32_t B, int64_t total_nodes, const uint8_t* d_col_cat,
                     int32_t p, int32_t layout, void* d_nodes,
                     int32_t* d_leaf_counts, void* stream);

/* Host-side packing (upload boundary, csrc/host/host_pack.cpp): the same
 * records as rfxc_forest_pack, built on the host from PER-TREE host arrays
 * (h pointer tables of length B: the reference's Tree fields, dtypes int8 /
 * int32 / f64 / int64 / int32 / int32) into a caller (pinned) buffer, so only
 * 8 or 16 B/node cross PCIe.  Trees with right != left + 1 are relaid out
 * breadth-first, keeping the reference leaf ordinals.  Also fills
 * h_node_off (B+1) and h_leaf_counts (B).  Synchronous, multi-threaded
 * (nthreads <= 0: all cores). */
int rfxc_forest_pack_host(const void* const* h_status, const void* const* h_split_var,
                          const void* const* h_threshold, const void* const* h_cat_mask,
                          const void* const* h_left, const void* const* h_right,
                          const int64_t* h_node_counts, int32_t B,
                          const uint8_t* h_col_cat, int32_t p, int32_t layout,
                          void* h_nodes, int64_t* h_node_off, int32_t* h_leaf_counts,
                          int32_t nthreads);

/* Host f64 -> f32 copy of the values with an exactness verdict
 * (*h_exact = 1 when every value is f32-representable). */
int rfxc_values_to_f32_host(const double* h_values, int64_t count, float* h_out,
                            int32_t* h_exact, int32_t nthreads);

/* K1 — leaf code of every sample in trees [tree_lo, tree_hi) into
 * d_codes_tm ((tree_hi - tree_lo) x n).  Replaces descend/descend_all
 * (_kernels.py:333-374) driven by leaf_membership (proximity.py:100-116).
 * d_values: f32 (layout F32) or f64 (layout F64) column-major (n, p). */
int rfxc_leaf_codes(const void* d_nodes, const int64_t* d_node_off,
                    int32_t layout, int32_t p, int32_t tree_lo, int32_t tree_hi,
                    const void* d_values, int64_t n, int32_t* d_codes_tm,
                    void* stream);

/* The same for samples [row_lo, row_hi) only (d_values and d_codes_tm keep
 * their full n stride). */
int rfxc_leaf_codes_rows(const void* d_nodes, const int64_t* d_node_off,
                         int32_t layout, int32_t p, int32_t tree_lo, int32_t tree_hi,
                         const void* d_values, int64_t n, int64_t row_lo, int64_t row_hi,
                         int32_t* d_codes_tm, void* stream);
/* Rows [row_lo, row_hi) of a column-major (n, p) host matrix (element size
 * elem bytes) into the same rows of the device copy, stream-ordered. */
int rfxc_h2d_rows(void* d_dst, const void* h_src, int64_t n, int64_t p, int32_t elem,
                  int64_t row_lo, int64_t row_hi, void* stream);

/* (rows, cols) int32 transpose: tm <-> nb layouts. */
int rfxc_transpose_i32(const int32_t* d_in, int64_t rows, int64_t cols,
                       int32_t* d_out, void* stream);
/* General form: d_out[map(c) * ld_out + r] = d_in[r * ld_in + c] for r < rows,
 * c < cols (map = identity when d_col_map is NULL).  The traversal uses it to
 * bring the codes of samples walked in leaf order back to sample order. */
int rfxc_transpose_i32_ex(const int32_t* d_in, int64_t rows, int64_t cols, int64_t ld_in,
                          int32_t* d_out, int64_t ld_out, const int32_t* d_col_map,
                          void* stream);

/* K1 helpers (no reference counterpart; traversal scheduling only): d_order (n)
 * = the samples grouped by their leaf code in d_codes (one tree, codes <
 * nleaf; d_scratch: nleaf ints), so a traversal tile's samples share paths;
 * the order inside a leaf is not reproducible and never changes a code.
 * rfxc_permute_rows_f32: d_Xp[f * n + j] = d_X[f * n + d_order[j]]
 * (column-major (n, p) values in that order). */
int rfxc_leaf_order(const int32_t* d_codes, int64_t n, int32_t nleaf, int32_t* d_order,
                    int32_t* d_scratch, void* stream);
int rfxc_permute_rows_f32(const float* d_X, int64_t n, int32_t p, const int32_t* d_order,
                          float* d_Xp, void* stream);

/* OOB votes (oob_votes_tree, _kernels.py:377-385; forest.py:287-290) from
 * the leaf codes: d_votes (n, C) int64 = #{trees b with d_inbag[b, i] == 0
 * whose leaf of sample i has class c}.  d_leaf_class: class of every leaf
 * (node_class of the terminal nodes in node order), indexed by
 * d_leaf_base[b] + code; d_inbag (Bl, n) int32 bootstrap counts. */
int rfxc_oob_votes(const int32_t* d_codes_tm, int64_t n, int32_t Bl,
                   const int64_t* d_leaf_base, const int32_t* d_leaf_class,
                   const int32_t* d_inbag, int32_t C, int64_t* d_votes, void* stream);

/* -------------------------------------------------------------------- K2 */
/* Stable per-tree sort of samples by leaf (the counting sort inside
 * accumulate_pair_counts[_block], _kernels.py:458-468, :491-501), done once
 * and reused by K3/K4: LSD radix over 8-bit leaf digits, one CTA per tree.
 * Inputs: codes_tm (Bl x n), leaf_base (Bl+1, int64, exclusive prefix of
 * leaf_counts), max_leaf_count.  Outputs: d_perm (Bl x n): samples of tree b
 * sorted by leaf, ascending within a leaf, the first member of every leaf
 * tagged with RFXC_PERM_FIRST; d_seg (leaf_base[Bl]+1): absolute start of
 * every leaf's run in d_perm (d_seg[last] = Bl*n; an empty leaf starts where
 * the next one does); *d_has_empty = 1 when some leaf has no member.
 * d_scratch: rfxc_bucket_scratch_bytes(n, Bl) bytes. */
int64_t rfxc_bucket_scratch_bytes(int64_t n, int32_t Bl);
int rfxc_bucket(const int32_t* d_codes_tm, int64_t n, int32_t Bl,
                const int64_t* d_leaf_base, int32_t max_leaf_count,
                uint32_t* d_perm, int64_t* d_seg, void* d_scratch,
                int32_t* d_has_empty, void* stream);
/* The same for trees [tree_lo, tree_hi) only (d_has_empty is not cleared;
 * the caller zeroes it once), so tree chunks can be bucketed as soon as
 * their codes exist.  d_scratch: rfxc_bucket_scratch_bytes(n, tree_hi -
 * tree_lo) bytes, private to the call until it completes. */
int rfxc_bucket_trees(const int32_t* d_codes_tm, int64_t n, int32_t Bl,
                      const int64_t* d_leaf_base, int32_t max_leaf_count,
                      int32_t tree_lo, int32_t tree_hi, uint32_t* d_perm, int64_t* d_seg,
                      void* d_scratch, int32_t* d_has_empty, void* stream);

/* -------------------------------------------------------------------- K3 */
/* Exact same-leaf co-occurrence counts for rows [row_lo, row_hi), j > i,
 * from codes_nb (n x B).  Replaces accumulate_pair_counts (:483-510) via
 * _pair_counts (proximity.py:159-185) + the /B of full_proximity
 * (proximity.py:200, IEEE f64 division) for RFXC_UPPER_F64, and
 * accumulate_pair_counts_block (:452-480) for RFXC_BLOCK_I32.
 * Packed layouts start at packed_index(row_lo, row_lo+1)
 * (proximity.py:59-61) relative to d_out. */
int rfxc_pair_counts(const int32_t* d_codes_nb, int64_t n, int32_t B,
                     int64_t row_lo, int64_t row_hi, int32_t layout,
                     void* d_out, const int32_t* d_gate, void* stream);

/* The same counts from the K2 buckets (the reference's per-leaf pair
 * formulation, accumulate_pair_counts _kernels.py:491-510): for every row i
 * and tree b, the members that follow i in its leaf's run of d_perm.
 * d_pos_nb (n x B) uint32: absolute index of sample i in d_perm for tree b
 * (rfxc_perm_positions, then rfxc_transpose_i32); d_codes_nb / d_seg /
 * d_leaf_base as for the sketch give the end of i's run.  d_perm: the K2 perm
 * (idx_bytes 4) or its 16-bit sample ids (idx_bytes 2, n <= 65536, from
 * rfxc_perm_positions).  Work ~ n*B + same-leaf
 * pairs instead of n^2*B/2; the host picks it when the same-leaf pairs
 * (rfxc_same_leaf_pairs) are a small fraction of n(n-1)/2*B.  B <= 4096.
 * Same layouts and output as rfxc_pair_counts. */
int rfxc_pair_counts_leaf(const uint32_t* d_pos_nb, const void* d_perm, int32_t idx_bytes,
                          const int32_t* d_codes_nb, const int64_t* d_seg,
                          const int64_t* d_leaf_base, int64_t n, int32_t B,
                          int64_t row_lo, int64_t row_hi, int32_t layout,
                          void* d_out, const int32_t* d_gate, void* stream);
/* d_gate (nullable, both K3 entry points, packed layouts only): the
 * device-side choice written by rfxc_pair_kernel_gate — rfxc_pair_counts
 * runs only if *d_gate == 0, rfxc_pair_counts_leaf only if *d_gate == 1, so
 * the host launches both and never waits for the choice.
 * rfxc_pair_kernel_gate: *d_gate = (*d_pairs <= share * n(n-1)/2 * B). */
int rfxc_pair_kernel_gate(const uint64_t* d_pairs, int64_t n, int32_t B, double share,
                          int32_t* d_gate, void* stream);
/* d_pos_tm (Bl x n) uint32: d_pos_tm[b*n + s] = index e with
 * d_perm[e] & ~RFXC_PERM_FIRST == s in tree b's row.  n*Bl < 2^32.
 * d_perm16 (nullable, n <= 65536): d_perm's sample ids as uint16. */
int rfxc_perm_positions(const uint32_t* d_perm, int64_t n, int32_t Bl,
                        uint32_t* d_pos_tm, uint16_t* d_perm16, void* stream);
/* *d_out = sum over leaves of s(s-1)/2, s = d_seg[g+1] - d_seg[g]. */
int rfxc_same_leaf_pairs(const int64_t* d_seg, int64_t leaves, uint64_t* d_out,
                         void* stream);

/* TriBlock tier routing (proximity.py:301-327) over packed int32 counts of
 * rows [row_lo,row_hi): two passes.  Pass 0 writes per-row counts of
 * hot (v >= tau) and cold (1e-6 < v < tau) entries into d_row_counts
 * (2 * rows int64).  Pass 1 takes the exclusive row offsets (d_row_offsets,
 * 2 * rows int64, same layout) and emits (i, j, v) sorted by (i, j). */
int rfxc_triblock_count(const int32_t* d_counts_upper, int64_t n, int32_t B,
                        int64_t row_lo, int64_t row_hi, double tau,
                        int64_t* d_row_counts, void* stream);
int rfxc_triblock_emit(const int32_t* d_counts_upper, int64_t n, int32_t B,
                       int64_t row_lo, int64_t row_hi, double tau,
                       const int64_t* d_row_offsets, int32_t* d_hot_i,
                       int32_t* d_hot_j, double* d_hot_v, int32_t* d_cold_i,
                       int32_t* d_cold_j, double* d_cold_v, void* stream);
/* Exclusive scan of int64 (single launch, any length). */
int rfxc_exclusive_scan_i64(const int64_t* d_in, int64_t count, int64_t* d_out,
                            int64_t* d_total, void* stream);

/* -------------------------------------------------------------------- K4 */
/* Standard normals of PCG32 stream (seed, seq) positions [0, count) as f64
 * (rng.py:102-115; stream jump-ahead so every thread starts mid-stream).
 * Replaces Pcg32(seed, SEQ_FACTOR).normals((n, k)) (proximity.py:392-393)
 * and Pcg32(seed + c, SEQ_POWER).normals(n) (mds.py:210-211). */
int rfxc_normals(int64_t seed, int64_t seq, int64_t count, double* d_out,
                 void* stream);

/* Row-major f64 (n, k) -> f32 (n, ld) with zero padding (sketch operand). */
int rfxc_pack_f32(const double* d_in, int64_t n, int32_t k, int32_t ld,
                  float* d_out, void* stream);

/* Leaf sums S[g, :] = sum_{i in leaf g} X[i, :] for global leaves
 * [g_lo, g_hi) (one phase of Mt @ X, proximity.py:394).  X: f32 (n, ld);
 * S: f32 ((g_hi - g_lo), ld). */
int rfxc_leaf_sums(const uint32_t* d_perm, const int64_t* d_seg, int64_t g_lo,
                   int64_t g_hi, const float* d_X, int32_t k, int32_t ld,
                   float* d_S, void* stream);

/* Gather Y[i, :] (+)= scale * sum_b S[leaf_base[b] + codes_nb[i, b], :]
 * over the Bl local trees (the M @ (.) phase, proximity.py:394).
 * Y: f64 (n, k).  accumulate != 0 adds into Y. */
int rfxc_leaf_gather(const int32_t* d_codes_nb, int64_t n, int32_t Bl,
                     const int64_t* d_leaf_base, const float* d_S, int32_t k,
                     int32_t ld, double scale, int32_t accumulate, double* d_Y,
                     void* stream);

/* One whole sketch pass Y = scale * sum_b E_b E_b^T X over the Bl local
 * trees (M @ (Mt @ X) of proximity.py:394, :397, :398 with M the
 * 1/sqrt(B)-scaled one-hot, so scale = 1/B) as one cooperative kernel:
 * trees in batches of T whose leaf sums stay in L2: per batch a leaf-sum
 * kernel and a gather kernel; with nbuf = 2 the leaf sums of batch e+1 run
 * on an auxiliary stream, overlapping the gather of batch e.  X: f32 (n, ld), ld = k
 * rounded up to 4 (k <= 128); Y: f64 (n, k).  rfxc_sketch_plan (host) picks
 * T so that two batches of leaf sums fit budget_bytes and sizes the
 * workspace; rfxc_sketch_prepare runs once per (bucketed membership, plan);
 * d_perm / d_seg / d_has_empty come from rfxc_bucket.  Deterministic. */
int rfxc_sketch_plan(const int32_t* h_leaf_counts, int32_t Bl, int64_t n, int32_t k,
                     int64_t budget_bytes, int32_t* T_out, int64_t* s_rows_out,
                     int32_t* nbuf_out, int64_t* work_bytes_out);
int rfxc_sketch_prepare(const int64_t* d_seg, const int64_t* d_leaf_base, int64_t n,
                        int32_t Bl, int32_t k, int32_t T, int64_t s_rows, int32_t nbuf,
                        void* d_work, void* stream);
int rfxc_sketch_pass(const uint32_t* d_perm, const int64_t* d_seg, const int32_t* d_codes_nb,
                     const int64_t* d_leaf_base, const int32_t* d_has_empty, int64_t n,
                     int32_t Bl, const float* d_X, int32_t k, int32_t ld, double scale,
                     int32_t T, int64_t s_rows, int32_t nbuf, double* d_Y, void* d_work,
                     void* stream);

/* -------------------------------------------------------------------- K5 */
/* C = A^T B for row-major f64 A (n, ka), B (n, kb): deterministic two-level
 * reduction (Gram of the QR steps, proximity.py:395-398, and
 * T = Q^T (P Q)).  d_partials: nparts * ka * kb f64, nparts from
 * rfxc_gram_parts().  Result C (ka x kb) row-major f64 on device. */
int rfxc_gram_parts(int64_t n);
int rfxc_gram(const double* d_A, const double* d_B, int64_t n, int32_t ka,
              int32_t kb, double* d_partials, double* d_C, void* stream);

/* Y (n, ka) times small M (ka, kb) -> Z (n, kb) f64; optional f32 copy
 * (n, ld32) for the next sketch pass (d_Z32 may be NULL). */
int rfxc_matmul_small(const double* d_Y, int64_t n, int32_t ka,
                      const double* d_M, int32_t kb, double* d_Z,
                      float* d_Z32, int32_t ld32, void* stream);

/* k x k steps of the basis / Rayleigh-Ritz (np.linalg.qr, proximity.py:395,
 * :397; np.linalg.eigh of T, proximity.py:399-403) on one CTA, k <= 110, so
 * the factorisation never waits on the host.  All matrices row-major f64.
 *   rfxc_orth_map: G = Y^T Y -> M (k x k): Q1 = Y M has orthonormal columns
 *     (eigen-directions of G, strongest first, scaled by l^-1/2; directions
 *     with l <= 1e-13 l_max become zero columns).
 *   rfxc_chol_inv: G + shift_rel tr(G) I = R^T R (Cholesky) -> R^-1 (upper;
 *     non-positive pivots give zero rows/columns).  Q = Y R^-1 is one
 *     CholeskyQR step; the basis is shifted CholeskyQR3 (first step shifted).
 *   rfxc_ritz_factor_map: T -> Wr (k x r) = W_r sqrt(clip(l_r, 0)), the
 *     top-r eigenpairs (descending) of the symmetrised T.
 *   rfxc_sym_eig: eigenvalues (descending) and eigenvectors (columns). */
int rfxc_orth_map(const double* d_G, int32_t k, double* d_M, void* stream);
int rfxc_chol_inv(const double* d_G, int32_t k, double shift_rel, double* d_Rinv, void* stream);
int rfxc_ritz_factor_map(const double* d_T, int32_t k, int32_t r, double* d_Wr, void* stream);
int rfxc_sym_eig(const double* d_A, int32_t k, double* d_w, double* d_V, void* stream);

/* -------------------------------------------------------------------- K6 */
/* factor = Q (n, k) @ Wr (k, r) followed by quantisation (quantize.py:83-117,
 * i8: per-column absmax/127, rint half-even, clip +-127).
 * d_factor: f64 (n, r) scratch/output; d_colmax_parts: rfxc_gram_parts(n)*r
 * f64; d_scales: r f64 (i8) / nblocks (nf4); d_data: mode-dependent output
 * (i8: int8 (n, r); f32; f16; nf4: packed uint8, column-major 64-blocks). */
int rfxc_factor_quantize(const double* d_Q, int64_t n, int32_t k,
                         const double* d_Wr, int32_t r, int32_t mode,
                         double* d_factor, double* d_colmax_parts,
                         double* d_scales, void* d_data, void* stream);

/* -------------------------------------------------------------------- K7 */
/* pmax (proximity.py:406-417): max over diag(dq dq^T) and 1024 sampled
 * off-diagonal pairs drawn on device from Pcg32(seed, SEQ_PMAX).
 * d_dq: dequantised factor f64 (n, r).  d_out: 1 f64. d_parts: scratch of
 * rfxc_gram_parts(n) f64. */
int rfxc_dequantize(const void* d_data, const double* d_scales, int64_t n,
                    int32_t r, int32_t mode, double* d_dq, void* stream);
int rfxc_pmax(const double* d_dq, int64_t n, int32_t r, int64_t seed,
              double* d_parts, double* d_out, void* stream);
/* The 2048 bounded draws Pcg32(seed, SEQ_PMAX).bounded(n) that rfxc_pmax
 * pairs up (i = draw 2t, j = draw 2t+1), exactly as the sampler inside
 * rfxc_pmax generates them (known-answer tests; proximity.py:409-417). */
int rfxc_pmax_draws(int64_t seed, int64_t n, uint32_t* d_out, void* stream);

/* ----------------------------------------------------------------- K8/K9 */
/* Factor-space MDS power iteration (mds.py:184-268) as one persistent
 * cooperative kernel: k eigenpairs, implicit deflation, Rayleigh quotient,
 * tol on max|v_new - v|, iteration cap, stop at lambda <= 0.  The Gram
 * matvec is gram_matvec (mds.py:161-181) on the UNclamped P = dq dq^T.
 * Outputs: d_coords (n, k) row-major f64 = sqrt(lambda) * sign_fixed v
 * (mds.py:257-261); d_info: per component {lambda, iterations, residual,
 * converged} as 4 f64; *d_k_used (int32).  d_work: rfxc_mds_work_bytes().
 * d_pmax (nullable): device copy of pmax (rfxc_pmax's output), read instead of
 * pmax so the launch needs no host round trip.
 * d_codes / d_scales (nullable): the INT8 factor; when given, large-n runs
 * keep the factor slice of every CTA resident in shared memory as int8
 * codes (code * scale is bit-identical to d_dq). */
int64_t rfxc_mds_work_bytes(int64_t n, int32_t r, int32_t k);
int rfxc_mds_power(const double* d_dq, const int8_t* d_codes, const double* d_scales,
                   int64_t n, int32_t r, double pmax, const double* d_pmax,
                   int32_t k, int32_t max_iterations, double tol, int64_t seed,
                   double* d_coords, double* d_info, int32_t* d_k_used,
                   void* d_work, void* stream);
/* One gram_matvec (mds.py:161-181): d_w = G v. */
int rfxc_gram_matvec(const double* d_dq, int64_t n, int32_t r, double pmax,
                     const double* d_v, double* d_w, void* d_work,
                     void* stream);

/* ------------------------------------------------------- outlier scores */
/* outlier_scores (proximity.py:432-485): score_i = mean over j != i of
 * 1 / max(p_ij, floor)^2.  FullTriangle: d_packed is the packed f64 upper
 * triangle (n(n-1)/2), d_work rfxc_outlier_work_bytes(n) bytes.  Low rank:
 * p_ij = clip(dq_i . dq_j, 0, 1) over the (n, r) f64 dequantised factor,
 * the diagonal term subtracted from the full row sum (:475-479).  Fixed-order
 * sums (bit-reproducible).  n >= 2, floor > 0, r <= ~100. */
int64_t rfxc_outlier_work_bytes(int64_t n);
int rfxc_outlier_packed(const double* d_packed, int64_t n, double floor_,
                        double* d_scores, void* d_work, void* stream);
int rfxc_outlier_lowrank(const double* d_dq, int64_t n, int32_t r, double floor_,
                         double* d_scores, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RFXC_H */
