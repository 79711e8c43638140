/*
 * mvamg_b200.h -- C ABI of libmvamg_b200.so, the B200 (sm_100a) solve phase of
 * the composite bootstrap / multi-vector aggregation AMG of arXiv 1907.04417.
 *
 * The reference (`mvamg`, pure Python + numba) has no FFI; its drop-in surface
 * is the duck-typed operator API that this ABI sits under:
 *   - preconditioner slot   pcg(A, b, precond, rtol, itmax, x0, callback)
 *                           pkg/src/mvamg/krylov.py:28            -> mvamg_pcg_*
 *   - operator object       MultigridOperator(...).apply / error_propagation
 *                           pkg/src/mvamg/cycles.py:100-190       -> mvamg_hierarchy_*
 *   - composite slot        apply_composite_symmetrized(composite, x)
 *                           pkg/src/mvamg/bootstrap.py:98-113     -> mvamg_composite_*
 *   - sparse kernels        spmv / galerkin_product / a_norm
 *                           pkg/src/mvamg/sparse.py:30,50,69      -> mvamg_csr_*
 *   - smoother kernels      gs_forward / gs_backward
 *                           pkg/src/mvamg/_kernels.py:15-38       -> mvamg_gs_*
 * The ctypes binding a maintainer adds on the reference side is in
 * INTEGRATION.md; the in-tree binding is paper_1907_04417_b200/_lib.py.
 *
 * Conventions: plain C types only.  Matrices are CSR with int32 indptr/indices
 * and fp64 values (scipy's layout for < 2^31 nonzeros).  Pointers documented as
 * "device" must be CUDA device memory owned by the caller (PyTorch tensors in
 * the Python host layer); the library never frees caller memory.  `stream` is a
 * cudaStream_t passed as void*.  Every call returns 0 on success or a nonzero
 * MVAMG_E* code; mvamg_last_error() returns a thread-local message.
 */
#ifndef MVAMG_B200_H
#define MVAMG_B200_H

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes --------------------------------------------------------- */
#define MVAMG_OK 0
#define MVAMG_E_ARG 1          /* bad argument / dimension mismatch (ValueError)  */
#define MVAMG_E_CUDA 2         /* CUDA runtime failure                            */
#define MVAMG_E_NOT_SPD 3      /* Krylov breakdown / zero diagonal (NotSpdError) */
#define MVAMG_E_TIMEOUT 4      /* GS dependency wait exceeded its bound           */
#define MVAMG_E_STATE 5        /* call out of order (workspace not bound, ...)    */

/* device status word bits (mvamg_pcg_* status_out) */
#define MVAMG_ST_RZ_BREAKDOWN 1    /* r'z <= 0   krylov.py:46-47,68-69 */
#define MVAMG_ST_PQ_BREAKDOWN 2    /* p'Ap <= 0  krylov.py:54-55       */
#define MVAMG_ST_FCG_BREAKDOWN 4   /* FCG p'Ap <= 0  krylov.py:101-102 */
#define MVAMG_ST_GS_TIMEOUT 8

/* smoother kinds (cycles.py:24-26) and cycle kinds (cycles.py:43-52) */
#define MVAMG_GS_FORWARD 0
#define MVAMG_GS_BACKWARD 1
#define MVAMG_WEIGHTED_JACOBI 2
#define MVAMG_CYCLE_V 0
#define MVAMG_CYCLE_K 1

int mvamg_version(void);
const char* mvamg_last_error(void);
/* Kernels launched by this library since the last reset (CUDA-graph replays
 * count every kernel node).  Host-side counter, for the benchmark's
 * gpu_launches figure. */
int mvamg_kernel_launches(long long* count, int reset);
/* Diagnostics: when trace_dev (device, 8 x long long per warp of the largest GS
 * launch, zeroed by the caller) is non-NULL, GS sweeps accumulate per-warp
 * rounds / progress rounds / cycles.  NULL (default) disables tracing. */
int mvamg_gs_set_trace(long long* trace_dev);

/* ---- GS schedule analysis (host) -------------------------------------------
 * Splits the rows of a CSR matrix (host arrays) into dependency chains
 * (maximal runs where row i couples to row i-1, at most max_chain rows) and
 * groups consecutive chains into tiles of <= max_threads (<= 1024) chains whose
 * position-major shared window (threads x longest chain slots) fits
 * max_window slots.  Call first with the out arrays
 * NULL to get counts, then with arrays of nchains+1 / ntiles+1 ints.
 * chain_order (nchains ints, or NULL for the natural order): the processing
 * order of the chains -- tiles (and warps) are ranges of it, e.g. 2-D blocks
 * of the grid lines of a 3-D problem, so that most line-to-line dependences
 * stay inside a tile's shared window.
 * Replaces nothing in the reference (numba runs rows serially,
 * _kernels.py:15-38); the schedule preserves that order's dependency DAG, so
 * the sweep result is bit-identical.                                          */
int mvamg_gs_analyse(int n, const int* indptr, const int* indices, int max_chain,
                     int max_threads, int max_window, int* nchains, int* ntiles,
                     int* chain_ptr, int* tile_ptr, int* threads_out, int* window_out,
                     int* depth_out, const int* chain_order);

/* ---- stream-level kernels (device pointers) ------------------------------- */
/* y = A x  (sparse.py:30-40; scipy csr_matvec order, bit-exact). */
int mvamg_csr_spmv_f64(int n, const int* indptr, const int* indices, const double* data,
                       const double* x, double* y, void* stream);
/* r = b - A x  (cycles.py:156 inner term). */
int mvamg_csr_residual_f64(int n, const int* indptr, const int* indices, const double* data,
                           const double* b, const double* x, double* r, void* stream);
/* y = y + (A x)  (cycles.py:170, prolongation; sum formed first). */
int mvamg_csr_spmv_add_f64(int n, const int* indptr, const int* indices, const double* data,
                           const double* x, double* y, void* stream);
/* The three SpMV forms with the matrix's nnz (mode 0: y = A x, 1: y = b - A x,
 * 2: y = y + A x; sparse.py:30-40, cycles.py:156,170).  Knowing nnz, small
 * matrices with long rows (n <= 65,536, >= 4 entries per row on average, the
 * cycle's coarse levels) run one warp per row: a row's products are formed in
 * parallel and added in CSR order, bit-identical to the forms above. */
int mvamg_csr_spmv_mode_f64(int mode, int n, int nnz, const int* indptr, const int* indices, const double* data,
                            const double* x, const double* b, double* y, void* stream);
/* GS static round schedule (host).  For sweep `mode` (0 forward from x = 0,
 * 1 forward from a nonzero guess, 2 backward) and the chains / tiles of
 * mvamg_gs_analyse, assigns every row a round inside its warp (one more than
 * its chain predecessor and every same-warp row it depends on) and writes the
 * row records round-major, lane-minor (word w of lane L of global round g at
 * round_off[g] + 32 w + L): [cnt | flags][diag][RN(1/diag)] then cnt pairs
 * [coefficient][source code] -- the entries still contributing to the serial
 * loop's sum at sweep time, in CSR order.  Rounds of a warp are padded to a
 * multiple of R; uniform_S > 0 pads every round to that many words (the lean
 * kernel's fixed record size).  rows_per_round = K > 1 (lean records only)
 * lets a row share its chain predecessor's round (up to K rows of a lane per
 * round, K slots of S words each, slot-major) when every other intra-warp
 * input comes from an earlier round.  perm[i] = 32 * (K * global round + slot)
 * + lane.  Query with
 * rec == NULL for *nwords / *nrounds / *nwarps / *max_S; then round_off holds
 * nrounds+1, tbase nwarps+1, tile_wbase ntiles+1, perm n ints.  chain_order:
 * as in mvamg_gs_analyse (every inter-warp input must lie in an earlier warp
 * of that order; MVAMG_E_ARG otherwise).  wpos > 0 (a power of two; one-warp
 * tiles): the shared window keeps chain positions modulo wpos -- 32 x wpos
 * slots instead of 32 x the chain length, so several tiles fit an SM -- and
 * every window read is verified to come before its slot's next write. */
int mvamg_gs_schedule(int n, const int* indptr, const int* indices, const double* data, int ntiles,
                      const int* chain_ptr, const int* tile_ptr, int window, int mode, int R,
                      int uniform_S, int rows_per_round, long long* nwords, int* nrounds, int* nwarps,
                      int* max_S, unsigned long long* rec, int* round_off, int* tbase, int* tile_wbase,
                      int* perm, const int* chain_order, int wpos);
/* One lexicographic GS sweep (_kernels.py:15-38) on device data.  direction
 * 0 = forward, 1 = backward; x_old is the iterate before the sweep (NULL for a
 * zero guess); x_new receives the result and must not alias x_old.  The CSR
 * matrix is read by the backward sweep from a nonzero guess (old upper
 * neighbours folded into the right-hand side).  tperm: device buffer of
 * 32 * nrounds doubles.  R (rounds per chunk: 1, 2, 4, 8), D (ring slots:
 * 2, 4, 8), slot_words (>= R*(32*max_S+32), even) and rec_words_max
 * (R*32*max_S) size the per-warp TMA ring.  lean_C > 0 selects the lean
 * kernel: records built with uniform_S = 3 + 2*C, no x_old sources,
 * (R, D) in {(8,3), (8,2), (4,4), (4,2), (2,8), (2,2), (1,8)}; lean_C = C | K << 8 with
 * K > 1 rows per lane per round (C <= 4, (R, D, K) in {(2,2,4), (2,3,4),
 * (4,2,2)}).  ws: device
 * int workspace (>= 4 ints: tile ticket, status word).  Bit-identical to the
 * serial loop. */
int mvamg_gs_sweep_f64(int direction, int n, const int* indptr, const int* indices, const double* data,
                       const unsigned long long* rec, const int* round_off, const int* tbase,
                       const int* tile_wbase, const int* perm, double* tperm, int R, int D,
                       int lean_C, int slot_words, int rec_words_max, int ntiles,
                       const int* chain_ptr, const int* tile_ptr, const int* chain_order, int threads,
                       int window, int wpos, const double* b, const double* x_old, double* x_new, int* ws,
                       void* stream);
/* GS level-set schedule for small / mid-size levels (host).  mode 0 forward
 * from x = 0, 1 forward, 2 backward from x = 0, 3 backward.  Rows are
 * block-partitioned over a cluster of ncta (1..16) CTAs and, per CTA, ordered
 * by the level of the sweep's dependency DAG.  rows_out receives n 32-byte
 * records {int row, estart, cnt, pad; double diag, RN(1/diag)}, ents_out the
 * entries {double coef; int src (owner CTA << 26 | local row), pad} of every
 * row in CSR order, lev_ptr / lev_eptr ncta x (nlev+1) offsets, perm the
 * layout position of each row.  Levels whose per-CTA rows or entries exceed
 * row_cap / ent_cap (0 = unlimited) are split into cluster-uniform sub-levels
 * (the staging buffer's capacity).  Query with rows_out == NULL first. */
int mvamg_gs_levels(int n, const int* indptr, const int* indices, const double* data, int mode, int ncta,
                    int row_cap, int ent_cap, int* nlev, long long* nents, int* max_rows, int* max_ents,
                    int* rows_per_cta, int* lev_ptr, int* lev_eptr, void* rows_out, void* ents_out,
                    int* perm);
/* One GS sweep of a small / mid-size level on one thread-block cluster: x
 * resident in (distributed) shared memory, one cluster barrier per level set.
 * group = 1: one thread per row, bit-identical to the serial loop; group = 2,
 * 4, 8 or 16: that many lanes per row with a shuffle-tree sum (same order of
 * rows, tolerance parity); group | 0x100 with ncta = 1: the register-prefetch
 * variant (only x in shared memory, each level's entries loaded into
 * registers while the previous level computes; schedules built unsplit).  tperm: n + 2 doubles of device scratch;
 * ws: >= 4 device ints. */
int mvamg_gs_level_sweep_f64(int direction, int n, const int* indptr, const int* indices,
                             const double* data, int ncta, int rows_per_cta, int nlev, int max_rows,
                             int max_ents, int threads, int group, const int* lev_ptr, const int* lev_eptr,
                             const void* rows, const void* ents, const int* perm, double* tperm,
                             const double* b, const double* x_old, double* x_new, int* ws, void* stream);
/* Streamed level-set GS plan for one SM (csrc/gs_stream.cuh) -- replaces the
 * serial gs_forward / gs_backward loops of pkg/src/mvamg/_kernels.py:15-38 on
 * coarse levels whose x (and, for a sweep from x_old, b) fit in shared memory.
 * mode: 0 forward from x = 0, 1 forward from x_old, 2 backward from x = 0,
 * 3 backward from x_old.  Rows are batched by their level in the sweep's
 * dependency DAG and the batches packed, in sweep order, into stages of at
 * most slot_bytes per CTA.  ncta > 1 (zero-guess modes 0 and 2 only): a
 * thread-block cluster of that many CTAs, CTA c holding rows [c R, (c+1) R),
 * R = ceil(n / ncta), and reading the others' x over DSMEM.  Call with blob ==
 * NULL to get *blob_bytes and *nstages, then with a host blob of that size and
 * stage_off of nstages * ncta + 1 entries. */
int mvamg_gs_stream_plan(int n, const int* indptr, const int* indices, const double* data, int mode,
                         int slot_bytes, int ncta, long long* blob_bytes, int* nstages, int* nlevels,
                         unsigned char* blob, long long* stage_off);
/* One GS sweep with a stream plan (device blob and stage offsets): ncta CTAs
 * of 256 threads (one, or a cluster), x in shared memory, nslots stages of the plan in flight by TMA
 * bulk copies.  group = 1: one thread per row, bit-identical to the serial
 * loop; 2, 4, 8, 16: lanes per row with an FMA / shuffle-tree sum (tolerance
 * parity).  x_old is read only by modes 1 and 3. */
int mvamg_gs_stream_sweep_f64(int n, int mode, int nstages, int nslots, int slot_bytes, int group, int ncta,
                              const void* blob, const long long* stage_off, const double* b,
                              const double* x_old, double* x_new, void* stream);
/* Backward GS sweep from x_old with a mode-2 (backward, zero guess) stream
 * plan: t = b - (old lower neighbours) in CSR order into tfold (n doubles),
 * then the zero-guess sweep on t -- bit-identical to the serial loop with
 * group 1.  ws: >= 4 device ints. */
int mvamg_gs_stream_sweep_folded_f64(int n, const int* indptr, const int* indices, const double* data, int nstages,
                                     int nslots, int slot_bytes, int group, int ncta, const void* blob,
                                     const long long* stage_off, double* tfold, const double* b,
                                     const double* x_old, double* x_new, int* ws, void* stream);
/* Backward GS sweep from x_old with the mode-2 (backward, zero guess) level
 * schedule: the old upper neighbours are folded into the right-hand side
 * first (same roundings), so the sweep reads only new values. */
int mvamg_gs_level_sweep_folded_f64(int n, const int* indptr, const int* indices, const double* data,
                                    int ncta, int rows_per_cta, int nlev, int max_rows, int max_ents,
                                    int threads, int group, const int* lev_ptr, const int* lev_eptr,
                                    const void* rows, const void* ents, const int* perm,
                                    double* tperm, const double* b, const double* x_old,
                                    double* x_new, int* ws, void* stream);
/* GS dataflow row schedule for mid-size coarse levels (host).  mode as in
 * mvamg_gs_levels.  Rows are put in topological order of the sweep's DAG
 * (level, then longest row first); position p holds row rowid[p] with cnt[p]
 * entries, diagonal dg[p] and RN(1/diag) rdg[p]; perm[row] = p; crit[p] =
 * e1 | e2 << 16 (0xffff = none): the entry whose input is published last (the
 * highest DAG level) and the latest one at least two levels earlier -- the
 * kernel waits on e2, forms every published product, then waits on e1.  Entries
 * (entry_order 0: CSR order, bit-exact with the serial sweep; 1: by the DAG
 * level at which each input becomes final, old values first -- tolerance
 * parity; zero-guess modes keep only the DAG direction) are stored per
 * warp of 32 positions as an ELL slice: entry u of position 32w + l at
 * (wofs[w] + u) * 32 + l, padded to the warp's longest row; src is the row of
 * the value, with bit 31 set for an x_old value (modes 1 and 3).  Query with
 * rowid == NULL first (*nslots = total slice rows, so coef / src hold
 * 32 * nslots elements; wofs holds ceil(n/32) + 1 ints).  row_lo, row_hi:
 * only rows [row_lo, row_hi) become positions (-1, -1: all); the others are
 * external inputs -- the ghosts of a row-partitioned level -- read, never
 * written (perm still holds n entries; the position arrays row_hi - row_lo). */
int mvamg_gs_rows(int n, const int* indptr, const int* indices, const double* data, int mode, int entry_order,
                  long long* nslots, int* nlev, int* rowid, int* cnt, int* crit, double* dg, double* rdg,
                  int* perm, int* wofs, double* coef, int* src, int row_lo, int row_hi);
/* One GS sweep with a row schedule of `mode` (gs_row_kernel: one thread per
 * row over the whole GPU, x_new itself as the ready flag, each row's CSR-order
 * chain advanced as its inputs are published).  A mode-2 schedule with x_old
 * runs the folded backward sweep.  threads 32..128 per CTA, ctas resident
 * CTAs (0 = one per SM); max_tile_slots = the largest slice-row count of any
 * `threads`-position tile (its entries are staged in 384 * max_tile_slots
 * bytes of shared memory).  Bit-identical to the serial loop.  tperm: n
 * doubles of scratch; ws: >= 2 device ints (ticket, status). */
int mvamg_gs_row_sweep_f64(int mode, int n, const int* indptr, const int* indices, const double* data,
                           const int* rowid, const int* cnt, const int* crit, const double* dg, const double* rdg,
                           const int* perm, const int* wofs, const double* coef, const int* src,
                           int threads, int ctas, int max_tile_slots, double* tperm, const double* b,
                           const double* x_old, double* x_new, int* ws, void* stream);
/* Cluster dataflow sweep (gs_cluster_kernel): the sweep's rows in topological
 * order, one warp per row, run by ONE thread-block cluster of ncta CTAs (1, 2,
 * 4, 8 or 16) x wpc worker warps (1..32) with the iterate in the cluster's
 * distributed shared memory: a row is published by a local st.shared and
 * polled with ld.shared::cluster, so no dependency crosses L2 (a few hundred
 * ns per DAG level instead of ~1.4 us).  Replaces pkg/src/mvamg/_kernels.py:
 * 15-38 on coarse levels whose x fits the cluster (8 bytes per row, spread
 * over the CTAs' shared memory).  Same row
 * order as the serial loop; row sums in a fixed tree (reproducible, tolerance
 * parity -- not the CSR-order roundings).
 * mvamg_gs_cluster_plan (host): the rows in topological (DAG level) order
 * are dealt to the ncta * wpc worker warps (worker g = warp * ncta + cta) --
 * a row to the CTA owning its latest input while that CTA holds no more than
 * its share of the row's level (*local_late = rows so placed), round-robin
 * over that CTA's warps -- and stored worker by worker (q = a row's index in
 * that storage; rows wptr[g] .. wptr[g+1]; rowid: q -> row, perm: row -> q) as
 * row records packed into pages of page_bytes (a multiple of 128; pages
 * wpage[g] .. wpage[g+1], which the warp streams through shared memory with
 * TMA bulk copies).  Page: int nrows, 12 bytes of padding, then records {int
 * cnt, early, row, slot; double diag, RN(1/diag); cnt coefficients; cnt
 * sources; padding to 16 bytes}; a record's entries are ordered by the DAG level of their
 * inputs (old values first), entries early .. cnt-1 (same, last level, at
 * most 4) being its late tail; source = cta << 24 | slot of the value, or
 * bit 31 | row for an x_old value (modes 1, 3).  Query with blob == NULL
 * first (*npages, *nlev DAG levels, *slots_per_cta 8-byte x slots per CTA);
 * MVAMG_E_ARG when a row's record does not fit a page.
 * grid != 0: the grid form -- the same workers on ncta ordinary CTAs (1 ..
 * the SM count, all resident), early inputs and other CTAs' late inputs
 * polled in x_new through L2, only a late input of the row's own CTA in
 * shared memory; sources are then the input's row, or bit 30 | slot for such
 * a local late input, and only rows polled that way get an x slot (slot -1
 * otherwise). */
int mvamg_gs_cluster_plan(int n, const int* indptr, const int* indices, const double* data, int mode, int grid,
                          int ncta, int wpc, int page_bytes, long long* npages, int* nlev, int* slots_per_cta,
                          int* local_late, int* wptr, int* wpage, int* rowid, int* perm, void* blob);
/* One sweep (device pointers; a mode-2 plan with x_old runs the folded
 * backward sweep).  Shared memory per CTA: 8 * slots + 2 * wpc * (page_bytes +
 * 8).  sleep_ns: back-off of a warp whose poll found nothing new.  tperm: n
 * doubles of scratch; ws: >= 2 device ints (ticket, status). */
int mvamg_gs_cluster_sweep_f64(int mode, int n, const int* indptr, const int* indices, const double* data,
                               const int* wptr, const int* wpage, const void* blob, const int* perm, int grid,
                               int ncta, int wpc, int slots, int page_bytes, int sleep_ns, double* tperm,
                               const double* b, const double* x_old, double* x_new, int* ws, void* stream);
/* Pipelined sweep of one rank of a row-partitioned level (distributed.py;
 * SURVEY.md 8(e)): a row schedule of mode 0 / 2 built with row range
 * [row_lo, row_hi) = the own rows of the extended layout [lower ghosts | own |
 * upper ghosts] (n_ext rows; indptr covers all, ghost rows empty).  Ghost
 * inputs are polled in x_ext at system scope: their owners' kernels store them
 * there over NVLink the moment they are final (mirror_dst[mirror_ptr[p]..] =
 * peer << 24 | slot into peers[peer], device pointers from mvamg_ipc_open), so
 * the exact-order sweep runs as one wavefront across the ranks instead of a
 * rank-by-rank relay.  Own and ghost slots of x_ext must hold the sentinel
 * (all-ones bytes) when any rank starts; x_old_ext (mode 2 only) folds the old
 * lower neighbours into the right-hand side first.  ws: >= 2 device ints. */
int mvamg_gs_row_sweep_ext_f64(int mode, int n_ext, int row_lo, int row_hi, const int* indptr, const int* indices,
                               const double* data, const int* rowid, const int* cnt, const int* crit,
                               const double* dg, const double* rdg, const int* wofs, const double* coef,
                               const int* src, int threads, int ctas, int max_tile_slots, double* tperm,
                               const double* b_own, const double* x_old_ext, double* x_ext,
                               const int* mirror_ptr, const unsigned* mirror_dst, double* const* peers,
                               int* ws, void* stream);
/* CUDA IPC of a device buffer: its 64-byte handle, and open / close of a
 * peer's (the extended x a rank's mirror stores go to). */
int mvamg_ipc_handle(const void* dptr, void* handle64);
int mvamg_ipc_open(const void* handle64, void** dptr);
int mvamg_ipc_close(void* dptr);
/* z = Inv r, Inv dense row-major n x n (coarsest solve; cycles.py:88-97). */
int mvamg_dense_gemv_f64(int n, const double* inv, const double* r, double* z, void* stream);
/* *result = x . y (deterministic two-level reduction; device scalar).
 * ws: device workspace of >= 1024 doubles + 1 int (mvamg_dot_ws_bytes()). */
int mvamg_dot_f64(int n, const double* x, const double* y, double* result, void* ws, void* stream);
int mvamg_dot_ws_bytes(void);

/* ---- setup helpers (host) --------------------------------------------------- */
/* Greedy vertex-disjoint acceptance of edges in the given sorted order
 * (pkg/src/mvamg/_kernels.py:41-61): partner[v] = matched vertex or -1. */
int mvamg_greedy_match(long long ne, const long long* ei, const long long* ej, int n, long long* partner,
                       long long* pair_i, long long* pair_j, long long* npairs);
/* The same matching on the GPU (device pointers; A symmetric CSR, diag its
 * diagonal, w the smooth vector): partner[v] = matched vertex or -1.  Rounds of
 * best-edge picks with mutual picks matched (the locally dominant matching,
 * equal to the greedy order's result; matching.cuh).  Edge weights are
 * computed as pkg/src/mvamg/matching.py:99-102 with one rounding per operation.
 * Synchronises `stream` once per round; *rounds_out = rounds. */
int mvamg_greedy_match_device(int n, const int* indptr, const int* indices, const double* data,
                              const double* diag, const double* w, double weight_floor, int* partner,
                              int* rounds_out, void* stream);
/* Batched one-sided Jacobi thin SVD of stacked row-major blocks
 * (pkg/src/mvamg/svd.py:17-55, _kernels.py:64-121): U (same layout as A) and
 * sigma (nblk x k, descending).  On non-convergence returns MVAMG_E_NOT_SPD
 * with *failed_block set (SvdConvergenceError in the Python layer). */
int mvamg_jacobi_svd_batch(int nblk, const int* row_ptr, int k, const double* A, int max_sweeps,
                           double tol, double* U, double* sigma, int* failed_block);
/* The same batched SVD on the GPU (device pointers row_ptr, A, U, sigma; k <= 16;
 * one thread per block, svd.cuh): U and sigma bit-identical to
 * mvamg_jacobi_svd_batch.  *failed_block (host) = the smallest non-converged
 * block, as the host loop reports the first.  Synchronises `stream` once. */
int mvamg_jacobi_svd_batch_device(int nblk, const int* row_ptr, int k, const double* A, int max_sweeps,
                                  double tol, double* U, double* sigma, int* failed_block, void* stream);

/* ---- row-partitioned solve: halo packing, Krylov updates -- */
/* dst[i] = src[idx[i]] (pack a halo message) / dst[idx[i]] = src[i] (unpack). */
int mvamg_gather_f64(int n, const int* idx, const double* src, double* dst, void* stream);
int mvamg_scatter_f64(int n, const int* idx, const double* src, double* dst, void* stream);
/* y = y + (alpha * x)  (krylov.py:57-58) and y = x + (beta * y)  (krylov.py:70). */
int mvamg_axpy_f64(int n, double alpha, const double* x, double* y, void* stream);
int mvamg_xpby_f64(int n, const double* x, double beta, double* y, void* stream);

/* ---- Galerkin product (setup) -------------------------- */
/* Device CSR owned by the library. */
typedef struct mvamg_spmat mvamg_spmat;
/* A_c = galerkin_product(P, A) of pkg/src/mvamg/sparse.py:50-66, bit for bit:
 * G = P^T (A P) in scipy csr_matmat's summation order (exact zeros dropped),
 * then (G + G^T) * 0.5 as csr_plus_csr + scalar multiply; canonical (sorted)
 * CSR.  A: n x n, P: n x nc, all device pointers (int32 / fp64).  On success
 * *out holds A_c (nc x nc, *nnz_out nonzeros) until mvamg_spmat_destroy;
 * phase_ms (host, 4 floats, may be NULL) receives the device time of
 * P^T, A P, P^T (A P) and the symmetrisation.  Synchronises `stream`. */
int mvamg_galerkin_f64(int n, int nc, const int* a_indptr, const int* a_indices, const double* a_data,
                       const int* p_indptr, const int* p_indices, const double* p_data, mvamg_spmat** out,
                       long long* nnz_out, float* phase_ms, void* stream);
/* Copy a library-owned CSR into caller device buffers (n+1, nnz, nnz). */
int mvamg_spmat_copy(const mvamg_spmat* m, int* indptr, int* indices, double* data, void* stream);
int mvamg_spmat_destroy(mvamg_spmat* m);

/* ---- hierarchy (MultigridOperator) ---------------------------------------- */
typedef struct mvamg_hierarchy mvamg_hierarchy;

/* cycles.py:108-128.  kinds are MVAMG_GS_* / MVAMG_WEIGHTED_JACOBI. */
int mvamg_hierarchy_create(mvamg_hierarchy** h, int nlevels, int cycle_kind, int inner_fcg_iters,
                           int pre_kind, int pre_sweeps, double pre_omega, int post_kind,
                           int post_sweeps, double post_omega);
int mvamg_hierarchy_destroy(mvamg_hierarchy* h);
/* Level k matrix (device CSR) with its diagonal, RN reciprocal diagonal and GS
 * schedule (device chain_ptr / tile_ptr from mvamg_gs_analyse). */
int mvamg_hierarchy_set_level(mvamg_hierarchy* h, int k, int n, int nnz, const int* indptr,
                              const int* indices, const double* data, const double* diag,
                              const double* rdiag, int ntiles, const int* chain_ptr,
                              const int* tile_ptr, const int* chain_order, int gs_threads, int gs_window,
                              int gs_wpos);
/* GS schedule of level k for sweep `mode` (see mvamg_gs_schedule), device. */
int mvamg_hierarchy_set_gs_schedule(mvamg_hierarchy* h, int k, int mode, const unsigned long long* rec,
                                    const int* round_off, const int* tbase, const int* tile_wbase,
                                    const int* perm, double* tperm, int R, int D, int lean_C,
                                    int slot_words, int rec_words_max);
/* Small-level GS schedule of level k for sweep `mode` (see mvamg_gs_levels);
 * when set it takes precedence over the wavefront schedule. */
int mvamg_hierarchy_set_gs_levels(mvamg_hierarchy* h, int k, int mode, int ncta, int rows_per_cta,
                                  int nlev, int max_rows, int max_ents, int threads, int group,
                                  const int* lev_ptr, const int* lev_eptr, const void* rows, const void* ents,
                                  const int* perm, double* tperm);
/* ---- NCCL for the row-partitioned solve --------------
 * One communicator per process / GPU.  libnccl.so.2 is opened at run time (the
 * copy PyTorch already loaded, when it did); every call is stream-ordered on the
 * caller's stream.  Replaces nothing in the reference (it is single-process);
 * used by paper_1907_04417_b200/distributed.py's halo exchanges and the
 * fused PCG dot allreduces. */
typedef struct mvamg_comm mvamg_comm;
/* 128 bytes of ncclUniqueId (rank 0 creates it, the others receive it). */
int mvamg_comm_unique_id(void* id128);
int mvamg_comm_init(mvamg_comm** comm, int rank, int nranks, const void* id128);
int mvamg_comm_destroy(mvamg_comm* comm);
/* One grouped exchange: send_buf[q] (send_count[q] doubles, device) to
 * send_peer[q], recv_buf[q] from recv_peer[q]. */
int mvamg_halo_exchange(mvamg_comm* comm, int nsend, const int* send_peer, const double* const* send_buf,
                        const long long* send_count, int nrecv, const int* recv_peer, double* const* recv_buf,
                        const long long* recv_count, void* stream);
/* In-place sum over the ranks of `count` device doubles (the PCG dots). */
int mvamg_allreduce_sum_f64(mvamg_comm* comm, double* buf, long long count, void* stream);
/* SpMV kernel choice for rows handled one thread per row (1, the default:
 * CSR-stream tiles -- coalesced products into shared memory, then CSR-order
 * row sums; 0: the plain thread-per-row loop).  Both bit-identical. */
int mvamg_set_spmv_stream(int enable);
/* Diagnostics: CTA 0 of every streamed sweep writes (tag, clock64) pairs --
 * tag -2 before a stage's wait, -3 after it, the batch's rows after its
 * barrier -- into trace_dev (cap int64s; [0] = entries used).  NULL: off. */
int mvamg_gs_stream_set_trace(long long* trace_dev, int cap);
/* Stream plan of level k for sweep `mode` (see mvamg_gs_stream_plan); used
 * before every other schedule of that mode.  A mode-2 plan with tfold (n
 * device doubles) also serves backward sweeps from x_old: the old lower
 * neighbours are folded into the right-hand side first (same roundings). */
int mvamg_hierarchy_set_gs_stream(mvamg_hierarchy* h, int k, int mode, int nstages, int nslots, int slot_bytes,
                                  int group, int ncta, const void* blob, const long long* stage_off, double* tfold);
/* Dataflow row schedule of level k for sweep `mode` (see mvamg_gs_rows);
 * used when set and no level-set schedule is set for that mode. */
int mvamg_hierarchy_set_gs_rows(mvamg_hierarchy* h, int k, int mode, const int* rowid, const int* cnt,
                                const int* crit, const double* dg, const double* rdg, const int* perm, const int* wofs,
                                const double* coef, const int* src, int threads, int ctas,
                                int max_tile_slots, double* tperm);
/* Cluster dataflow plan of level k for sweep `mode` (mvamg_gs_cluster_plan);
 * used before every other schedule of that mode; a mode-2 plan also serves
 * backward sweeps from x_old (folded). */
int mvamg_hierarchy_set_gs_cluster(mvamg_hierarchy* h, int k, int mode, const int* wptr, const int* wpage,
                                   const void* blob, const int* perm, int grid, int ncta, int wpc, int slots,
                                   int page_bytes, int sleep_ns, double* tperm);
/* Transfer k: P (n_k x n_{k+1}) and R = P^T (n_{k+1} x n_k), device CSR.
 * Levels k and k+1 must be set first (their sizes give P's and R's shapes):
 * otherwise MVAMG_E_STATE.  Synchronises the device once to read nnz(P), nnz(R). */
int mvamg_hierarchy_set_transfer(mvamg_hierarchy* h, int k, const int* p_indptr,
                                 const int* p_indices, const double* p_data,
                                 const int* r_indptr, const int* r_indices,
                                 const double* r_data);
/* Coarsest level: dense inverse (row-major, device) built from the reference's
 * own LU factors: Inv = lu_solve((lu, piv), I). */
int mvamg_hierarchy_set_coarse(mvamg_hierarchy* h, const double* inv);
/* Workspace: query its size in bytes, then bind caller-owned device memory. */
int mvamg_hierarchy_workspace_bytes(mvamg_hierarchy* h, long long* bytes);
int mvamg_hierarchy_bind_workspace(mvamg_hierarchy* h, void* ws, void* stream);
/* Use CUDA graphs for repeated cycles (default 1). */
int mvamg_hierarchy_set_graphs(mvamg_hierarchy* h, int enable);

/* z = B^{-1} r, one cycle (cycles.py:174-179).  Device vectors of length n_0. */
int mvamg_cycle_apply(mvamg_hierarchy* h, const double* r, double* z, void* stream);
/* e = x - B^{-1} (A_0 x) (cycles.py:181-184). */
int mvamg_error_propagation(mvamg_hierarchy* h, const double* x, double* e, void* stream);
/* Device status word accumulated since the last reset (MVAMG_ST_* bits). */
int mvamg_hierarchy_status(mvamg_hierarchy* h, int* status, int reset);

/* ---- PCG (krylov.py:28-72), x0 = 0 ---------------------------------------
 * precond: the hierarchy's cycle (pc_kind 1), the symmetrized multiplicative
 * composite (pc_kind 2, mvamg_composite_*), or none (pc_kind 0).  The matrix is
 * the finest level of `h`.  hist (device, itmax+1 doubles) receives
 * ||r_k||; on return *nit = iterations, *converged, *status = MVAMG_ST_* bits
 * (nonzero -> the Python layer raises NotSpdError like the reference). */
#define MVAMG_PC_NONE 0
#define MVAMG_PC_CYCLE 1
#define MVAMG_PC_COMPOSITE 2
typedef struct mvamg_composite mvamg_composite;
int mvamg_pcg_solve(mvamg_hierarchy* h, int pc_kind, mvamg_composite* comp, const double* b,
                    double* x, double rtol, int itmax, double* hist, int* nit, int* converged,
                    int* status, void* stream);
/* Same, with HOST b / x / hist (pinned or pageable): H2D of b and D2H of x and
 * the residual history are inside the call (the end-to-end boundary). */
int mvamg_pcg_solve_host(mvamg_hierarchy* h, int pc_kind, mvamg_composite* comp,
                         const double* b_host, double* x_host, double rtol, int itmax,
                         double* hist_host, int* nit, int* converged, int* status,
                         void* stream);

/* ---- composite of cycles (bootstrap.py:75-113) ---------------------------- */
int mvamg_composite_create(mvamg_composite** c, int ncomp, mvamg_hierarchy* const* comps);
int mvamg_composite_destroy(mvamg_composite* c);
/* x <- E_1..E_r E_r..E_1 x, E_i = I - B_i A (bootstrap.py:98-113), in place. */
int mvamg_composite_apply_symmetrized(mvamg_composite* c, double* x, void* stream);
/* z = Bsym r: z=0; for i in 1..r, r..1: z += B_i (r - A z). */
int mvamg_composite_precond(mvamg_composite* c, const double* r, double* z, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MVAMG_B200_H */
