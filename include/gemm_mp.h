/*
 * gemm_mp.h -- C ABI of the B200-native tile-centric mixed-precision GEMM
 *
 *     C <- alpha * A * B + beta * C
 *
 * of arxiv 2508.14848 ("Leveraging Hardware-Aware Computation in Mixed-Precision
 * Matrix Multiply: A Tile-Centric Approach"), Algorithm 1:
 * A (M x K), B (K x N) and C (M x N) are cut into nb x nb tiles (PAPER.md:145,
 * 179); every tile of A, B and C carries its own precision (the #, $, * of
 * PAPER.md:146), chosen here by a tile-norm criterion against a user tolerance
 * (R1-R5); tiles are converted once into packed low-precision storage;
 * each tile-GEMM runs at the lower precision of its two operands and is folded
 * into C at C's tile precision; data moves between GPUs in the STORED precision
 * and is converted at the receiver.  Multi-GPU: 2D block-cyclic
 * over a P x Q grid "as square as possible" with a SUMMA schedule
 * (PAPER.md:145).
 *
 * Conventions (all entry points):
 *   - extern "C", no C++ types; every call returns gmp_status_t and never throws.
 *     On error, gemm_mp_last_error() returns a thread-local message.
 *   - Memory ownership: the CALLER owns all device memory (operands, scratch,
 *     workspace), the CUDA stream and the NCCL communicator.  A plan owns host
 *     metadata only (tile maps, job lists); gemm_mp_destroy frees it.
 *   - Pointers named A, B, C, scratch, ws are DEVICE pointers; pointers named
 *     host_* or the optional maps in gmp_desc_t are HOST pointers.
 *   - Operand layout: binary64, row-major, leading dimension in elements.  On a
 *     P x Q grid each rank passes ITS LOCAL tiles only.  Default: 2D block-cyclic
 *     (PAPER.md:179): rank (p, q) = rank p*Q + q holds the tiles (i, l) of A with
 *     i = p mod P, l = q mod Q at local tile position (i div P, l div Q); B tiles
 *     (l, j) with l = p mod P, j = q mod Q; C tiles (i, j) with i = p mod P,
 *     j = q mod Q.  With desc.row_owner / col_owner (NEXT-3, gemm_mp_balance) tile
 *     row i of A and C lives on process row row_owner[i] and tile column j of B
 *     and C on process column col_owner[j] (K stays block-cyclic: A column l on
 *     process column l mod Q, B row l on process row l mod P); a rank's local
 *     tiles keep increasing global order.  P = Q = 1 is the single-GPU layout.
 *   - Asynchronous calls enqueue work on the given stream; asynchronous CUDA or
 *     NCCL failures surface at the next call or at gemm_mp_sync.
 */
#ifndef GEMM_MP_H
#define GEMM_MP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Precision classes, ordered by unit roundoff; the class
 * of a tile-GEMM is max(code_A, code_B) = the lower of its operands' precisions
 * (north_star; R6). */
typedef enum { GMP_FP64 = 0, GMP_FP32 = 1, GMP_FP16 = 2, GMP_BF16 = 3, GMP_E4M3 = 4, GMP_E5M2 = 5,
               GMP_MXFP4 = 6 /* OCP MXFP4: E2M1 + E8M0 scale per 32 K-elements; A/B only (R31) */
} gmp_class_t;
#define GMP_NCLASS_ABI 7   /* classes; ordered by unit roundoff, so a pair's class is max(code_A, code_B) */

typedef enum {
  GMP_OK = 0,
  GMP_ERR_ARG = 1,           /* null/invalid argument, tol <= 0 or not finite, ld too small */
  GMP_ERR_NOT_DIVISIBLE = 2, /* nb does not divide M, N or K, or nb is not a multiple of 128 */
  GMP_ERR_MAP_SHAPE = 3,     /* explicit map holds a code > 6                                  */
  GMP_ERR_NONFINITE = 4,     /* A, B (or C with beta != 0) holds a NaN or an infinity          */
  GMP_ERR_GRID = 5,          /* P*Q, rank and communicator are inconsistent                    */
  GMP_ERR_WORKSPACE = 6,     /* scratch or workspace smaller than the size query returned      */
  GMP_ERR_STATE = 7,         /* call out of order (execute before convert, ...)                */
  GMP_ERR_CUDA = 8,          /* a CUDA runtime/driver call failed                              */
  GMP_ERR_NCCL = 9,          /* an NCCL call failed                                            */
  GMP_ERR_UNSUPPORTED = 10   /* configuration outside what this build supports                 */
} gmp_status_t;

/* flags */
#define GMP_FLAG_SIMT_ONLY 1u /* run classes 2..4 on the SIMT (binary32 FMA) kernel: cross-check only */
#define GMP_FLAG_TIMING 2u    /* record CUDA events around each class launch of execute (stats.class_ms) */
#define GMP_FLAG_FP64_INT8 8u /* experimental: FP64 class on the INT8 tensor pipe (7 exact int8 digits
                                 per element, 28 tcgen05 kind::i8 MMAs) instead of DMMA (default)    */
#define GMP_FLAG_FP32_FFMA 4u /* FP32 class on the FP32 pipe (packed FFMA2, bitwise O8) instead of the
                                 default tensor-pipe path (exact BF16x3 split, six BF16 MMAs per block) */
#define GMP_FLAG_FP32_X9 1024u /* FP32 class on the tensor pipe with all nine BF16 part products (exact
                                 products, BF16x9) instead of the default six with i + j <= 2 (BF16x6: the
                                 three dropped terms are below 2^-26 of each product; R32)  */
#define GMP_FLAG_SPLIT16 2048u /* one launch per 16-bit class; default: the FP16 pairs of a SUMMA step ride
                                 on the BF16 launch (k_tc_class<3>, per item BF16 then FP16 pairs in the
                                 fold order, one W read/write for both; C bit-identical)             */
#define GMP_FLAG_NCCL_BCAST 4096u /* SUMMA panels through ncclBroadcast on the row / column communicators
                                 (the round-1 transport) instead of the default copy-engine pulls:
                                 each receiver copies the tiles it needs straight from the root's
                                 payload slot over NVLink (workspaces mapped with CUDA IPC, no SMs) */
#define GMP_FLAG_DYN_SCHED 8192u /* tcgen05 class launches take their next item from a device counter
                                 when the TMA producer needs it (CTAs stay on a narrow window of items)
                                 instead of the default static walk (CTA b: items b, b + grid, ...).
                                 Measured at cfg3: 834-841 vs 858-860 TF/s, DRAM bytes unchanged.   */
#define GMP_FLAG_SPLIT_BN128 16384u /* FP32 class (BF16x6) always at BN = 128 (128-byte K blocks); default
                                 BN = 256 with 64-byte K blocks when every W of the launch is binary32
                                 and nb % 256 == 0 (fewer staged bytes per flop)                       */
#define GMP_FLAG_SEPARATE_MAXABS 32768u /* max|W| of every binary32-W C tile in k_c_maxabs (one extra W
                                 read); default: the last 1-SM tcgen05 launch of a tile emits it from
                                 its registers (same value: max is order-free)                        */
#define GMP_FLAG_TC_PAIR 32u /* opt-in: FP16/BF16/E4M3/E5M2 launches whose C tiles fold into binary32 W
                                 and whose nb is a multiple of 256 run on SM pairs (tcgen05 cta_group::2,
                                 256 x 256 sub-tiles, half the B bytes per SM), rastered by C tile row
                                 bands.  Faster alone (all-BF16 32768^3: 1107 vs 1035 TF/s under the
                                 power cap) but slower inside the cfg3 step (702 vs 790 TF/s: the
                                 later FP32-class launches run at a lower clock), DESIGN.md 7.       */
#define GMP_FLAG_TC_SINGLE 512u /* the 1-SM 128 x 256 kernel for those launches (the default; the flag
                                 makes the choice explicit and overrides GMP_FLAG_TC_PAIR)          */
/* 64u, 128u: retired (round 2) -- the B-multicast 2-CTA kernel and the all-tensor-classes
   launch measured slower than the per-class 1-SM kernels; the FP16 / BF16 W
   sharing they aimed at is the default merged 16-bit launch (R33)                          */
#define GMP_FLAG_SENDER_SIDE 16u /* SURVEY 8(f) NEXT-2, hybrid conversion (PAPER.md:148 defers it): a
                                 SUMMA panel tile whose receivers in its process row (A) / column (B)
                                 together need a set of classes S whose payloads are smaller than the
                                 stored one is broadcast as those |S| payloads, converted at the SENDER
                                 from its stored payload (RN_c(decode(stored)), the same bytes a
                                 receiver would make); otherwise the stored payload is sent.  Maps,
                                 packed bytes and C are bit-identical to the default receiver-side
                                 mode; only the bytes on NVLink (stats.recv_bytes_local) change.     */
#define GMP_FLAG_LOOPBACK 256u /* TEST ONLY: the P*Q > 1 exchanges run through an in-process loopback
                                 transport (gemm_mp_loopback_create) instead of NCCL, so that one process
                                 can drive all P*Q rank plans of a grid on ONE GPU, one host thread per
                                 rank (the calls of different ranks meet at host barriers inside plan
                                 and convert, so they must run concurrently).  The statistics all-reduce
                                 becomes a rank-order sum of the G contributions (exact: one owner per
                                 entry) and each SUMMA broadcast one
                                 device-to-device copy per receiving rank from the root plan's payload
                                 slot.  Everything else -- maps, slots, receiver-side shadows and
                                 splits, step events, fold order -- is the NCCL path's code.         */

typedef struct {
  int64_t M, N, K;     /* global GEMM shape                                                    */
  int32_t nb;          /* tile edge; multiple of 128 dividing M, N, K (PAPER.md:179 uses 1024/2048) */
  double tol;          /* accuracy tolerance: ||C - C_fp64||_F <= tol (|a| ||A|| ||B|| + |b| ||C||) */
  double alpha, beta;  /* GEMM scalars; beta == 0 means C is not read (BLAS convention)          */
  uint32_t class_mask; /* bit c enables class c (gmp_class_t); FP64 always on; E4M3/E5M2/MXFP4 opt-in;
                          bits above 6 are ignored                                           */
  uint32_t flags;      /* GMP_FLAG_*                                                           */
  int32_t P, Q, rank;  /* process grid and this rank (= p*Q + q); 1, 1, 0 on one GPU            */
  /* optional explicit per-tile codes (host, row-major global tile grids: mt x kt, kt x nt,
   * mt x nt) -- the paper's own "aD:bS" experiment mode.  NULL = criterion. */
  const uint8_t *a_map, *b_map, *c_map;
  /* optional tile ownership (host arrays, NEXT-3): row_owner[i] in [0, P) for each of
   * the M/nb tile rows, col_owner[j] in [0, Q) for each of the N/nb tile columns;
   * NULL = block-cyclic (i mod P, j mod Q).  Every rank must pass the same arrays
   * (gemm_mp_balance computes them identically on every rank).  Read during
   * gemm_mp_plan / gemm_mp_plan_host only.  GMP_ERR_GRID for an entry out of range. */
  const int32_t *row_owner, *col_owner;
} gmp_desc_t;

typedef struct gmp_plan_s *gmp_plan_t;

/* Run statistics (gemm_mp_get_stats). Counts are global (identical on every rank)
 * except the *_local fields. */
typedef struct {
  int64_t tiles_a[7], tiles_b[7], tiles_c[7]; /* tiles per stored class                  */
  int64_t pairs[7];                           /* tile-GEMMs per pair class (global)      */
  double flops[7];                            /* 2 nb^3 x pairs[c]                       */
  int64_t pairs_local[7];                     /* tile-GEMMs this rank computes            */
  int64_t shadows_local[7];                   /* shadow tiles this rank materialises      */
  int64_t packed_bytes_local;                 /* packed A/B payload bytes stored locally  */
  int64_t recv_bytes_local;                   /* SUMMA panel bytes this rank receives     */
  int64_t workspace_bytes;
  int32_t steps;                              /* SUMMA steps (K tiles / step depth)        */
  int32_t launches_execute;                   /* kernels one gemm_mp_execute launches      */
  int32_t launches_plan, launches_convert;    /* kernels of gemm_mp_plan / gemm_mp_convert */
  double class_ms[7];                         /* GMP_FLAG_TIMING: device ms of the class-c tile-GEMM
                                                 launches of the last execute (waits for them) */
  int32_t class_launches[7];                  /* launches per class in one execute             */
  double exec_other_ms[3];                    /* GMP_FLAG_TIMING: device ms of the last execute outside
                                                 the class launches: before the first (W0, uploads),
                                                 between them (SUMMA waits, gaps), after the last
                                                 (C-finalize)                                     */
  double convert_ms[4];                       /* GMP_FLAG_TIMING: device ms of the last convert: table
                                                 uploads + barriers, pack, shadows (incl. MXFP4 and the
                                                 step-0 pull issue), FP32 splits / FP64 digit planes */
} gmp_stats_t;

/* Device scratch needed by gemm_mp_plan (tile statistics + maps; KB-sized).     */
gmp_status_t gemm_mp_scratch_size(const gmp_desc_t *desc, size_t *bytes);

/* S1 + S2 of SURVEY 8(a): per-tile canonical sums of squares and maxabs of the
 * local tiles (map-stats kernel), an all-reduce of the statistics over the grid
 * (NCCL, P*Q > 1), the precision map / scale kernel, then ONE host
 * synchronisation to read the maps back and size the packed arena.
 * A, B (and C if beta != 0) must stay unchanged until gemm_mp_convert has
 * completed on the stream.  nccl_comm: ncclComm_t of all P*Q ranks, NULL iff
 * P*Q == 1.  Collective over the grid.  On success *out is a new plan.        */
gmp_status_t gemm_mp_plan(const gmp_desc_t *desc, const double *A, int64_t lda, const double *B,
                          int64_t ldb, const double *C, int64_t ldc, void *scratch,
                          size_t scratch_bytes, void *nccl_comm, void *stream, gmp_plan_t *out);

/* Device workspace for convert + execute: job tables, packed arenas (stored,
 * shadows, SUMMA receive slots), W accumulators, packed C_in / C_out.          */
gmp_status_t gemm_mp_workspace_size(gmp_plan_t plan, size_t *bytes);

/* S3 + S5 (local tiles): convert-and-pack every local tile of A, B (and C_in)
 * into its class with one RNE rounding and its power-of-two scale (PAPER.md:148,
 * DESIGN.md O3/O6), then the receiver-side shadows needed by local tile-GEMMs
 * (and, under GMP_FLAG_SENDER_SIDE, the shadows this rank sends).  Host tables
 * reach the device through pinned staging read by a kernel, never through a
 * copy engine.  ws must be 1024-byte aligned.  On a P*Q > 1 grid (default
 * copy-engine transport) the workspaces are mapped into the peers with CUDA IPC
 * when they change: every rank must switch to a new workspace at the same
 * convert (one all-gather of the handles).  Async on `stream`.  After
 * completion A and B may be freed.  ws stays owned by the caller and must
 * outlive every execute of this plan.                                          */
gmp_status_t gemm_mp_convert(gmp_plan_t plan, void *ws, size_t ws_bytes, void *stream);

/* S4 - S7: per SUMMA step, NCCL broadcasts of the step's A/B panels in stored
 * precision (P*Q > 1; or their needed shadow classes under GMP_FLAG_SENDER_SIDE)
 * + shadows of received tiles on a comm stream, then one
 * grouped tile-GEMM launch per precision class present, folding into the W
 * accumulators; finally C-finalize writes the packed C and the binary64 user C
 * (local layout, ldc).  Collective over the grid.  Async on `stream`; may be
 * called repeatedly after one convert (a repeated execute reuses the received
 * panels: no SUMMA traffic).  The C tile descriptors are uploaded only when ldc
 * or the workspace changed, so on one GPU a repeated execute with the same
 * arguments issues kernels only and may be captured into a CUDA graph.
 * C: 16-byte aligned, ldc even (GMP_ERR_ARG otherwise; C-finalize writes 16-byte vectors). */
gmp_status_t gemm_mp_execute(gmp_plan_t plan, double *C, int64_t ldc, void *stream);

/* S7 of SURVEY 8(a) (C-finalize, north_star "accumulating into C at C's tile precision"),
 * with the C lifetime of SURVEY 8(b) ("C is written at execute") narrowed to the finalize:
 * gemm_mp_execute whose C-finalize (the only step that writes C) first waits for the CUDA
 * event c_free_event (a cudaEvent_t; NULL = gemm_mp_execute): a caller streaming results
 * out of C (e.g. a device->host copy of the previous GEMM's C on another stream) overlaps
 * that copy with this execute's tile-GEMMs instead of serialising the whole execute behind
 * it.  The event is waited on at the finalize launch; it must have been recorded (or never
 * recorded) when this call is made.                                                       */
gmp_status_t gemm_mp_execute_after(gmp_plan_t plan, double *C, int64_t ldc, void *stream, void *c_free_event);

/* Waits for the plan's streams; returns the first asynchronous error.          */
gmp_status_t gemm_mp_sync(gmp_plan_t plan);

/* Global precision maps (host arrays, row-major tile grids) and STORED scales.
 * Any pointer may be NULL.  C scales are the finalize scales of the last
 * execute for local tiles (0 elsewhere).                                       */
gmp_status_t gemm_mp_get_maps(gmp_plan_t plan, uint8_t *a, uint8_t *b, uint8_t *c, int16_t *a_scale,
                              int16_t *b_scale, int16_t *c_scale);

/* Copies one LOCAL tile's payload to host memory: which = 'A' or 'B' (class
 * `cls` = the stored code or a materialised shadow class (0..5); cls = 6: the
 * three K-major BF16 parts of the FP32 class's tensor-pipe split; cls = 7: the
 * seven int8 digit planes of the FP64 class's INT8 path), 'C' (packed C_out of
 * the last execute, cls = code), 'I' (packed C_in), 'W' (accumulator, binary64
 * or binary32).  (ti, tj) are GLOBAL tile indices.  *bytes in: capacity, out:
 * bytes written; *scale receives the tile's power-of-two scale.  Synchronous. */
gmp_status_t gemm_mp_get_tile(gmp_plan_t plan, char which, int64_t ti, int64_t tj, int32_t cls,
                              void *host_dst, size_t *bytes, int16_t *scale);

gmp_status_t gemm_mp_get_stats(gmp_plan_t plan, gmp_stats_t *out);

/* Debug export of S1 (O4): the GLOBAL per-tile statistics
 * the map kernel used, as read back at gemm_mp_plan's one synchronisation --
 * S = the canonical CNORM sum of squares, maxabs, finite flag (1 = no NaN/Inf) --
 * for which = 'A' (mt x kt), 'B' (kt x nt) or 'C' (mt x nt; zeros when beta == 0),
 * row-major tile grids.  On P*Q > 1 these are the all-reduced statistics
 * (identical on every rank).  Host arrays, any may be NULL.  GMP_ERR_STATE on a
 * gemm_mp_plan_host plan (no statistics were computed).                         */
gmp_status_t gemm_mp_get_tile_stats(gmp_plan_t plan, char which, double *S, double *maxabs,
                                    uint8_t *finite);

/* Host-only plan from given maps (no device work): the same tile lists, arena
 * layout, work lists and SUMMA schedule as gemm_mp_plan builds after its map
 * kernels.  acode/bcode/ccode: global code grids; ascale5/bscale5: [tile][7]
 * class-c scales; cin_scale may be NULL.  For inspecting the schedule and the
 * multi-rank bookkeeping without a GPU: it holds no operands, statistics or
 * communicators, so gemm_mp_convert / gemm_mp_execute / gemm_mp_get_tile_stats
 * on it fail with GMP_ERR_STATE.                                               */
gmp_status_t gemm_mp_plan_host(const gmp_desc_t *desc, const uint8_t *acode, const uint8_t *bcode,
                               const uint8_t *ccode, const int16_t *ascale5, const int16_t *bscale5,
                               const int16_t *cin_scale, gmp_plan_t *out);

/* SUMMA broadcasts of step `step` on this rank, 5 int64 per entry:
 * {which (0 = A on the row communicator, 1 = B on the column communicator),
 *  global tile index, class of the payload on the wire (the stored class, or a
 *  shadow class under GMP_FLAG_SENDER_SIDE), root rank inside that
 *  communicator, payload bytes}.  entries may be NULL to query the count *n;
 *  cap counts entries (5 int64 each).                                          */
gmp_status_t gemm_mp_get_schedule(gmp_plan_t plan, int32_t step, int64_t *entries, int64_t cap,
                                  int64_t *n);

/* NCCL bootstrap helpers (the unique id travels over torch.distributed).
 * The first plan on a world communicator splits it into the SUMMA row and
 * column communicators (cached); environment variables GMP_NCCL_MAX_CTAS and
 * GMP_NCCL_CTA_POLICY, when set, go into their ncclConfig_t (maxCTAs,
 * CTAPolicy).  Default: NCCL's own (profiles/nccl_cta_r01.md).                 */
gmp_status_t gemm_mp_nccl_unique_id(void *out128);
gmp_status_t gemm_mp_nccl_comm_create(const void *id128, int nranks, int rank, void **comm);
gmp_status_t gemm_mp_nccl_comm_destroy(void *comm);
/* TEST ONLY (GMP_FLAG_LOOPBACK): an in-process transport for nranks (2..16) plans on one
 * GPU.  Pass it as gemm_mp_plan's nccl_comm with GMP_FLAG_LOOPBACK set in desc.flags.
 * The caller destroys it after every plan on it is destroyed.  GMP_ERR_ARG for a bad
 * nranks, GMP_ERR_CUDA if its events cannot be created. */
gmp_status_t gemm_mp_loopback_create(int nranks, void **comm);
gmp_status_t gemm_mp_loopback_destroy(void *comm);

/* N1 synthetic generator (benchmark inputs): fills
 * the local block-cyclic part of a rows x cols global matrix.  mode 0 uniform,
 * 1 graded, 2 random.  Async.                                                  */
gmp_status_t gemm_mp_synth(double *out, int64_t ld, int64_t rows, int64_t cols, int32_t nb,
                           int32_t P, int32_t Q, int32_t p, int32_t q, uint64_t seed,
                           uint64_t tau, int32_t mode, int32_t E, int32_t s, void *stream);

/* The same generator for any ownership: local tile (il, jl) of `out` (nrt x nct
 * tiles, row-major, ld >= nct*nb) is global tile (row_tiles[il], col_tiles[jl]).
 * row_tiles / col_tiles are HOST arrays (copied before return).  GMP_ERR_ARG for a
 * tile index out of range.  Async.                                             */
gmp_status_t gemm_mp_synth_tiles(double *out, int64_t ld, int64_t rows, int64_t cols, int32_t nb,
                                 const int32_t *row_tiles, int64_t nrt, const int32_t *col_tiles,
                                 int64_t nct, uint64_t seed, uint64_t tau, int32_t mode, int32_t E,
                                 int32_t s, void *stream);

/* NEXT-3, precision-aware load balancing (PaRSEC's dynamic scheduling
 * absorbs "the imbalanced workload introduced by the adaptive tile-centric
 * mixed-precision algorithm").  Host-only.  From the GLOBAL maps acode (mt x kt)
 * and bcode (kt x nt) -- e.g. gemm_mp_get_maps of a first, block-cyclic plan --
 * chooses tile-row owners row_owner[mt] in [0, P) and tile-column owners
 * col_owner[nt] in [0, Q) (desc->P, desc->Q) that minimise the largest per-rank
 * cost = sum over the rank's C tiles (i, j) of sum_l cost[max(codeA(i,l),
 * codeB(l,j))] + cost[7] x (A + B + C tiles it owns), by alternating row / column
 * local search (moves and swaps) from the block-cyclic start (R30).
 * cost: 8 doubles (relative per-pair time of classes 0..6, per-owned-tile time) or
 * NULL for the built-in B200 model (per pair 2 nb^3 / library peak of the class; the
 * FP32 entry follows the FP32-class kernel desc->flags select: BF16x6 by default,
 * GMP_FLAG_FP32_X9, GMP_FLAG_FP32_FFMA).  Deterministic: every rank gets the same
 * owners from the same maps.  imbalance (may be NULL): {max/mean rank cost of the
 * block-cyclic layout, of the returned layout} -- never worse than block-cyclic.
 * Pass the owners as desc.row_owner / col_owner to gemm_mp_plan; the caller
 * places its local tiles accordingly (gemm_mp_synth_tiles for synthetic inputs).
 * C is bitwise the same for every ownership (the fold order is fixed, R15).     */
gmp_status_t gemm_mp_balance(const gmp_desc_t *desc, const uint8_t *acode, const uint8_t *bcode,
                             const double *cost, int32_t *row_owner, int32_t *col_owner,
                             double *imbalance);

/* Frees the plan's host metadata (NULL-safe).                                  */
void gemm_mp_destroy(gmp_plan_t plan);

/* Thread-local message of the last failing call on this thread.               */
const char *gemm_mp_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* GEMM_MP_H */
