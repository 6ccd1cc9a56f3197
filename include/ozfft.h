/*
 * ozfft.h -- C ABI of the B200 (sm_100a) fp64-accurate FFT built from 32-bit NTTs.
 *
 * Method: arXiv 2603.29129 (Kawakami & Takahashi).  References "P:N" are lines of
 * /root/reference/PAPER.md; "S:N" lines of SPEC.md; "SURVEY" = SURVEY.md.
 *
 *   y = DFT(x), x in F64^n + i F64^n, any n >= 1 (Alg.4 Require/Ensure, P:464-465;
 *   eq:dft P:152-156, omega_n = e^{-2 pi i / n}).
 *   Bluestein (Alg.1) with cyclic length m = 2^ceil(log2(2n-1)),
 *   Ozaki split of Re/Im of x' = x (.) omega into <= K int32 slices (Alg.6, P:768-793;
 *   cap K), exact slice convolutions by 32-bit NTTs modulo p0 and p1
 *   (P:670-716), NTT-domain accumulation of <= L equal-scale products before each
 *   inverse NTT (Alg.8), two-prime Garner CRT, scaled DD
 *   recombination and post-chirp (Alg.4).
 *
 * Conventions (all entry points):
 *   - Every call returns an ozfft_status; nothing throws across the ABI.  On error
 *     ozfft_last_error_string() (thread-local) describes it.
 *   - Device pointers are CUDA device addresses on the plan's device; `stream` is a
 *     cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Complex data are contiguous [batch][n] interleaved (re, im) binary64 -- the
 *     memory of a contiguous torch.complex128 tensor; 16-byte aligned.
 *   - The caller owns every buffer: input/output, the plan's persistent buffer and
 *     its workspace.  execute never allocates, never synchronizes the host, and
 *     never falls back to the CPU.
 *   - A plan is immutable after bind; one execute at a time per bound workspace.
 *   - Plan options (descriptor): conv_mode (padded m >= 2n-1 / the paper's cyclic m = n),
 *     accum_mode (the paper's four real convolutions / complex images), precision
 *     (double-double / the paper's triple-single) -- see the OZFFT_CONV_*, OZFFT_ACCUM_*
 *     and OZFFT_PREC_* blocks below; the defaults are the north star's path.
 */
#ifndef OZFFT_H
#define OZFFT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  OZFFT_OK = 0,
  OZFFT_ERR_INVALID_ARGUMENT = 1,   /* null pointer, n < 1, batch < 1, K/L out of range */
  OZFFT_ERR_UNSUPPORTED_LENGTH = 2, /* m > 2^min(two-adicity(p0), two-adicity(p1)) */
  OZFFT_ERR_BAD_PRIMES = 3,         /* not prime, equal, >= 2^31, or p0*p1 >= 2^62        */
  OZFFT_ERR_ALPHA = 4,              /* alpha < 1: no slice width fits            */
  OZFFT_ERR_NOT_BOUND = 5,          /* execute before bind                              */
  OZFFT_ERR_MISALIGNED = 6,         /* buffer not 16-byte (256-byte for plan buffers) aligned */
  OZFFT_ERR_CUDA = 7,               /* a CUDA runtime error (message in last_error)      */
  OZFFT_ERR_SHARD = 8,              /* bad shard index / count                          */
  OZFFT_ERR_BUFFER_TOO_SMALL = 9    /* persistent or workspace size below plan_get_info  */
} ozfft_status;

/* Test-only environment knob (read at ozfft_plan_create): OZFFT_FAULT_INJECT=1 flips one
 * bit of one NTT-domain group value after the row pass of every execute (transform 0,
 * prime 0, conv rr, the last Alg.8 group) -- the GPU parity tests must then fail
 * (tests/test_gpu_fault.py).  Never set it otherwise. */

/* Plan descriptor.  Defaults (zeros) mean: K = 3, L = 3, p0 = 2,130,706,433,
 * p1 = 2,113,929,217 (the paper's primes), device = current device,
 * max_workspace_bytes = 16 GiB (the batch is processed in chunks that fit). */
typedef struct {
  int64_t n;                  /* DFT length, >= 1                                  */
  int64_t batch;              /* independent transforms per execute, >= 1          */
  int32_t K;                  /* split cap per real vector, 1..8       */
  int32_t L;                  /* NTT-domain accumulation bound, 1..8   */
  uint32_t p0, p1;            /* NTT primes, < 2^31, p-1 divisible by m            */
  int32_t device;             /* CUDA device ordinal, -1 = current                 */
  int32_t conv_mode;          /* OZFFT_CONV_PADDED (0) or OZFFT_CONV_CYCLIC (1), below */
  int32_t accum_mode;         /* OZFFT_ACCUM_REAL (0) or OZFFT_ACCUM_IMAGE (1), below  */
  int32_t precision;          /* OZFFT_PREC_DD (0) or OZFFT_PREC_TS (1), below          */
  uint64_t max_workspace_bytes;
} ozfft_plan_desc;

/* Bluestein convolution length (desc.conv_mode).
 *  OZFFT_CONV_PADDED: m = 2^ceil(log2(2n-1)) >= 2n-1, x' zero-padded and omega* padded with
 *    index reversal (ZeroPad / ZeroPad_pm, Alg.4) -- any n; the north star's path.
 *  OZFFT_CONV_CYCLIC: m = n for a power-of-two n (the Bluestein convolution is
 *    then already cyclic -- omega*(j) = omega_2n^{-j^2} has period n for even n -- so "the FFT
 *    length N can be kept equal to n").  Same alpha, digits and schedule as the padded plan;
 *    the CRT integers and the fp64 output are bitwise identical to it, at half the NTT
 *    length.  OZFFT_ERR_UNSUPPORTED_LENGTH if n is not a power of two. */
#define OZFFT_CONV_PADDED 0
#define OZFFT_CONV_CYCLIC 1

/* How the complex convolution is assembled from exact modular convolutions
 * (desc.accum_mode).
 *  OZFFT_ACCUM_REAL: the paper's method -- Re x' and Im x' (and Re, Im of omega~*) are
 *    split separately and the complex convolution is four real ones, rr - ii and ir + ri
 *    (P:1010-1021), each with its own Alg.8 schedule: 12 forward + 40 inverse NTTs per
 *    transform at (K, L) = (3, 3).
 *  OZFFT_ACCUM_IMAGE: complex-image accumulation (beyond the paper).
 *    Both parts of each split level share one exponent (Alg.6 with mu = max over both
 *    parts), and the complex digit vectors are convolved through the two ring maps
 *    a + i b -> a +- iota b mod p (iota^2 = -1; both paper primes are 1 mod 4): two image
 *    convolutions per Alg.8 group instead of four real ones, re = (z+ + z-)/2 and
 *    im = (z+ - z-)/(2 iota) per prime, then Garner.  alpha uses the bound
 *    2 L n 4^alpha < P/2.  12 forward + 20 inverse NTTs at (3, 3).  Results differ from
 *    OZFFT_ACCUM_REAL (different digits); the oracle's image mode is the reference.
 *    Not available with ozfft_shard_partial (OZFFT_ERR_SHARD). */
#define OZFFT_ACCUM_REAL 0
#define OZFFT_ACCUM_IMAGE 1

/* Working precision of the O(n) steps a1 (premultiply), a2 (split) and a7 (recombination,
 * post-chirp) (desc.precision).
 *  OZFFT_PREC_DD: binary64 double-double (DESIGN ruling 1; the default).
 *  OZFFT_PREC_TS: the paper's triple-single arithmetic (Alg.4 TS form, TS split
 *    P:784-798): x, omega, omega~* converted to TS, x' = x (.) omega with
 *    TSMul / TSAdd, the split on the TS words with rho = 24 - alpha, z / c accumulated with
 *    TSAdd, post-chirp in TS, fl64 at the end.  TSAdd / TSMul are this build's reading
 *    (the paper gives none; DESIGN ruling 24).  Inputs must stay inside the fp32 exponent
 *    range (|x| <= ~2^100 and well above 2^-100); only with OZFFT_ACCUM_REAL. */
#define OZFFT_PREC_DD 0
#define OZFFT_PREC_TS 1

typedef struct {
  int64_t n, m, batch, chunk;   /* m: Bluestein cyclic length; chunk: transforms per pass */
  int32_t K, L, alpha, rho;     /* alpha = floor((log2(p0p1/2) - log2(L n))/2), rho = 53-alpha */
  int32_t log2_rows, log2_cols; /* NTT decomposition m = R x C (two passes when R > 1) */
  uint64_t persistent_bytes;    /* caller allocates; 256-byte aligned              */
  uint64_t workspace_bytes;     /* caller allocates; 256-byte aligned              */
  int32_t cached_ntts;          /* forward NTTs of omega~* slices done at bind */
  int32_t conv_mode;            /* as in the descriptor                                */
  int32_t accum_mode;           /* as in the descriptor                                */
  int32_t precision;            /* as in the descriptor                                */
} ozfft_plan_info;

typedef struct {
  int32_t k[4];          /* slices of Re x', Im x' (transform 0), Re w~*, Im w~*      */
  int64_t fwd_ntts;      /* runtime forward NTTs over the last execute (all transforms) */
  int64_t inv_ntts;      /* runtime inverse NTTs (= 2 x groups)                      */
  int64_t cached_ntts;   /* plan-time forward NTTs of omega~* slices                 */
  int64_t groups;        /* Alg.8 flush groups over the batch                        */
  int64_t nonfinite;     /* transforms whose input had NaN/Inf (output set to NaN)   */
  uint32_t flags;        /* bit0: some input non-finite; bits 1-31: reserved, 0 */
  int32_t reserved;
} ozfft_exec_stats;

/* Test-only stage outputs (device pointers, any may be NULL), for ONE execute of a
 * plan whose batch fits in a single chunk.  Layouts match the oracle's taps, in the
 * natural (paper) order -- internal orders are converted by tap kernels:
 *   digits int32 [B][2][K][n]     E int32 [B][2][K]    kv int32 [B][2]
 *   X   uint32 [B][2 part][K][2 prime][m]     forward NTTs of the slices
 *   sched int32 [B][4 conv][1 + K*K*(2+2L)]   Alg.8 groups: ngroups, then per group
 *                                             cexp, npairs, (s,t) x L
 *   Z   uint32 [B][4][K*K][2][m]  NTT-domain accumulated groups (Alg.8 l.981-982)
 *   res uint32 [B][4][K*K][2][n]  inverse-NTT outputs j < n (l.973)
 *   crt int64  [B][4][K*K][n]     Garner integers (l.974)
 *   W   uint32 [2 part][K][2 prime][m]        cached omega~* spectra (plan data)
 * conv order: rr, ii, ir, ri as (x part, w part) = (0,0),(1,1),(1,0),(0,1).      */
typedef struct {
  void* digits;
  void* E;
  void* kv;
  void* X;
  void* sched;
  void* Z;
  void* res;
  void* crt;
  void* W;
} ozfft_taps;

typedef struct ozfft_plan ozfft_plan;

/* Host-side plan math only (alpha, roots of unity, twiddle tables, the correctly
 * rounded chirp table (ruling 3) and omega~* = ZeroPad_pm(omega*, m)
 * ).  No device memory is touched.  Errors: INVALID_ARGUMENT,
 * UNSUPPORTED_LENGTH, BAD_PRIMES, ALPHA.  On success *out owns a host plan. */
ozfft_status ozfft_plan_create(const ozfft_plan_desc* desc, ozfft_plan** out);

/* Sizes and derived parameters; valid right after create. */
ozfft_status ozfft_plan_get_info(const ozfft_plan* plan, ozfft_plan_info* info);

/* Bind caller-owned device memory (persistent >= info.persistent_bytes, workspace >=
 * info.workspace_bytes, both 256-byte aligned) and precompute on `stream`: uploads
 * tables, splits omega~* (Alg.6) and runs its 4K forward NTTs into the
 * cached W spectra, using the workspace as scratch (no device allocation).
 * Synchronizes `stream` (plan time, not on the hot path).  Re-binding is allowed; it
 * drops the execute graphs captured against the previous buffers.
 * Errors: INVALID_ARGUMENT, MISALIGNED, BUFFER_TOO_SMALL, CUDA. */
ozfft_status ozfft_plan_bind(ozfft_plan* plan, void* persistent, size_t persistent_bytes,
                             void* workspace, size_t workspace_bytes, void* stream);

/* y = DFT(x) (direction -1) or x = DFT^-1(y) (direction +1, P:158-160,
 * computed as conj(DFT(conj(y)))/n with RN division, ruling 16), for the plan's
 * batch.  `in` and `out` are device complex128 [batch][n]; in == out is allowed.
 * The calling thread's current device must be the plan's (desc.device), as for every
 * call that takes a stream; `stream` belongs to that device.
 * Asynchronous on `stream`.  Plans with batch * m <= 2^25 (env OZFFT_GRAPH_MAX_WORK) and
 * one workspace chunk capture the launch sequence as a CUDA graph on the second execute
 * with the same (in, out, direction) and replay it from then on (up to 8 cached per plan;
 * a re-bind drops them); not while the stage profiler is on.
 * Errors: NOT_BOUND, INVALID_ARGUMENT, MISALIGNED, CUDA. */
ozfft_status ozfft_execute(const ozfft_plan* plan, const void* in, void* out, int direction,
                           void* stream);

/* Same as ozfft_execute but `in`/`out` are HOST buffers (pinned for overlap): the batch
 * runs as sub-batches (small first and last ones) in disjoint staging + workspace slots;
 * host->device copies, the device pipeline (alternating between two internal compute
 * streams) and device->host copies of neighbouring sub-batches overlap.  Ordered after
 * the work already queued on `stream`; returns after the last D2H copy has completed
 * (synchronizes `stream`).  Uses the workspace's staging area.  Env OZFFT_HOST_SUBS
 * ("1,3,4,...", summing to the batch) overrides the sub-batch sizes (tuning only).
 * Errors: NOT_BOUND, INVALID_ARGUMENT, CUDA. */
ozfft_status ozfft_execute_host(const ozfft_plan* plan, const double* in, double* out,
                                int direction, void* stream);

/* The sub-batch sizes ozfft_execute_host uses for this plan (host-side planning, no device
 * work, callable before bind): writes min(count, cap) sizes to `sizes` (may be NULL) and
 * returns the count (-1 for a NULL plan).  Every size is <= plan_get_info's chunk (one
 * workspace slot) and they sum to the batch. */
int64_t ozfft_host_subbatches(const ozfft_plan* plan, int64_t* sizes, int64_t cap);

/* As ozfft_execute, additionally writing the stage outputs listed in ozfft_taps.
 * Requires info.chunk == info.batch.  Test-only; not on the hot path. */
ozfft_status ozfft_execute_taps(const ozfft_plan* plan, const void* in, void* out,
                                int direction, void* stream, const ozfft_taps* taps);

/* Statistics of the last execute on this plan (synchronizes `stream`). */
ozfft_status ozfft_last_stats(const ozfft_plan* plan, ozfft_exec_stats* stats, void* stream);

/* ---- single large transform sharded over `nshards` ranks ----------
 * Unit u in [0, 8) = (prime q = u % 2, real conv cv = u / 2) (conv order as in taps).
 * Rank `shard` computes the contiguous units [shard*8/nshards, (shard+1)*8/nshards)
 * (with 8 ranks: rank r = (prime r % 2, conv r / 2)) of transform 0: it redoes the O(n)
 * premultiply/split of `in` (identical digits, exponents and Alg.8 schedules on every
 * rank), then -- with nshards > 1 -- reads the four group counts ng_cv (one 16-byte D2H
 * copy; synchronizes `stream`) and returns g = max_cv ng_cv in *groups (nshards == 1:
 * g = K*K, no synchronization).  It runs its forward NTTs, NTT-domain accumulation and
 * inverse NTTs and writes the residues of its units straight into their place of
 * `residues`, a device uint32 buffer laid out [8 units][g groups][n]: bytes
 * [shard * 8/nshards * g * n * 4, (shard + 1) * 8/nshards * g * n * 4).  An in-place
 * all-gather of those equal slices (torch.distributed / NCCL all_gather_into_tensor)
 * completes the buffer on every rank -- 8 g n 4 bytes, 160 n at (K, L) = (3, 3) -- and
 * ozfft_shard_finish(g) performs Garner's CRT, the recombination and the post-chirp.
 * `residues` must hold ozfft_shard_residue_bytes(plan, 0) bytes (the K*K-group capacity);
 * ozfft_shard_residue_bytes(plan, g) is the exchanged size.  nshards must divide 8.
 * Errors: SHARD, NOT_BOUND, INVALID_ARGUMENT, CUDA. */
uint64_t ozfft_shard_residue_bytes(const ozfft_plan* plan, int32_t groups);
ozfft_status ozfft_shard_partial(const ozfft_plan* plan, int shard, int nshards, const void* in,
                                 int direction, void* residues, int32_t* groups, void* stream);
ozfft_status ozfft_shard_finish(const ozfft_plan* plan, const void* residues_all, int32_t groups,
                                void* out, int direction, void* stream);

/* ---- the same exchange fused into the producing kernel (peer memory) ---------------
 * BASELINE.json north_star (single transform: primes / slice pairs sharded, the residues
 * gathered before CRT) with the gather done by the kernel that computes the residues: the
 * inverse-NTT epilogue (k_col_inv; one-pass plans: the row kernel) stores every residue of
 * this rank's units into the exchange buffer of EVERY rank, over NVLink peer memory, so
 * the transfer overlaps the NTT tile by tile and no collective runs afterwards.
 * `residues_by_rank[r]` (r < nshards) is rank r's exchange buffer ([8][g][n] uint32, the
 * capacity of ozfft_shard_residue_bytes(plan, 0)) as a device pointer valid in this
 * process: its own buffer for r == shard, a CUDA IPC mapping (ozfft_ipc_open_handle) or a
 * peer-accessible allocation for the others.  Same split, schedule read and *groups as
 * ozfft_shard_partial.  Completion: a rank may call ozfft_shard_finish on its own buffer
 * once every rank's ozfft_shard_partial_p2p has completed on its stream (the caller's
 * barrier, e.g. stream synchronize + a process-group barrier, or a device-side
 * collective enqueued after it).  nshards <= 8 and must divide 8.
 * Errors: SHARD, NOT_BOUND, INVALID_ARGUMENT, CUDA. */
ozfft_status ozfft_shard_partial_p2p(const ozfft_plan* plan, int shard, int nshards, const void* in,
                                     int direction, void* const* residues_by_rank, int32_t* groups,
                                     void* stream);
/* CUDA IPC for those buffers: the 64-byte handle of the device allocation that contains
 * `dev_ptr` (cudaIpcGetMemHandle) and the byte offset of `dev_ptr` inside it (a caching
 * allocator's tensor need not start its allocation); the mapping of another process's
 * (handle, offset) in this process -- *dev_ptr = mapped base + offset (cudaIpcOpenMemHandle,
 * lazy peer access) -- and its release (the pointer and offset ozfft_ipc_open_handle gave).
 * Errors: INVALID_ARGUMENT, CUDA. */
ozfft_status ozfft_ipc_get_handle(const void* dev_ptr, void* handle64, uint64_t* offset);
ozfft_status ozfft_ipc_open_handle(const void* handle64, uint64_t offset, void** dev_ptr);
ozfft_status ozfft_ipc_close(void* dev_ptr, uint64_t offset);

/* ---- profiling (tracing) -----------------------------------------------------------
 * Per-stage CUDA-event timers.  While enabled, every execute records an event pair
 * around each stage kernel on the execute stream (no host synchronization).
 * ozfft_profile_read synchronizes `stream`, returns the summed milliseconds and the
 * launch count of each stage since enable (or the previous read) and clears them.
 * Stage ids: */
#define OZFFT_STAGE_SPLIT_MAX 0    /* k_split_max: premultiply + per-level max (a1, a2) */
#define OZFFT_STAGE_SPLIT_DIGITS 1 /* k_split_digits: digits + Alg.8 schedule (a2)     */
#define OZFFT_STAGE_COL_FWD 2      /* k_col_fwd: forward NTT column pass (a3)          */
#define OZFFT_STAGE_ROW_FUSED 3    /* k_row_fused: fwd rows + accumulate + inv rows (a3-a5) */
#define OZFFT_STAGE_COL_INV 4      /* k_col_inv: inverse NTT column pass (a5)          */
#define OZFFT_STAGE_CRT_FINISH 5   /* k_crt_finish: CRT + recombine + post-chirp (a6, a7) */
#define OZFFT_NSTAGES 6
ozfft_status ozfft_profile_enable(ozfft_plan* plan, int on);
ozfft_status ozfft_profile_read(ozfft_plan* plan, double* ms, int64_t* launches, void* stream);

/* Process-wide number of kernels this library has launched (all plans, all calls). */
uint64_t ozfft_kernel_launches(void);

/* Free the host plan (device buffers stay owned by the caller). */
ozfft_status ozfft_plan_destroy(ozfft_plan* plan);

const char* ozfft_status_string(ozfft_status s);
const char* ozfft_last_error_string(void);

/* Library build identity, e.g. "ozfft sm_100a <git-describe>". */
const char* ozfft_version(void);

#ifdef __cplusplus
}
#endif
#endif /* OZFFT_H */
