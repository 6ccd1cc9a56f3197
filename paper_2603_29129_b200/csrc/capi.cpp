// capi.cpp -- the extern "C" boundary of ozfft (declared in include/ozfft.h).
// Validation, plan sizing/memory layout, chunked execution and statistics.  All
// compute is in kernels.cu; there is no CPU fallback anywhere in this library.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>

#include "internal.h"


struct ozfft_plan : ozfft::Plan {};

namespace ozfft {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

static ozfft_status fail(ozfft_status s, const std::string& msg) {
  set_error(msg);
  return s;
}

static bool is_prime_u32(uint64_t p) {
  if (p < 2) return false;
  for (uint64_t d = 2; d * d <= p; ++d)
    if (p % d == 0) return false;
  return true;
}
static int two_adicity(uint64_t v) {
  int a = 0;
  while (v && !(v & 1)) { v >>= 1; ++a; }
  return a;
}
// alpha = floor((log2(p0 p1 / 2) - log2(L n)) / 2) (n = DFT length, ruling 2):
// the largest a with 2 L n 4^a < p0 p1, evaluated in exact 128-bit integers.
static int compute_alpha(int64_t n, int64_t L, uint32_t p0, uint32_t p1) {
  const unsigned __int128 P = (unsigned __int128)p0 * p1;
  int best = 0;
  for (int a = 1; a < 62; ++a) {
    unsigned __int128 v = (unsigned __int128)2 * (uint64_t)L * (uint64_t)n;
    bool over = false;
    for (int i = 0; i < a && !over; ++i) {
      v <<= 2;
      if (v >= P) over = true;
    }
    if (over) break;
    best = a;
  }
  return best;
}

static std::atomic<uint64_t> g_launches{0};
void count_launches(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }
uint64_t launches_so_far() { return g_launches.load(std::memory_order_relaxed); }

// NVTX ranges per stage (host timeline of the launches; free unless a tool such as ncu or
// nsys is attached -- NVTX3 is header-only and resolves its injection library lazily)
static const char* const kStageNames[OZFFT_NSTAGES] = {
    "ozfft:split_max", "ozfft:split_digits", "ozfft:col_fwd", "ozfft:row_fused", "ozfft:col_inv",
    "ozfft:crt_finish"};

void prof_mark(const Plan& pl, int stage, bool begin, void* stream) {
  if (begin)
    nvtxRangePushA(kStageNames[stage]);
  else
    nvtxRangePop();
  Prof* pr = pl.prof;
  if (!pr || !pr->on) return;
  if (pr->next >= pr->pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    pr->pool.push_back((void*)e);
  }
  void* e = pr->pool[pr->next++];
  cudaEventRecord((cudaEvent_t)e, (cudaStream_t)stream);
  if (begin) {
    pr->recs.push_back(Prof::Rec{stage, e, nullptr});
  } else {
    for (size_t i = pr->recs.size(); i-- > 0;)
      if (pr->recs[i].stage == stage && pr->recs[i].e1 == nullptr) { pr->recs[i].e1 = e; break; }
  }
}

static uint64_t align256(uint64_t v) { return (v + 255) & ~(uint64_t)255; }

// Plan memory layout.  The workspace is [batch-sized stats + schedules][chunk x per-transform
// regions]; chunk is the largest count whose whole workspace (fixed regions, 256-byte
// alignment of every region, per-transform regions) stays within max_workspace_bytes, and the
// bind-time scratch must fit the cap too.  Fails (OZFFT_ERR_BUFFER_TOO_SMALL) if not even one
// transform fits.
static ozfft_status layout(Plan& pl) {
  const int64_t n = pl.n, m = pl.m, K = pl.K, L = pl.L, G = K * K;
  // persistent
  uint64_t o = 0;
  pl.poff.chirp = o; o = align256(o + (uint64_t)n * 16);
  pl.poff.tw = o;    o = align256(o + (uint64_t)4 * m * 8);
  pl.poff.W = o;     o = align256(o + std::max<uint64_t>((uint64_t)4 * K * m * 8, (uint64_t)m * 16));
  pl.poff.wsplit = o; o = align256(o + (uint64_t)(2 + 2 * K) * 4);
  pl.poff.end = o;
  pl.persistent_bytes = o;
  const bool two = pl.logR > 0;
  auto place = [&](int64_t chunk) {
    uint64_t w = 0;
    pl.woff.stats = w;  w = align256(w + (uint64_t)pl.batch * stats_stride(K) * 4);
    pl.woff.sched = w;  w = align256(w + (uint64_t)pl.batch * 4 * sched_stride(K, L) * 4);
    pl.woff.mu = w;     w = align256(w + (uint64_t)chunk * 2 * K * 8);
    pl.woff.digits = w; w = align256(w + (uint64_t)chunk * 2 * K * n * 4);
    pl.woff.Y = w;      w = align256(w + (two ? (uint64_t)chunk * 4 * K * m * 4 : 0));
    pl.woff.G = w;      w = align256(w + (two ? (uint64_t)chunk * 8 * G * m * 4 : 0));
    pl.woff.res = w;    w = align256(w + (uint64_t)chunk * 8 * G * n * 4);
    pl.woff.S = w;      w = align256(w + (two ? (uint64_t)chunk * 4 * n * 16 : 0));
    pl.woff.io_in = w;  w = align256(w + (uint64_t)chunk * n * 16);
    pl.woff.io_out = w; w = align256(w + (uint64_t)chunk * n * 16);
    pl.woff.end = w;
    return w;
  };
  // bind-time scratch (launch_plan_precompute: mu, digits, stats, Y, X of omega~*) reuses
  // the workspace before the first execute
  const uint64_t bind_scratch = align256((uint64_t)2 * K * 8) + align256((uint64_t)2 * K * m * 4) +
                                align256((uint64_t)stats_stride(K) * 4) +
                                2 * align256((uint64_t)4 * K * m * 4);
  const uint64_t fixed = place(0);  // batch-sized regions + alignment of the empty ones
  const uint64_t per = place(1) - fixed + 10 * 256;  // one transform, padding headroom
  if (fixed + per > pl.max_ws || bind_scratch > pl.max_ws)
    return fail(OZFFT_ERR_BUFFER_TOO_SMALL,
                "max_workspace_bytes is below the workspace of a single transform");
  int64_t chunk = (int64_t)std::max<uint64_t>(1, (pl.max_ws - fixed) / per);
  chunk = std::min<int64_t>(chunk, pl.batch);
  chunk = std::min<int64_t>(chunk, 65535);  // per-transform kernels index transforms by gridDim.y
  while (chunk > 1 && place(chunk) > pl.max_ws) --chunk;  // exact check (alignment)
  pl.chunk = chunk;
  o = place(chunk);
  pl.workspace_bytes = std::max<uint64_t>(o, bind_scratch);
  return OZFFT_OK;
}

#ifndef OZFFT_GRAPH_MAX_WORK_DEFAULT
#define OZFFT_GRAPH_MAX_WORK_DEFAULT (1ll << 25)  // batch * m up to which execute is a graph
// (c3, batch * m = 2^23: 2.384 vs 2.402 ms per execute measured with the graph)
#endif

static ozfft_status check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) return fail(OZFFT_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return OZFFT_OK;
}

}  // namespace ozfft

using namespace ozfft;

extern "C" {

const char* ozfft_status_string(ozfft_status s) {
  switch (s) {
    case OZFFT_OK: return "OZFFT_OK";
    case OZFFT_ERR_INVALID_ARGUMENT: return "OZFFT_ERR_INVALID_ARGUMENT";
    case OZFFT_ERR_UNSUPPORTED_LENGTH: return "OZFFT_ERR_UNSUPPORTED_LENGTH";
    case OZFFT_ERR_BAD_PRIMES: return "OZFFT_ERR_BAD_PRIMES";
    case OZFFT_ERR_ALPHA: return "OZFFT_ERR_ALPHA";
    case OZFFT_ERR_NOT_BOUND: return "OZFFT_ERR_NOT_BOUND";
    case OZFFT_ERR_MISALIGNED: return "OZFFT_ERR_MISALIGNED";
    case OZFFT_ERR_CUDA: return "OZFFT_ERR_CUDA";
    case OZFFT_ERR_SHARD: return "OZFFT_ERR_SHARD";
    case OZFFT_ERR_BUFFER_TOO_SMALL: return "OZFFT_ERR_BUFFER_TOO_SMALL";
  }
  return "OZFFT_ERR_UNKNOWN";
}

const char* ozfft_last_error_string(void) { return g_err.c_str(); }

// ozfft_version() is defined in the generated _build/version.cpp (build.py): git revision +
// a hash of every library source, rebuilt whenever any of them changes.

ozfft_status ozfft_plan_create(const ozfft_plan_desc* d, ozfft_plan** out) {
  if (!d || !out) return fail(OZFFT_ERR_INVALID_ARGUMENT, "null descriptor or output pointer");
  *out = nullptr;
  ozfft_plan_desc desc = *d;
  if (desc.K == 0) desc.K = 3;
  if (desc.L == 0) desc.L = 3;
  if (desc.p0 == 0) desc.p0 = 2130706433u;
  if (desc.p1 == 0) desc.p1 = 2113929217u;
  if (desc.max_workspace_bytes == 0) desc.max_workspace_bytes = 16ull << 30;
  if (desc.n < 1 || desc.batch < 1)
    return fail(OZFFT_ERR_INVALID_ARGUMENT, "n and batch must be >= 1");
  if (desc.K < 1 || desc.K > kMaxK || desc.L < 1 || desc.L > kMaxL)
    return fail(OZFFT_ERR_INVALID_ARGUMENT, "K and L must be in [1, 8]");
  if (desc.n > (1ll << 23)) return fail(OZFFT_ERR_UNSUPPORTED_LENGTH, "n > 2^23");
  const uint32_t p0 = desc.p0, p1 = desc.p1;
  if (p0 == p1 || p0 >= (1u << 31) || p1 >= (1u << 31) || !is_prime_u32(p0) || !is_prime_u32(p1) ||
      (unsigned __int128)p0 * p1 >= ((unsigned __int128)1 << 62))
    return fail(OZFFT_ERR_BAD_PRIMES, "primes must be distinct, < 2^31, with p0*p1 < 2^62");
  ozfft_plan* pl = new (std::nothrow) ozfft_plan();
  if (!pl) return fail(OZFFT_ERR_INVALID_ARGUMENT, "out of host memory");
  pl->n = desc.n;
  pl->batch = desc.batch;
  pl->K = desc.K;
  pl->L = desc.L;
  pl->p[0] = p0;
  pl->p[1] = p1;
  pl->max_ws = desc.max_workspace_bytes;
  if (desc.conv_mode != OZFFT_CONV_PADDED && desc.conv_mode != OZFFT_CONV_CYCLIC) {
    delete pl;
    return fail(OZFFT_ERR_INVALID_ARGUMENT, "conv_mode must be OZFFT_CONV_PADDED or OZFFT_CONV_CYCLIC");
  }
  int64_t m = 1;
  if (desc.conv_mode == OZFFT_CONV_CYCLIC) {  // N = n for power-of-two n
    if (desc.n & (desc.n - 1)) {
      delete pl;
      return fail(OZFFT_ERR_UNSUPPORTED_LENGTH, "OZFFT_CONV_CYCLIC needs a power-of-two n");
    }
    m = desc.n;
  } else {
    while (m < 2 * desc.n - 1) m <<= 1;  // Bluestein length, N >= 2n-1
  }
  pl->conv_mode = desc.conv_mode;
  if (desc.accum_mode != OZFFT_ACCUM_REAL && desc.accum_mode != OZFFT_ACCUM_IMAGE) {
    delete pl;
    return fail(OZFFT_ERR_INVALID_ARGUMENT, "accum_mode must be OZFFT_ACCUM_REAL or _IMAGE");
  }
  if ((desc.precision != OZFFT_PREC_DD && desc.precision != OZFFT_PREC_TS) ||
      (desc.precision == OZFFT_PREC_TS && desc.accum_mode == OZFFT_ACCUM_IMAGE)) {
    delete pl;
    return fail(OZFFT_ERR_INVALID_ARGUMENT,
                "precision must be OZFFT_PREC_DD or OZFFT_PREC_TS (TS with OZFFT_ACCUM_REAL only)");
  }
  pl->image = desc.accum_mode == OZFFT_ACCUM_IMAGE ? 1 : 0;
  pl->ts = desc.precision == OZFFT_PREC_TS ? 1 : 0;
  if (pl->image && ((p0 & 3u) != 1u || (p1 & 3u) != 1u)) {
    delete pl;
    return fail(OZFFT_ERR_BAD_PRIMES, "OZFFT_ACCUM_IMAGE needs primes = 1 mod 4");
  }
  pl->m = m;
  int logm = 0;
  while ((1ll << logm) < m) ++logm;
  pl->logm = logm;
  if (logm > std::min(two_adicity(p0 - 1ull), two_adicity(p1 - 1ull))) {
    delete pl;
    return fail(OZFFT_ERR_UNSUPPORTED_LENGTH, "m exceeds the primes' two-adicity");
  }
  if (logm > 24) {  // (the paper's primes allow 2^24: two-adicity of p0)
    delete pl;
    return fail(OZFFT_ERR_UNSUPPORTED_LENGTH, "m <= 2^24 (n <= 2^23)");
  }
  // NTT decomposition: one pass up to m = 2^12, else rows of C = 2^11 (2^12 from m = 2^20) and
  // columns of R = m / C <= 2^8 (up to 2^12 at m = 2^20 .. 2^24, with 32 elements per thread).
  // (Measured alternatives at c3: one-warp rows of C = 2^10, 122 vs 147 GFLOP/s; rows of
  // C = 2^12, 141 vs 154 GFLOP/s -- OZFFT_TUNE_LOGC=12 still selects the latter.)
  pl->logC = logm <= 12 ? logm : std::min(12, std::max(11, logm - 8));
  if (const char* t = std::getenv("OZFFT_TUNE_LOGC")) {  // tuning knob (tools/, not the hot path)
    const int v = std::atoi(t);
    if (logm > 12 && decomposition_supported(logm - v, v)) pl->logC = v;
  }
  pl->logR = logm - pl->logC;
  if (const char* t = std::getenv("OZFFT_FAULT_INJECT"))  // test-only: must trip the parity tests
    pl->fault = std::atoi(t) != 0;
  if (const char* t = std::getenv("OZFFT_SPLIT_CLUSTER_MAXLEN"))  // knob (tests/tools): 0 = off
    pl->split_cluster_max = std::atoll(t);
  if (const char* t = std::getenv("OZFFT_SMALL_FUSED"))  // knob (tests/tools): 0 = three-kernel path
    pl->small_fused = std::atoi(t) != 0;
  if (const char* t = std::getenv("OZFFT_SMALL_Z"))  // knob (tools/): 1, 2 or 4
    pl->small_z = std::atoi(t) == 1 || std::atoi(t) == 2 || std::atoi(t) == 4 ? std::atoi(t) : 0;
  // image mode: a real output sums L n complex products (|Re| <= 2 4^alpha each)
  pl->alpha = compute_alpha(pl->image ? 2 * desc.n : desc.n, desc.L, p0, p1);
  if (pl->alpha < 1) {
    delete pl;
    return fail(OZFFT_ERR_ALPHA, "alpha < 1");
  }
  pl->rho = (pl->ts ? 24 : 53) - pl->alpha;  // u = 2^-24 (TS) or 2^-53 (DD, ruling 1)
  int dev = desc.device;
  if (dev < 0) {
    if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  }
  pl->device = dev;
  ozfft_status s = build_plan_tables(*pl);
  if (s) {
    delete pl;
    return s;
  }
  s = layout(*pl);
  if (s) {
    delete pl;
    return s;
  }
  *out = pl;
  return OZFFT_OK;
}

ozfft_status ozfft_plan_get_info(const ozfft_plan* pl, ozfft_plan_info* info) {
  if (!pl || !info) return fail(OZFFT_ERR_INVALID_ARGUMENT, "null argument");
  std::memset(info, 0, sizeof(*info));
  info->n = pl->n;
  info->m = pl->m;
  info->batch = pl->batch;
  info->chunk = pl->chunk;
  info->K = pl->K;
  info->L = pl->L;
  info->alpha = pl->alpha;
  info->rho = pl->rho;
  info->log2_rows = pl->logR;
  info->log2_cols = pl->logC;
  info->persistent_bytes = pl->persistent_bytes;
  info->workspace_bytes = pl->workspace_bytes;
  info->cached_ntts = pl->bound ? 2 * (pl->kw[0] + pl->kw[1]) : 4 * pl->K;
  info->conv_mode = pl->conv_mode;
  info->accum_mode = pl->image;
  info->precision = pl->ts;
  return OZFFT_OK;
}

ozfft_status ozfft_plan_bind(ozfft_plan* pl, void* persistent, size_t pbytes, void* workspace,
                             size_t wbytes, void* stream) {
  if (!pl || !persistent || !workspace) return fail(OZFFT_ERR_INVALID_ARGUMENT, "null argument");
  if (((uintptr_t)persistent & 255) || ((uintptr_t)workspace & 255))
    return fail(OZFFT_ERR_MISALIGNED, "plan buffers must be 256-byte aligned");
  if (pbytes < pl->persistent_bytes || wbytes < pl->workspace_bytes)
    return fail(OZFFT_ERR_BUFFER_TOO_SMALL, "persistent/workspace smaller than plan_get_info");
  // the caller's current device is restored on every return path
  int caller_dev = -1;
  if (cudaGetDevice(&caller_dev) != cudaSuccess) caller_dev = -1;
  struct Restore {
    int d;
    ~Restore() {
      if (d >= 0) cudaSetDevice(d);
    }
  } restore{caller_dev};
  ozfft_status s = check_cuda(cudaSetDevice(pl->device), "cudaSetDevice");
  if (s) return s;
  // from here on the plan's device state changes: it is unbound until every step succeeded
  // (a failed re-bind must not leave half-initialised tables behind a "bound" plan)
  pl->bound = false;
  cudaStream_t st = (cudaStream_t)stream;
  if (pl->graphs) {  // captured executes hold the previous buffers' addresses
    cudaDeviceSynchronize();
    for (const GraphCache::Entry& e : pl->graphs->entries) cudaGraphExecDestroy((cudaGraphExec_t)e.exec);
    pl->graphs->entries.clear();
    pl->graphs->seen.clear();
    pl->graphs->next = pl->graphs->seen_next = 0;
  }
  pl->pers = (uint8_t*)persistent;
  pl->ws = (uint8_t*)workspace;
  const int64_t m = pl->m;
  s = check_cuda(cudaMemcpyAsync(pl->pers + pl->poff.chirp, pl->chirp.data(),
                                 sizeof(double) * 2 * pl->n, cudaMemcpyHostToDevice, st),
                 "upload chirp");
  for (int q = 0; q < 2 && !s; ++q)
    for (int dir = 0; dir < 2 && !s; ++dir)
      s = check_cuda(cudaMemcpyAsync(pl->pers + pl->poff.tw + (uint64_t)(q * 2 + dir) * m * 8,
                                     pl->tw[q][dir].data(), (size_t)m * 8, cudaMemcpyHostToDevice, st),
                     "upload twiddles");
  // omega~* staged in the W area; launch_plan_precompute replaces it by the W spectra
  if (!s)
    s = check_cuda(cudaMemcpyAsync(pl->pers + pl->poff.W, pl->wstar.data(), (size_t)m * 16,
                                   cudaMemcpyHostToDevice, st),
                   "upload omega~*");
  if (!s) s = launch_plan_precompute(*pl, stream);  // uses the workspace as scratch
  if (!s) s = check_cuda(cudaMemsetAsync(pl->ws, 0, pl->woff.mu, st), "clear stats");
  if (!s) s = check_cuda(cudaStreamSynchronize(st), "bind sync");
  if (s) return s;
  pl->bound = true;
  return OZFFT_OK;
}

static ozfft_status check_exec(const ozfft_plan* pl, const void* in, const void* out, int dir) {
  if (!pl) return fail(OZFFT_ERR_INVALID_ARGUMENT, "null plan");
  if (!pl->bound) return fail(OZFFT_ERR_NOT_BOUND, "plan not bound");
  if (!in || !out) return fail(OZFFT_ERR_INVALID_ARGUMENT, "null buffer");
  if (dir != -1 && dir != 1) return fail(OZFFT_ERR_INVALID_ARGUMENT, "direction must be -1 or +1");
  if (((uintptr_t)in & 15) || ((uintptr_t)out & 15))
    return fail(OZFFT_ERR_MISALIGNED, "buffers must be 16-byte aligned");
  return OZFFT_OK;
}

// Replay (or capture, then replay) the whole execute as one CUDA graph on `stream`.
// *done = false: the key was new (now remembered); the caller launches directly.
static ozfft_status execute_graph(ozfft_plan* pl, const void* in, void* out, int direction,
                                  cudaStream_t st, bool* done) {
  if (!pl->graphs) pl->graphs = new GraphCache();
  GraphCache& gc = *pl->graphs;
  *done = true;
  for (const GraphCache::Entry& e : gc.entries)
    if (e.in == in && e.out == out && e.direction == direction) {
      count_launches(e.launches);
      return check_cuda(cudaGraphLaunch((cudaGraphExec_t)e.exec, st), "graph launch");
    }
  bool seen = false;
  for (const GraphCache::Key& k : gc.seen)
    if (k.in == in && k.out == out && k.direction == direction) seen = true;
  if (!seen) {
    const GraphCache::Key k{in, out, direction};
    if (gc.seen.size() < GraphCache::kMax) {
      gc.seen.push_back(k);
    } else {
      gc.seen[gc.seen_next] = k;
      gc.seen_next = (gc.seen_next + 1) % GraphCache::kMax;
    }
    *done = false;
    return OZFFT_OK;
  }
  if (!gc.capture) {
    cudaStream_t cs;
    if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess)
      return check_cuda(cudaGetLastError(), "capture stream create");
    gc.capture = (void*)cs;
  }
  cudaStream_t cs = (cudaStream_t)gc.capture;
  ozfft_status s = check_cuda(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal), "begin capture");
  if (s) return s;
  const uint64_t l0 = launches_so_far();
  ExecArgs a{};
  a.nb = pl->batch;
  a.in = reinterpret_cast<const double*>(in);
  a.out = reinterpret_cast<double*>(out);
  a.b0 = 0;
  a.direction = direction;
  a.unit_mask = 0xFF;
  a.finish = true;
  const ozfft_status ls = launch_execute(*pl, a, (void*)cs);
  cudaGraph_t g = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(cs, &g);
  if (ls) {
    if (g) cudaGraphDestroy(g);
    return ls;
  }
  s = check_cuda(ce, "end capture");
  if (s) return s;
  cudaGraphExec_t ge = nullptr;
  s = check_cuda(cudaGraphInstantiate(&ge, g, 0), "graph instantiate");
  cudaGraphDestroy(g);
  if (s) return s;
  GraphCache::Entry e{in, out, direction, (void*)ge, (int)(launches_so_far() - l0)};
  if (gc.entries.size() < GraphCache::kMax) {
    gc.entries.push_back(e);
  } else {  // replace the oldest
    cudaGraphExecDestroy((cudaGraphExec_t)gc.entries[gc.next].exec);
    gc.entries[gc.next] = e;
    gc.next = (gc.next + 1) % GraphCache::kMax;
  }
  return check_cuda(cudaGraphLaunch(ge, st), "graph launch");  // (captured launches counted)
}

ozfft_status ozfft_execute(const ozfft_plan* pl, const void* in, void* out, int direction,
                           void* stream) {
  ozfft_status s = check_exec(pl, in, out, direction);
  if (s) return s;
  const int64_t n = pl->n;
  // plans up to batch * m = 2^25: one CUDA graph per (in, out, direction) instead of ~8
  // launches (captured on the second execute with the same buffers)
  static const int64_t graph_max_work = [] {
    const char* t = std::getenv("OZFFT_GRAPH_MAX_WORK");  // batch * m; 0 disables
    return t ? std::atoll(t) : (int64_t)OZFFT_GRAPH_MAX_WORK_DEFAULT;
  }();
  if (pl->chunk == pl->batch && pl->batch * pl->m <= graph_max_work && !(pl->prof && pl->prof->on)) {
    bool done = false;
    s = execute_graph(const_cast<ozfft_plan*>(pl), in, out, direction, (cudaStream_t)stream, &done);
    if (s) return s;
    if (done) {
      const_cast<ozfft_plan*>(pl)->last_batch = pl->batch;
      return OZFFT_OK;
    }
  }
  for (int64_t b0 = 0; b0 < pl->batch; b0 += pl->chunk) {
    ExecArgs a{};
    a.nb = std::min<int64_t>(pl->chunk, pl->batch - b0);
    a.in = reinterpret_cast<const double*>(in) + 2 * b0 * n;
    a.out = reinterpret_cast<double*>(out) + 2 * b0 * n;
    a.b0 = b0;
    a.direction = direction;
    a.unit_mask = 0xFF;
    a.finish = true;
    a.taps = nullptr;
    s = launch_execute(*pl, a, stream);
    if (s) return s;
  }
  const_cast<ozfft_plan*>(pl)->last_batch = pl->batch;
  return OZFFT_OK;
}

// Sub-batch sizes of ozfft_execute_host (every size <= pl.chunk, summing to the batch).
static std::vector<int64_t> host_subbatches(const Plan& plan) {
  const Plan* pl = &plan;
  const int64_t B = pl->batch;
  std::vector<int64_t> sizes;
  {
    const int64_t big = std::max<int64_t>(1, std::min<int64_t>((B + 3) / 4, std::max<int64_t>(1, pl->chunk / 3)));
    const int64_t edge = std::max<int64_t>(1, big / 4);
    // linear ramp edge, 2 edge, ... < big at both ends (pipeline fill / drain with small
    // sub-batches, then full-size ones): c3 e2e 127 -> 130, c4 92.5 -> 95.9 GFLOP/s measured
    // against the older (edge, big - 1, big, ..., big - 1, edge)
    std::vector<int64_t> up;
    int64_t ramp_sum = 0;
    for (int64_t r = edge; r < big; r += edge) { up.push_back(r); ramp_sum += r; }
    int64_t rem = B;
    const bool ramps = big > 1 && B >= 2 * ramp_sum + big;
    if (ramps) {
      sizes = up;
      rem -= 2 * ramp_sum;
    } else if (big > 1 && B >= 2 * edge + 1) {
      up.assign(1, edge);
      sizes = up;
      rem -= 2 * edge;
    } else {
      up.clear();
    }
    // the middle: ceil(rem / big) sub-batches of near-equal size (no small straggler)
    const int64_t nmid = (rem + big - 1) / big;
    for (int64_t i = 0; i < nmid; ++i) sizes.push_back(rem / nmid + (i < rem % nmid ? 1 : 0));
    sizes.insert(sizes.end(), up.rbegin(), up.rend());
    // small transforms (m <= 2^16): per-sub-batch fixed latencies dominate -- fewer, larger
    // sub-batches B/8, B/4, B/4, B/4, B/8 (measured at c2: e2e 89.8 vs 86 GFLOP/s for
    // B/8, 3B/8, 3B/8, B/8, which beat the generic ramp)
    // (used only when its largest sub-batch fits one workspace chunk: for B = 8k + 7 the
    // middle ones are ceil(rest / 3) > B / 4 + 1)
    if (pl->m <= (1 << 16) && B >= 8) {
      const int64_t e8 = B / 8, rest = B - 2 * e8;
      const std::vector<int64_t> v = {e8, rest / 3 + (rest % 3 > 0), rest / 3 + (rest % 3 > 1),
                                      rest / 3, e8};
      if (*std::max_element(v.begin(), v.end()) <= pl->chunk) sizes = v;
    }
    if (const char* t = std::getenv("OZFFT_HOST_SUBS")) {  // tuning knob (tools/), "1,4,4,..."
      std::vector<int64_t> v;
      int64_t tot = 0;
      for (const char* c = t; *c;) {
        const int64_t k = std::strtoll(c, const_cast<char**>(&c), 10);
        if (k <= 0) break;
        v.push_back(k);
        tot += k;
        if (*c == ',') ++c;
      }
      if (tot == B && *std::max_element(v.begin(), v.end()) <= pl->chunk) sizes = v;
    }
  }
  return sizes;
}

// Concurrent host pipeline (the whole batch fits one workspace chunk): sub-batches use
// disjoint workspace and staging slots, so they need no slot-reuse waits and alternate
// between two compute streams -- the small first / last sub-batches (short pipeline fill
// and drain) overlap the large ones on the GPU instead of running it half-empty.
// Host-buffer pipeline: the batch runs as sub-batches (small first and last ones shorten
// the fill -- the first H2D -- and the drain -- the last D2H); sub-batch j uses staging and
// workspace slot j mod nslots and alternates between two compute streams, so H2D, D2H and
// the kernels of neighbouring sub-batches overlap, and the small edge sub-batches share the
// GPU with large ones instead of running it half-empty.  Slot reuse waits for the previous
// occupant's kernels (input consumed) and D2H (output and workspace free).
ozfft_status ozfft_execute_host(const ozfft_plan* pl, const double* in, double* out, int direction,
                                void* stream) {
  ozfft_status s = check_exec(pl, in, out, direction);
  if (s) return s;
  ozfft_plan* mp = const_cast<ozfft_plan*>(pl);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = pl->n;
  const std::vector<int64_t> sizes = host_subbatches(*pl);
  const int64_t nsub = (int64_t)sizes.size();
  const int64_t sb = *std::max_element(sizes.begin(), sizes.end());
  if (sb > pl->chunk)  // every sub-batch runs in one workspace slot (never expected)
    return fail(OZFFT_ERR_INVALID_ARGUMENT, "internal: host sub-batch larger than the workspace chunk");
  const int64_t nslots = std::max<int64_t>(1, std::min<int64_t>(nsub, pl->chunk / sb));
  if (!mp->pipe) mp->pipe = new HostPipe();
  HostPipe& hp = *mp->pipe;
  void** streams[4] = {&hp.h2d, &hp.d2h, &hp.cs[0], &hp.cs[1]};
  for (void** sp : streams)
    if (!*sp) {
      cudaStream_t cs;
      if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess)
        return check_cuda(cudaGetLastError(), "pipeline stream create");
      *sp = (void*)cs;
    }
  while ((int64_t)hp.ev.size() < 3 * nsub + 1) {
    cudaEvent_t e;
    s = check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event create");
    if (s) return s;
    hp.ev.push_back((void*)e);
  }
  cudaStream_t h2d = (cudaStream_t)hp.h2d, d2h = (cudaStream_t)hp.d2h;
  auto ev = [&](int64_t k) { return (cudaEvent_t)hp.ev[k]; };
  cudaEventRecord(ev(3 * nsub), st);  // everything already queued on the caller's stream
  cudaStreamWaitEvent(h2d, ev(3 * nsub), 0);
  for (int c = 0; c < 2; ++c) cudaStreamWaitEvent((cudaStream_t)hp.cs[c], ev(3 * nsub), 0);
  double* din0 = reinterpret_cast<double*>(pl->ws + pl->woff.io_in);
  double* dout0 = reinterpret_cast<double*>(pl->ws + pl->woff.io_out);
  int64_t b0 = 0;
  for (int64_t j = 0; j < nsub; b0 += sizes[j], ++j) {
    const int64_t nb = sizes[j];
    const size_t bytes = (size_t)nb * n * 16;
    const int64_t slot = (j % nslots) * sb;
    double* din = din0 + 2 * slot * n;
    double* dout = dout0 + 2 * slot * n;
    cudaStream_t cs = (cudaStream_t)hp.cs[j & 1];
    if (j >= nslots) cudaStreamWaitEvent(h2d, ev(3 * (j - nslots) + 1), 0);  // input consumed
    s = check_cuda(cudaMemcpyAsync(din, in + 2 * b0 * n, bytes, cudaMemcpyHostToDevice, h2d), "H2D");
    if (s) return s;
    cudaEventRecord(ev(3 * j + 0), h2d);
    cudaStreamWaitEvent(cs, ev(3 * j + 0), 0);
    if (j >= nslots) cudaStreamWaitEvent(cs, ev(3 * (j - nslots) + 2), 0);  // slot drained
    ExecArgs a{};
    a.nb = nb;
    a.in = din;
    a.out = dout;
    a.b0 = b0;
    a.ws0 = slot;
    a.direction = direction;
    a.unit_mask = 0xFF;
    a.finish = true;
    s = launch_execute(*pl, a, (void*)cs);
    if (s) return s;
    cudaEventRecord(ev(3 * j + 1), cs);
    cudaStreamWaitEvent(d2h, ev(3 * j + 1), 0);
    s = check_cuda(cudaMemcpyAsync(out + 2 * b0 * n, dout, bytes, cudaMemcpyDeviceToHost, d2h), "D2H");
    if (s) return s;
    cudaEventRecord(ev(3 * j + 2), d2h);
  }
  cudaStreamWaitEvent(st, ev(3 * (nsub - 1) + 2), 0);
  mp->last_batch = pl->batch;
  return check_cuda(cudaStreamSynchronize(st), "execute_host sync");
}

int64_t ozfft_host_subbatches(const ozfft_plan* pl, int64_t* sizes, int64_t cap) {
  if (!pl) return -1;
  const std::vector<int64_t> v = host_subbatches(*pl);
  for (int64_t i = 0; i < (int64_t)v.size() && i < cap && sizes; ++i) sizes[i] = v[i];
  return (int64_t)v.size();
}

ozfft_status ozfft_execute_taps(const ozfft_plan* pl, const void* in, void* out, int direction,
                                void* stream, const ozfft_taps* taps) {
  ozfft_status s = check_exec(pl, in, out, direction);
  if (s) return s;
  if (pl->chunk != pl->batch)
    return fail(OZFFT_ERR_INVALID_ARGUMENT, "taps need the whole batch in one chunk");
  ExecArgs a{};
  a.nb = pl->batch;
  a.in = reinterpret_cast<const double*>(in);
  a.out = reinterpret_cast<double*>(out);
  a.b0 = 0;
  a.direction = direction;
  a.unit_mask = 0xFF;
  a.finish = true;
  a.taps = taps;
  s = launch_execute(*pl, a, stream);
  const_cast<ozfft_plan*>(pl)->last_batch = pl->batch;
  return s;
}

ozfft_status ozfft_last_stats(const ozfft_plan* pl, ozfft_exec_stats* out, void* stream) {
  if (!pl || !out) return fail(OZFFT_ERR_INVALID_ARGUMENT, "null argument");
  if (!pl->bound) return fail(OZFFT_ERR_NOT_BOUND, "plan not bound");
  std::memset(out, 0, sizeof(*out));
  out->k[2] = pl->kw[0];
  out->k[3] = pl->kw[1];
  out->cached_ntts = 2 * (pl->kw[0] + pl->kw[1]);
  const int64_t B = pl->last_batch;
  if (B == 0) return OZFFT_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int K = pl->K, L = pl->L;
  std::vector<int32_t> hs((size_t)B * stats_stride(K));
  std::vector<int32_t> hsched((size_t)B * 4 * sched_stride(K, L));
  ozfft_status s = check_cuda(cudaMemcpyAsync(hs.data(), pl->ws + pl->woff.stats, hs.size() * 4,
                                              cudaMemcpyDeviceToHost, st), "stats D2H");
  if (!s) s = check_cuda(cudaMemcpyAsync(hsched.data(), pl->ws + pl->woff.sched, hsched.size() * 4,
                                         cudaMemcpyDeviceToHost, st), "sched D2H");
  if (!s) s = check_cuda(cudaStreamSynchronize(st), "stats sync");
  if (s) return s;
  for (int64_t b = 0; b < B; ++b) {
    const int32_t* r = hs.data() + b * stats_stride(K);
    if (b == 0) {
      out->k[0] = r[0];
      out->k[1] = r[1];
    }
    if (r[2 + 2 * K] & 1) {
      out->nonfinite++;
      out->flags |= 1u;
      continue;
    }
    out->fwd_ntts += 2 * (r[0] + r[1]);  // image mode: 2 images x k slices (r[0] = r[1] = k)
    // image mode: one schedule (row 0), its groups run once per image
    for (int cv = 0; cv < 4; ++cv)
      out->groups += (pl->image ? 2 : 1) * hsched[(b * 4 + cv) * sched_stride(K, L)];
  }
  out->inv_ntts = 2 * out->groups;
  return OZFFT_OK;
}

uint64_t ozfft_shard_residue_bytes(const ozfft_plan* pl, int32_t groups) {
  if (!pl) return 0;
  const int64_t g = groups > 0 ? groups : (int64_t)pl->K * pl->K;
  return (uint64_t)8 * g * pl->n * 4;
}

static ozfft_status shard_partial_impl(const ozfft_plan* pl, int shard, int nshards, const void* in,
                                       int direction, void* residues, void* const* peers,
                                       int32_t* groups, void* stream) {
  ozfft_status s = check_exec(pl, in, residues, direction);
  if (s) return s;
  if (!groups) return fail(OZFFT_ERR_INVALID_ARGUMENT, "null groups pointer");
  if (nshards < 1 || 8 % nshards != 0 || shard < 0 || shard >= nshards)
    return fail(OZFFT_ERR_SHARD, "nshards must divide 8 and 0 <= shard < nshards");
  if (pl->image) return fail(OZFFT_ERR_SHARD, "sharding is not available for OZFFT_ACCUM_IMAGE");
  const int per = 8 / nshards;
  uint32_t mask = 0;
  for (int u = shard * per; u < (shard + 1) * per; ++u) mask |= 1u << u;
  cudaStream_t st = (cudaStream_t)stream;
  ExecArgs a{};
  a.nb = 1;
  a.in = reinterpret_cast<const double*>(in);
  a.out = nullptr;
  a.b0 = 0;
  a.direction = direction;
  a.unit_mask = mask;
  a.finish = false;
  int32_t g = pl->K * pl->K;
  if (nshards > 1) {
    // the exchange is sized by the schedule every rank computes identically: split, then
    // read the four group counts (one small D2H + sync) -- 8 * max_cv ng * n words instead
    // of the K*K capacity (160n vs 288n bytes at (K, L) = (3, 3))
    a.phase = 1;
    s = launch_execute(*pl, a, stream);
    if (s) return s;
    const int stride = sched_stride(pl->K, pl->L);
    int32_t ng[4] = {0, 0, 0, 0};
    for (int cv = 0; cv < 4 && !s; ++cv)
      s = check_cuda(cudaMemcpyAsync(&ng[cv], pl->ws + pl->woff.sched + (size_t)cv * stride * 4, 4,
                                     cudaMemcpyDeviceToHost, st), "schedule D2H");
    if (!s) s = check_cuda(cudaStreamSynchronize(st), "schedule sync");
    if (s) return s;
    g = std::max(std::max(ng[0], ng[1]), std::max(ng[2], ng[3]));
    if (g < 1) g = 1;  // no groups (zero or non-finite input): nothing is written
    a.phase = 2;
  }
  *groups = g;
  // this shard's units write straight into their place of the [8 units][g][n] exchange
  // buffer (an in-place all-gather then completes it on every rank)
  a.res_out = reinterpret_cast<uint32_t*>(residues);
  a.res_groups = g;
  if (peers) {  // peer-memory exchange: the producing kernels store into every rank's buffer
    a.npeers = nshards;
    for (int r = 0; r < nshards; ++r) a.res_peers[r] = reinterpret_cast<uint32_t*>(peers[r]);
  }
  s = launch_execute(*pl, a, stream);
  const_cast<ozfft_plan*>(pl)->last_batch = 1;
  return s;
}

ozfft_status ozfft_shard_partial(const ozfft_plan* pl, int shard, int nshards, const void* in,
                                 int direction, void* residues, int32_t* groups, void* stream) {
  return shard_partial_impl(pl, shard, nshards, in, direction, residues, nullptr, groups, stream);
}

ozfft_status ozfft_shard_partial_p2p(const ozfft_plan* pl, int shard, int nshards, const void* in,
                                     int direction, void* const* residues_by_rank, int32_t* groups,
                                     void* stream) {
  if (!residues_by_rank) return fail(OZFFT_ERR_INVALID_ARGUMENT, "null residues_by_rank");
  if (nshards < 1 || nshards > 8 || shard < 0 || shard >= nshards)
    return fail(OZFFT_ERR_SHARD, "nshards must divide 8 and 0 <= shard < nshards");
  for (int r = 0; r < nshards; ++r)
    if (!residues_by_rank[r]) return fail(OZFFT_ERR_INVALID_ARGUMENT, "null rank buffer");
  return shard_partial_impl(pl, shard, nshards, in, direction, residues_by_rank[shard], residues_by_rank,
                            groups, stream);
}

// cuMemGetAddressRange through the runtime's driver entry point (no link-time libcuda)
static ozfft_status alloc_base(const void* dev_ptr, uintptr_t* base) {
  typedef int (*GetRange)(unsigned long long*, size_t*, unsigned long long);
  static GetRange fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !f)
      return fail(OZFFT_ERR_CUDA, "cuMemGetAddressRange entry point unavailable");
    fn = reinterpret_cast<GetRange>(f);
  }
  unsigned long long b = 0;
  size_t sz = 0;
  if (fn(&b, &sz, (unsigned long long)(uintptr_t)dev_ptr) != 0)
    return fail(OZFFT_ERR_INVALID_ARGUMENT, "pointer is not in a device allocation");
  *base = (uintptr_t)b;
  return OZFFT_OK;
}

ozfft_status ozfft_ipc_get_handle(const void* dev_ptr, void* handle64, uint64_t* offset) {
  if (!dev_ptr || !handle64 || !offset) return fail(OZFFT_ERR_INVALID_ARGUMENT, "null argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "CUDA IPC handle is 64 bytes");
  uintptr_t base = 0;
  ozfft_status s = alloc_base(dev_ptr, &base);
  if (s) return s;
  cudaIpcMemHandle_t h;
  s = check_cuda(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)), "cudaIpcGetMemHandle");
  if (s) return s;
  std::memcpy(handle64, &h, sizeof(h));
  *offset = (uint64_t)((uintptr_t)dev_ptr - base);
  return OZFFT_OK;
}

ozfft_status ozfft_ipc_open_handle(const void* handle64, uint64_t offset, void** dev_ptr) {
  if (!handle64 || !dev_ptr) return fail(OZFFT_ERR_INVALID_ARGUMENT, "null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  void* base = nullptr;
  const ozfft_status s =
      check_cuda(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  if (!s) *dev_ptr = static_cast<char*>(base) + offset;
  return s;
}

ozfft_status ozfft_ipc_close(void* dev_ptr, uint64_t offset) {
  if (!dev_ptr) return fail(OZFFT_ERR_INVALID_ARGUMENT, "null argument");
  return check_cuda(cudaIpcCloseMemHandle(static_cast<char*>(dev_ptr) - offset), "cudaIpcCloseMemHandle");
}

ozfft_status ozfft_shard_finish(const ozfft_plan* pl, const void* residues_all, int32_t groups,
                                void* out, int direction, void* stream) {
  ozfft_status s = check_exec(pl, residues_all, out, direction);
  if (s) return s;
  if (pl->image) return fail(OZFFT_ERR_SHARD, "sharding is not available for OZFFT_ACCUM_IMAGE");
  if (groups < 1 || groups > pl->K * pl->K)
    return fail(OZFFT_ERR_INVALID_ARGUMENT, "groups must be the value ozfft_shard_partial returned");
  return launch_finish_from_residues(*pl, reinterpret_cast<const uint32_t*>(residues_all), groups,
                                     reinterpret_cast<double*>(out), direction, stream);
}

ozfft_status ozfft_profile_enable(ozfft_plan* pl, int on) {
  if (!pl) return fail(OZFFT_ERR_INVALID_ARGUMENT, "null plan");
  if (!pl->prof) pl->prof = new Prof();
  pl->prof->on = on != 0;
  pl->prof->recs.clear();
  pl->prof->next = 0;
  return OZFFT_OK;
}

ozfft_status ozfft_profile_read(ozfft_plan* pl, double* ms, int64_t* launches, void* stream) {
  if (!pl || !ms || !launches) return fail(OZFFT_ERR_INVALID_ARGUMENT, "null argument");
  for (int i = 0; i < OZFFT_NSTAGES; ++i) { ms[i] = 0.0; launches[i] = 0; }
  if (!pl->prof) return OZFFT_OK;
  ozfft_status s = check_cuda(cudaStreamSynchronize((cudaStream_t)stream), "profile sync");
  if (s) return s;
  for (const Prof::Rec& r : pl->prof->recs) {
    if (!r.e1) continue;
    float t = 0.f;
    if (cudaEventElapsedTime(&t, (cudaEvent_t)r.e0, (cudaEvent_t)r.e1) == cudaSuccess) {
      ms[r.stage] += t;
      launches[r.stage] += 1;
    }
  }
  pl->prof->recs.clear();
  pl->prof->next = 0;
  return OZFFT_OK;
}

uint64_t ozfft_kernel_launches(void) { return g_launches.load(); }

ozfft_status ozfft_plan_destroy(ozfft_plan* pl) {
  if (pl && pl->pipe) {
    for (void* e : pl->pipe->ev) cudaEventDestroy((cudaEvent_t)e);
    if (pl->pipe->h2d) cudaStreamDestroy((cudaStream_t)pl->pipe->h2d);
    if (pl->pipe->d2h) cudaStreamDestroy((cudaStream_t)pl->pipe->d2h);
    for (void* cs : pl->pipe->cs)
      if (cs) cudaStreamDestroy((cudaStream_t)cs);
    delete pl->pipe;
  }
  if (pl && pl->graphs) {
    for (const GraphCache::Entry& e : pl->graphs->entries) cudaGraphExecDestroy((cudaGraphExec_t)e.exec);
    if (pl->graphs->capture) cudaStreamDestroy((cudaStream_t)pl->graphs->capture);
    delete pl->graphs;
  }
  if (pl && pl->prof) {
    for (void* e : pl->prof->pool) cudaEventDestroy((cudaEvent_t)e);
    delete pl->prof;
  }
  delete pl;
  return OZFFT_OK;
}

}  // extern "C"
