// internal.h -- shared definitions of the ozfft CUDA library (not part of the ABI).
// References "P:N" = /root/reference/PAPER.md line N.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/ozfft.h"

#ifdef __CUDACC__
#define OZ_HD __host__ __device__
#else
#define OZ_HD
#endif

namespace ozfft {

constexpr int kMaxK = 8;  // split cap per real vector (plan K <= kMaxK)
constexpr int kMaxL = 8;  // accumulation bound (plan L <= kMaxL)

// Real convolutions of the complex Bluestein convolution:
// cv = 0 rr, 1 ii, 2 ir, 3 ri as (x' part a, omega~* part b).
OZ_HD inline int conv_a(int cv) { return (cv == 1 || cv == 2) ? 1 : 0; }
OZ_HD inline int conv_b(int cv) { return (cv == 1 || cv == 3) ? 1 : 0; }

// Host-side plan (immutable after bind).
struct Plan {
  // descriptor-derived
  int64_t n = 0, m = 0, batch = 0, chunk = 0;
  int K = 3, L = 3, alpha = 0, rho = 0;
  uint32_t p[2] = {0, 0};
  int logm = 0, logC = 0, logR = 0;  // m = R * C
  int64_t split_cluster_max = -1;     // longest vector for the one-launch split (-1: build default)
  int conv_mode = 0;                 // OZFFT_CONV_PADDED (m >= 2n-1) or OZFFT_CONV_CYCLIC (m = n)
  int image = 0;                     // OZFFT_ACCUM_IMAGE: complex-image accumulation (f2)
  int ts = 0;                        // OZFFT_PREC_TS: triple-single a1 / a2 / a7 (f4)
  uint32_t iota[2] = {0, 0};         // image mode: iota_q = g^((p_q - 1)/4), iota^2 = -1
  int device = 0;
  uint64_t max_ws = 0;
  int small_fused = 1;               // one-launch path of one-pass plans (env OZFFT_SMALL_FUSED=0: off)
  int small_z = 0;                   // its CTAs per (prime, part) (env OZFFT_SMALL_Z; 0: build default)
  int fault = 0;                     // test-only (env OZFFT_FAULT_INJECT at create): corrupt one residue
  // host tables (built at create)
  std::vector<double> chirp;       // [n][2] = (C_j, S_j), omega(j) = C_j + i S_j
  std::vector<double> wstar;       // [m][2] omega~* = ZeroPad_pm(conj(omega), m)
  std::vector<uint32_t> tw[2][2];  // [prime][dir] -> [m][2] = (w, shoup) at T[h + j] = w_{2h}^{+-j}
  uint32_t minv[2] = {0, 0};       // m^{-1} mod p
  uint32_t pinv[2] = {0, 0};       // -p^{-1} mod 2^32 (Montgomery REDC)
  uint32_t p0inv_mod_p1 = 0;       // Garner constant
  // sizes and layout
  uint64_t persistent_bytes = 0, workspace_bytes = 0;
  struct {
    uint64_t chirp, tw, W, wsplit, end;
  } poff{};
  struct {
    uint64_t stats, sched, mu, digits, Y, G, res, S, io_in, io_out, end;
  } woff{};
  // bound state
  bool bound = false;
  uint8_t* pers = nullptr;
  uint8_t* ws = nullptr;
  int kw[2] = {0, 0};
  int32_t Ew[2][kMaxK] = {{0}};
  int64_t last_batch = 0;  // transforms covered by the per-batch stats arrays
  struct Prof* prof = nullptr;  // profiling state (mutable through the pointer)
  struct HostPipe* pipe = nullptr;  // copy streams/events of ozfft_execute_host (lazy)
  struct GraphCache* graphs = nullptr;  // captured executes (ozfft_execute, small plans)
};

// CUDA graphs of ozfft_execute keyed by (in, out, direction): the launch sequence is
// captured on the second execute with the same buffers and replayed from then on (SURVEY 7,
// small-n latency; also the inter-kernel gaps of mid-size plans).
struct GraphCache {
  struct Entry {
    const void* in;
    void* out;
    int direction;
    void* exec;       // cudaGraphExec_t
    int launches;     // kernels in the graph (added to the launch counter per replay)
  };
  std::vector<Entry> entries;  // at most kMax, oldest replaced first
  size_t next = 0;
  // (in, out, direction) keys seen once: a key is captured on its second execute, so a
  // caller whose buffers change every call never pays for a capture
  struct Key {
    const void* in;
    void* out;
    int direction;
  };
  std::vector<Key> seen;  // at most kMax, oldest replaced first
  size_t seen_next = 0;
  void* capture = nullptr;     // cudaStream_t used for capture
  static constexpr size_t kMax = 8;
};

// Copy/compute pipelining of ozfft_execute_host: H2D and D2H run on their own streams,
// overlapping the device pipeline of neighbouring sub-batches.
struct HostPipe {
  void* h2d = nullptr;
  void* d2h = nullptr;
  void* cs[2] = {nullptr, nullptr};  // compute streams of the concurrent schedule
  std::vector<void*> ev;  // cudaEvent_t, 3 per sub-batch
};

// Per-stage CUDA-event timers (ozfft_profile_*).
struct Prof {
  bool on = false;
  std::vector<void*> pool;                     // cudaEvent_t
  size_t next = 0;
  struct Rec { int stage; void* e0; void* e1; };
  std::vector<Rec> recs;
};
void prof_mark(const Plan& pl, int stage, bool begin, void* stream);
// two-pass decompositions (log2 R, log2 C) instantiated in kernels.cu
bool decomposition_supported(int logR, int logC);
void count_launches(int n);
uint64_t launches_so_far();

// Schedule row length per (transform, conv): ngroups + K*K groups of (cexp, npairs, L pairs)
OZ_HD inline int sched_stride(int K, int L) { return 1 + K * K * (2 + 2 * L); }

// Per-transform stats record in the workspace (int32 words).
// [0..1] kv(re, im), [2..2+2K) E(re, im), [2+2K] flags (bit0 nonfinite), then mu bits (u64) separately.
OZ_HD inline int stats_stride(int K) { return 4 + 2 * K; }

void set_error(const std::string& msg);

// plan_host.cpp
ozfft_status build_plan_tables(Plan& pl);  // chirp, wstar, twiddles (host math)

// kernels.cu launchers (all asynchronous on `stream`)
struct ExecArgs {
  const double* in;    // device complex [chunk][n]
  double* out;         // device complex [chunk][n]
  int64_t b0;          // index of the first transform of the chunk within the batch
  int64_t nb;          // transforms in this chunk
  int direction;       // -1 forward, +1 inverse
  uint32_t unit_mask;  // bit (cv*2 + q): which (conv, prime) units to compute (0xFF = all)
  bool finish;         // run CRT/recombine/post-chirp
  const ozfft_taps* taps;
  int64_t ws0 = 0;     // first transform slot of the chunked workspace regions used
                       // (ws0 + nb <= chunk); disjoint slots may run on concurrent streams
  uint32_t* res_out = nullptr;  // unit-sharded transform: residues written here, [unit][res_groups][n]
  int res_groups = 0;
  uint32_t* res_peers[8] = {};  // ... and also into these buffers (peer memory), if npeers > 0
  int npeers = 0;
  int phase = 0;       // 0: whole path; 1: split only (stats, schedules); 2: everything after the split
};
ozfft_status launch_plan_precompute(Plan& pl, void* stream);
ozfft_status launch_execute(const Plan& pl, const ExecArgs& a, void* stream);
ozfft_status launch_finish_from_residues(const Plan& pl, const uint32_t* res, int groups, double* out,
                                         int direction, void* stream);

}  // namespace ozfft
