// parasim_cuda.cu -- B200 (sm_100a) strategy-evaluation path behind include/parasim.h.
//
// Kernels
//   k_rows / k_cols / k_pack
//       Region-overlap tables: for every op pair and every (src degree map, dst
//       degree map) combo, the (k, l, bytes) transfer list that _wire_pair
//       derives for one strategy (reference taskgraph.py:154-195,
//       partition.py:117-211), computed once per problem.  Rows (per src block
//       k) are sorted by l; a column index (per dst block l) serves the
//       backward pass; k_pack writes 32-byte records with the other end's task
//       slot and the transfer time per link class.
//   k_simulate_batch  one warp per candidate strategy (candidates from a work
//       queue): the task graph of the strategy is never materialised --
//       successors are walked straight out of the overlap tables -- and the
//       reference's global (ready, origin) heap order (simulate.py:68-117) is
//       reproduced exactly by lookahead rounds over a shared-memory ready set
//       (see "v2 simulator" below).  Per-queue (device / link) clocks live in
//       shared memory.
//   k_mcmc  persistent, one warp per chain: proposal (Philox4x32-10 or CPython
//       MT19937 stream), in-place fragment rewrite, re-simulation, Metropolis
//       accept, best snapshot, O(size) rollback (search.py:89-115,193-255);
//       time-boxed segments.
//   k_simulate_trace  one strategy with every task and dependency recorded
//       (the TaskGraph / timeline API); k_simulate_explicit  hand-built graphs.
//
// Exactness: the only floating-point operations on the simulated timeline are
// max() and one IEEE add per task (start + exe), plus lat + bytes/bw for
// transfers and shard/r for ring hops -- each a single correctly rounded op in
// the reference's operand order.  Built with -fmad=false.
#include <cuda_runtime.h>
#include <cub/device/device_scan.cuh>

#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <algorithm>
#include <string>
#include <vector>

#include "parasim.h"

#define FULLMASK 0xffffffffu
// threads per block the warp kernels are compiled for (registers: 65536 / this)
#ifndef PS_MAX_THREADS
#define PS_MAX_THREADS 256
#endif
// wide-problem (SIM_BACK) variants: threads per block and blocks per SM they are
// compiled for.  Their warps wait on global memory (back set, counters of big
// layouts), so more resident warps pay where they do not on the headline shape.
#ifndef PS_WIDE_THREADS
#define PS_WIDE_THREADS PS_MAX_THREADS
#endif
#ifndef PS_WIDE_MINB
#define PS_WIDE_MINB 1
#endif
#define PS_BOUNDS(S) __launch_bounds__(((S) & SIM_BACK) ? PS_WIDE_THREADS : PS_MAX_THREADS, ((S) & SIM_BACK) ? PS_WIDE_MINB : 1)

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

#define CK(x)                                                                             \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess) return fail(PS_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

enum { KIND_EDGE = 0, KIND_EDGE_BWD = 1, KIND_OP = 2, KIND_OP_BWD = 3, KIND_SYNC = 4 };
// ready-set queue field: queue index, plus a flag for tasks known to have no
// successors (the last hop of a ring), which never bound the lookahead
#define Q_SINK 0x40000000
#define Q_MASK 0x3fffffff
#define INF_BITS 0x7ff0000000000000ull

struct DevProb {
  int n_ops, n_dev, n_kinds, n_links, n_pairs, n_maps, full, n_slots, n_queues, cap;
  const int *dev_kind, *link_of;
  const double *link_bw, *link_lat;
  const int *op_ndim;
  const long long *op_dim;
  const int *op_esize, *op_param_mask, *op_map_off, *op_nmaps_enum, *op_slot_off, *slot_op;
  const int *op_in_off, *op_in_pairs, *op_out_off, *op_out_pairs;
  const int *map_deg, *map_size;
  const double *exe_fwd, *exe_bwd, *map_shard;
  const int *map_ngroups;
  const int *pair_src, *pair_dst, *pair_need_off, *need, *combo_off, *combo_row_off, *combo_col_off;
  // derived on the device
  const int *row_ent_off, *col_ent_off, *col_ent;
  const unsigned short *ent_k, *ent_l;
  const long long *ent_bytes;
  const void *ent16, *cent16;  // packed Ent32 records: rows, and column-ordered copies
  double mult;                 // backward_multiplier (exe_bwd == exe_fwd * mult, one IEEE product)
  const short *link16;         // 16-bit link table: link index, | class << 14 when n_cls > 0
  // Transfer-time classes: when the links carry at most two distinct (latency,
  // bandwidth) pairs, every overlap record also holds lat_c + bytes / bw_c for
  // each class c (the same two IEEE operations), so the simulator reads a
  // transfer's time instead of dividing.
  int n_cls;
  double cls_lat[2], cls_bw[2];
  // delta (checkpoint) evaluation: an upper bound of the dense ring-counter count,
  // and the smallest time any task can take (0: a zero-time task exists, so the
  // prefix-reuse argument does not hold and every evaluation runs from scratch)
  int n_rings;
  double min_exe;
  int snap_b;  // back-set entries a snapshot can hold (wide problems; 0: snapshots need an empty back set)
};

__host__ __device__ __forceinline__ unsigned long long pack_key(unsigned kind, unsigned a, unsigned b,
                                                               unsigned c, unsigned d) {
  return ((unsigned long long)kind << 61) | ((unsigned long long)a << 45) | ((unsigned long long)b << 29) |
         ((unsigned long long)c << 14) | (unsigned long long)d;
}
__device__ __forceinline__ unsigned key_kind(unsigned long long k) { return (unsigned)(k >> 61); }
__device__ __forceinline__ unsigned key_a(unsigned long long k) { return (unsigned)(k >> 45) & 0xffffu; }
__device__ __forceinline__ unsigned key_b(unsigned long long k) { return (unsigned)(k >> 29) & 0xffffu; }
__device__ __forceinline__ unsigned key_c(unsigned long long k) { return (unsigned)(k >> 14) & 0x7fffu; }
__device__ __forceinline__ unsigned key_d(unsigned long long k) { return (unsigned)k & 0x3fffu; }

// first index in [0, n) with a[i] > x
__device__ __forceinline__ int upper_bound(const int *a, int n, int x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ void block_bounds(const DevProb &P, int op, int g, int k, long long *lo, long long *hi) {
  int nd = P.op_ndim[op];
  for (int i = nd - 1; i >= 0; --i) {
    int d = P.map_deg[g * PS_MAXDIM + i];
    int c = k % d;
    k /= d;
    long long step = P.op_dim[op * PS_MAXDIM + i] / d;
    lo[i] = c * step;
    hi[i] = lo[i] + step;
  }
}

// Bytes src block k sends to dst block l over every tensor edge of pair p
// (taskgraph.py:168-195): sum over edges of esize * prod_dims |need ∩ block|.
__device__ long long overlap_bytes(const DevProb &P, int p, int gs, int gd, int k, int l) {
  int src = P.pair_src[p], dst = P.pair_dst[p];
  long long slo[PS_MAXDIM], shi[PS_MAXDIM], dlo[PS_MAXDIM], dhi[PS_MAXDIM];
  block_bounds(P, src, gs, k, slo, shi);
  block_bounds(P, dst, gd, l, dlo, dhi);
  int nd = P.op_ndim[src];
  long long total = 0;
  for (int e = P.pair_need_off[p]; e < P.pair_need_off[p + 1]; ++e) {
    long long prod = P.op_esize[src];
    bool ok = true;
    for (int j = 0; j < nd && ok; ++j) {
      const int *d = P.need + (e * PS_MAXDIM + j) * PS_NEED_STRIDE;
      int od = d[1];
      long long ext = d[2], nlo, nhi;
      switch (d[0]) {
        case PS_NEED_FULL: nlo = 0; nhi = ext; break;
        case PS_NEED_IDENT: nlo = dlo[od]; nhi = dhi[od]; break;
        case PS_NEED_WINDOW: {
          long long stride = d[4], pad = d[5], kern = d[3];
          nlo = dlo[od] * stride - pad;
          nhi = (dhi[od] - 1) * stride - pad + kern;
          if (nlo < 0) nlo = 0;
          if (nhi > ext) nhi = ext;
          break;
        }
        default: {  // CONCAT
          long long off = d[6];
          long long a = dlo[od] > off ? dlo[od] : off;
          long long b = dhi[od] < off + ext ? dhi[od] : off + ext;
          if (a >= b) { ok = false; nlo = nhi = 0; break; }
          nlo = a - off;
          nhi = b - off;
        }
      }
      if (!ok) break;
      long long size = P.op_dim[src * PS_MAXDIM + j];
      if (nlo < 0) nlo = 0;
      if (nhi > size) nhi = size;
      long long a = nlo > slo[j] ? nlo : slo[j];
      long long b = nhi < shi[j] ? nhi : shi[j];
      if (a >= b) { ok = false; break; }
      prod *= (b - a);
    }
    if (ok) total += prod;
  }
  return total;
}

struct ComboRef { int p, gs, gd, ns, nd; };

__device__ __forceinline__ ComboRef combo_ref(const DevProb &P, int c) {
  ComboRef r;
  r.p = upper_bound(P.combo_off, P.n_pairs + 1, c) - 1;
  int src = P.pair_src[r.p], dst = P.pair_dst[r.p];
  int nmd = P.op_map_off[dst + 1] - P.op_map_off[dst];
  int local = c - P.combo_off[r.p];
  r.gs = P.op_map_off[src] + local / nmd;
  r.gd = P.op_map_off[dst] + local % nmd;
  r.ns = P.map_size[r.gs];
  r.nd = P.map_size[r.gd];
  return r;
}

__global__ void k_rows(DevProb P, int n_rows, int n_combos, int *row_count, int *row_off_fill) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  int c = upper_bound(P.combo_row_off, n_combos + 1, r) - 1;
  int k = r - P.combo_row_off[c];
  ComboRef cr = combo_ref(P, c);
  if (row_off_fill == nullptr) {
    int cnt = 0;
    for (int l = 0; l < cr.nd; ++l) cnt += overlap_bytes(P, cr.p, cr.gs, cr.gd, k, l) > 0;
    row_count[r] = cnt;
  } else {
    int pos = row_off_fill[r];
    for (int l = 0; l < cr.nd; ++l) {
      long long b = overlap_bytes(P, cr.p, cr.gs, cr.gd, k, l);
      if (b > 0) {
        const_cast<unsigned short *>(P.ent_k)[pos] = (unsigned short)k;
        const_cast<unsigned short *>(P.ent_l)[pos] = (unsigned short)l;
        const_cast<long long *>(P.ent_bytes)[pos] = b;
        ++pos;
      }
    }
  }
}

__global__ void k_cols(DevProb P, int n_cols, int n_combos, int *col_count, const int *col_off_fill) {
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n_cols) return;
  int c = upper_bound(P.combo_col_off, n_combos + 1, q) - 1;
  int l = q - P.combo_col_off[c];
  ComboRef cr = combo_ref(P, c);
  int row0 = P.combo_row_off[c];
  int cnt = 0, pos = col_off_fill ? col_off_fill[q] : 0;
  for (int k = 0; k < cr.ns; ++k) {
    int a = P.row_ent_off[row0 + k], b = P.row_ent_off[row0 + k + 1];
    while (a < b) {  // entries of a row are sorted by l
      int m = (a + b) >> 1;
      if (P.ent_l[m] < l) a = m + 1; else b = m;
    }
    if (a < P.row_ent_off[row0 + k + 1] && P.ent_l[a] == l) {
      if (col_off_fill) const_cast<int *>(P.col_ent)[pos++] = a;
      else ++cnt;
    }
  }
  if (!col_off_fill) col_count[q] = cnt;
}

// 32-byte overlap record: k | l << 16, the task slot of the other end (row
// order: consumer block l; column order: producer block k), transfer bytes, and
// the transfer time on each link class (cost.py:128-130: latency + nbytes / bandwidth)
struct __align__(16) Ent32 { int kl; int slot; long long bytes; double exe[2]; };

__device__ inline Ent32 make_ent(const DevProb &P, int e, int n_rows, int n_combos, bool col) {
  Ent32 r;
  r.kl = (int)((unsigned)P.ent_k[e] | ((unsigned)P.ent_l[e] << 16));
  int row = upper_bound(P.row_ent_off, n_rows + 1, e) - 1;
  int pr = combo_ref(P, upper_bound(P.combo_row_off, n_combos + 1, row) - 1).p;
  r.slot = col ? P.op_slot_off[P.pair_src[pr]] + (int)P.ent_k[e] : P.op_slot_off[P.pair_dst[pr]] + (int)P.ent_l[e];
  r.bytes = P.ent_bytes[e];
  for (int c = 0; c < 2; ++c)
    r.exe[c] = c < P.n_cls ? __dadd_rn(P.cls_lat[c], __ddiv_rn((double)r.bytes, P.cls_bw[c])) : 0.0;
  return r;
}

__global__ void k_pack(DevProb P, int n_ent, int n_rows, int n_combos, void *ent32, void *cent32) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_ent) return;
  ((Ent32 *)ent32)[e] = make_ent(P, e, n_rows, n_combos, false);
  ((Ent32 *)cent32)[e] = make_ent(P, P.col_ent[e], n_rows, n_combos, true);
}

// ---------------------------------------------------------------- simulator


struct WarpSmem {
  double *qclock;
  unsigned long long *rhi, *rlo;
  int *raux;
};



struct TraceSink {
  ps_trace_task *tasks;
  int task_cap;
  int *n_tasks;
  int32_t *edge_pred;
  unsigned long long *edge_succ;
  int edge_cap;
  int *n_edges;
};

struct SimOut {
  double makespan;
  int status;
  int err_a, err_b;
};


__device__ __forceinline__ int nth_bit(unsigned long long m, int n) {
  for (int i = 0; i < n; ++i) m &= m - 1;  // (__fns is a long software sequence)
  return __ffsll((long long)m) - 1;
}

// Warp-collective append to the ready set.  `n` is warp-uniform.
__device__ __forceinline__ bool warp_push(bool want, double ready, unsigned long long key, int aux, int &n,
                                          int cap, const WarpSmem &w, int lane) {
  unsigned b = __ballot_sync(FULLMASK, want);
  if (!b) return true;
  int total = __popc(b);
  if (n + total > cap) return false;
  if (want) {
    int pos = n + __popc(b & ((1u << lane) - 1u));
    w.rhi[pos] = (unsigned long long)__double_as_longlong(ready);
    w.rlo[pos] = key;
    w.raux[pos] = aux;
  }
  n += total;
  return true;
}

// ================================================================ v2 simulator
// Latency-optimised replay used by k_simulate_batch and k_mcmc.
//
//  * Static per-op / per-pair / per-link tables are staged once per block in
//    shared memory; the candidate's degree maps, devices, per-pair combo bases,
//    queue clocks and ready set live in the warp's shared-memory slice, so the
//    only global reads on the critical path are the overlap rows/columns.
//  * Tasks get dense slots per candidate (fbase[o] + k), so the per-task
//    ready/remaining state of typical strategies also fits in shared memory
//    (larger candidates fall back to a global scratch slice).
//  * Conservative lookahead: with LB = min over the ready tasks that have
//    successors of max(ready, clock[queue]) + exe, no task that is not yet
//    ready can become ready before LB (its ready time is the end of some
//    predecessor chain rooted in the ready set, and clocks only grow).  Every
//    ready task u with ready_u < LB therefore pops before any future task, and
//    the heap pops them in (ready, origin) order.  A round runs all such tasks
//    (plus the global minimum): per queue in (ready, origin) order, queues in
//    parallel, so start = max(ready, clock[q]) is exactly the reference's
//    value.  (simulate.py:88-107; proof sketch in DESIGN.md "Lookahead rounds".)

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct Tab {  // block-shared copies of small static tables
  int *op_slot_off, *op_map_off, *op_in_off, *op_in_pairs, *op_out_off, *op_out_pairs, *op_param_mask;
  int *pair_src, *pair_dst, *combo_off, *dev_kind;
  short *link_of;                      // device pair -> link index (-1: none)
  const double *link_lat, *link_bw;    // global, read-only path
};

struct Lay {  // sizes shared by host and device
  size_t tab_bytes, warp_bytes;
  int SC;  // dense counter capacity (fwd + bwd + ring counters) kept in shared memory
  int GC;  // parameter-shard (ring) capacity
  int RC;  // staged row / column offset capacity
  int asg_global;  // device assignment read in place from global memory (very wide problems)
  int global_all;  // block tables and warp slices in global memory (problems too big for shared memory)
  int hot_bytes;   // warp slice in global memory: per-warp shared-memory slice for the per-round state (0: none)
  int warp_global; // warp slices in global memory, block tables in shared memory (wide problems)
};

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~(size_t)15; }

// per-warp phase counters of -DPS_PHASES builds (16 bytes otherwise)
#ifdef PS_PHASES
#define PH_N 40
#else
#define PH_N 2
#endif
#define PH_BYTES (PH_N * 8)

// ---------------------------------------------------------------- delta
// Checkpointed ("delta") evaluation, the B200 form of the reference's
// update_task_graph + delta_simulate (taskgraph.py:309-418, simulate.py:120-210).
//
// A simulation of strategy S records, every `stride` rounds, a snapshot of its
// state at the round boundary -- queue clocks, ready set, and per task counter
// the arrivals so far and the running ready time -- plus, per op, the first
// round in which one of its forward / backward tasks ran.  A single-op change at
// op o leaves every task that ran before the first round R_o in which a task with
// an o-dependent successor list ran (o's producers' forward tasks, o's own tasks,
// o's consumers' backward tasks) bit-identical, and touches no counter or ready
// entry of the state at that boundary except o's own (provided every task takes
// a positive time that is not absorbed into its start: then every task the
// change adds or rewires becomes ready strictly after every task already run).
// The changed strategy therefore resumes from the last snapshot at or before R_o
// (its counters rebuilt from the new in-degrees minus the recorded arrivals)
// instead of from time zero.  A source op (no producers) always runs from scratch.
// Arrivals, not remaining counts, are recorded, so snapshots stay valid for a
// later strategy that changed only ops whose tasks had not started at that point:
// an accepted proposal keeps the snapshots before its resume point and replaces
// the ones after it.
struct __align__(16) SnapHdr {
  int round, n, Tf, G;
  double makespan;
  int valid, epoch;        // epoch: in-degree buffer of the strategy that wrote it
  int nb, pad0_;           // back-set entries (wide problems)
  unsigned long long minb; // their lower bound
  int pad_[4];
};

// Snapshot layout: header, dense layout (fbase / gbase), queue clocks, ready set,
// and the raw dense counters (remaining count, ready time).  Arrivals are
// in-degree minus remaining, with the in-degrees of the writing strategy kept
// in a per-chain epoch buffer (written once per simulation, by its init).
struct SnapLay { size_t fb, gb, qc, rs, rm, rd, rb, total; };

__host__ __device__ inline size_t snap_counters(const DevProb &P) {
  return P.full ? 2 * (size_t)P.n_slots + (size_t)P.n_rings : (size_t)P.n_slots;
}

__host__ __device__ inline size_t snap_counters_pad(const DevProb &P) { return (snap_counters(P) + 7) & ~(size_t)7; }

__host__ __device__ inline SnapLay snap_layout(const DevProb &P) {
  SnapLay L;
  size_t o = sizeof(SnapHdr);
  L.fb = o; o += al16(4 * (size_t)(P.n_ops + 1));
  L.gb = o; o += al16(4 * (size_t)(P.n_ops + 1));
  L.qc = o; o += al16(8 * (size_t)P.n_queues);
  L.rs = o; o += al16(32 * (size_t)P.cap);
  L.rm = o; o += al16(2 * snap_counters_pad(P));
  L.rd = o; o += al16(8 * snap_counters_pad(P));
  L.rb = o; o += al16(32 * (size_t)P.snap_b);
  L.total = al16(o);
  return L;
}

// Per-chain delta bookkeeping (global; k_mcmc keeps it across launches)
struct ChainDelta {
  int stride, nvalid;      // snapshot spacing; indices [1, nvalid) are valid for the current strategy
  unsigned cur, bad;       // bit i: copy holding index i / index i unusable
  int fsel, pad_;          // which first-round buffer belongs to the current strategy
  long long rounds_run, rounds_reused;
  unsigned char ep[32];    // in-degree epoch buffer of the snapshot at index i (current copy)
};

// Per-simulation delta context, in the warp's shared-memory slice.
struct DeltaCtx {
  char *snap;              // this chain's snapshot slots: index i, copy b at snap + (2 i + b) snap_bytes
  const char *restore;     // snapshot to resume from (null: from time zero)
  int *frnd, *brnd;        // this simulation's first snapshot index per op at which one of its
                           // forward / backward tasks had run (0x7fffffff: not seen)
  unsigned short *indeg;   // this simulation's dense counter in-degrees (global epoch buffer)
  const unsigned short *indeg0;  // epoch buffer 0 of the chain (snapshot headers name theirs)
  unsigned long long ep_stride;  // elements per epoch buffer
  int epoch;               // this simulation's epoch buffer
  unsigned long long snap_bytes;
  int stride, nsnap;       // rounds between snapshots; snapshot indices per copy
  unsigned out_sel;        // bit i: the copy index i is written to
  int op;                  // the changed op (its counters start fresh on resume)
  int restore_idx;         // index of the resumed snapshot (0: none)
  int last;                // out: last snapshot index written
  unsigned bad;            // out: indices whose state did not fit a snapshot
  int rounds;              // out: round count at the end (resumed rounds included)
  int rounds_fwd;          // out: 1 + the last round in which a forward operator task ran
  int r0;                  // round of the resumed snapshot
  const int *fsrc, *bsrc;  // first rounds of the strategy resumed from (kept below r0)
  ChainDelta ch;           // k_mcmc: the chain's bookkeeping while the kernel runs
};



__host__ __device__ inline size_t tab_bytes_of(const DevProb &P) {
  size_t b = 0;
  b += al16(4 * (size_t)(P.n_ops + 1)) * 4;          // slot_off, map_off, in_off, out_off
  b += al16(4 * (size_t)(P.n_pairs + 1)) * 5;        // in_pairs, out_pairs, src, dst, combo_off
  b += al16(4 * (size_t)P.n_ops);                    // param mask
  b += al16(4 * (size_t)P.n_dev) + al16(2 * (size_t)P.n_dev * P.n_dev);
  return b;
}

__host__ __device__ inline size_t warp_bytes_of(const DevProb &P, int SC, int GC, int RC, int asg_global = 0) {
  size_t b = 0;
  b += al16(4 * (size_t)P.n_ops) * 2;                // mapl, gmap
  b += al16(4 * (size_t)(P.n_ops + 1)) * 2;          // fbase, gbase
  b += al16(4 * (size_t)P.n_pairs) * 2;              // prow, pcol
  b += asg_global ? 0 : al16((size_t)P.n_slots);     // asg
  b += al16(8 * (size_t)P.n_queues);                 // qclock (slow-path bids live in global scratch)
  b += al16(32 * (size_t)P.cap) + al16(4 * (size_t)P.cap);  // ready set + member list
  b += al16(8 * (size_t)P.n_ops) + 16 + 128;         // per-op forward exe cache, flags, winner lanes
  b += al16(8 * (size_t)SC) + al16(2 * (size_t)SC) + al16((size_t)SC / 2);  // counters: ready, remaining, shard id
  b += al16(8 * (size_t)GC);                         // ring device masks
  b += al16(4 * (size_t)RC) * 2;                     // staged row / column offsets
  b += 256 + PH_BYTES + 16;                          // proposal staging, phase counters
  b += al16(sizeof(DeltaCtx));                       // delta context
  b += al16(2 * (size_t)P.n_ops);                    // delta: ops seen running
  return b;
}

struct __align__(16) REnt { unsigned long long h, k; double e; int q, pad; };

struct W2 {
  int *mapl, *gmap, *fbase, *gbase, *prow, *pcol;
  unsigned char *asg;
  double *qclock;
  unsigned long long *qready, *qbest;
  REnt *rs;  // ready set: (ready bits, origin key, exe, queue | flags), one 32-byte entry each
  int *mem;
  double *exef;
  int *flags;  // [0]: slow-path queue bids may be dirty
  int *wlane;  // [32] lane holding the k-th winner of the round
  int rcap;    // ready-set capacity in effect (shared memory, or the global overflow slice)
  // Back ready set (global, unsorted): entries that did not fit in (or were
  // trimmed from) the front set w.rs.  Rounds run on the front set while the
  // back set's ready times are bounded below by the round's LB; see
  // "two-level ready set" at warp_simulate2.  bcap == 0: no back set.
  REnt *bq;
  int *bmem;
  unsigned long long *bh;  // bq[i].h mirrored: the refill's passes read 8 bytes per entry, not 32
  int bcap;
  double *opmin;  // optional [n_ops]: earliest end of each op's forward tasks (exhaustive bounds)
  const TraceSink *tr;  // optional: record every task and dependency (API materialisation)
  double *cready;
  unsigned short *crem;
  unsigned char *cgrp;
  unsigned long long *gmask;
  int *srow, *scol;
  unsigned char *oldasg;
  unsigned long long *ph;  // per-warp phase counters (PS_PHASES builds)
  DeltaCtx *dc;            // SIM_SNAP simulations: snapshots / resume
  unsigned char *ran;      // SIM_SNAP: [2 n_ops] op seen to have run a forward / backward task
};

__device__ inline void carve_tab(char *base, const DevProb &P, Tab &t) {
  char *p = base;
  auto take = [&](size_t bytes) { char *r = p; p += al16(bytes); return r; };
  t.op_slot_off = (int *)take(4 * (P.n_ops + 1));
  t.op_map_off = (int *)take(4 * (P.n_ops + 1));
  t.op_in_off = (int *)take(4 * (P.n_ops + 1));
  t.op_out_off = (int *)take(4 * (P.n_ops + 1));
  t.op_in_pairs = (int *)take(4 * (P.n_pairs + 1));
  t.op_out_pairs = (int *)take(4 * (P.n_pairs + 1));
  t.pair_src = (int *)take(4 * (P.n_pairs + 1));
  t.pair_dst = (int *)take(4 * (P.n_pairs + 1));
  t.combo_off = (int *)take(4 * (P.n_pairs + 1));
  t.op_param_mask = (int *)take(4 * P.n_ops);
  t.dev_kind = (int *)take(4 * P.n_dev);
  t.link_of = (short *)take(2 * P.n_dev * P.n_dev);
  t.link_lat = P.link_lat;
  t.link_bw = P.link_bw;
}

__device__ inline void tab_from_global(const DevProb &P, Tab &t) {
  t.op_slot_off = const_cast<int *>(P.op_slot_off);
  t.op_map_off = const_cast<int *>(P.op_map_off);
  t.op_in_off = const_cast<int *>(P.op_in_off);
  t.op_out_off = const_cast<int *>(P.op_out_off);
  t.op_in_pairs = const_cast<int *>(P.op_in_pairs);
  t.op_out_pairs = const_cast<int *>(P.op_out_pairs);
  t.pair_src = const_cast<int *>(P.pair_src);
  t.pair_dst = const_cast<int *>(P.pair_dst);
  t.combo_off = const_cast<int *>(P.combo_off);
  t.op_param_mask = const_cast<int *>(P.op_param_mask);
  t.dev_kind = const_cast<int *>(P.dev_kind);
  t.link_of = const_cast<short *>(P.link16);
  t.link_lat = P.link_lat;
  t.link_bw = P.link_bw;
}

__device__ inline void load_tab(const DevProb &P, const Tab &t) {
  int tid = threadIdx.x, nt = blockDim.x;
  for (int i = tid; i <= P.n_ops; i += nt) {
    t.op_slot_off[i] = P.op_slot_off[i];
    t.op_map_off[i] = P.op_map_off[i];
    t.op_in_off[i] = P.op_in_off[i];
    t.op_out_off[i] = P.op_out_off[i];
  }
  int nin = P.op_in_off[P.n_ops], nout = P.op_out_off[P.n_ops];
  for (int i = tid; i < nin; i += nt) t.op_in_pairs[i] = P.op_in_pairs[i];
  for (int i = tid; i < nout; i += nt) t.op_out_pairs[i] = P.op_out_pairs[i];
  for (int i = tid; i < P.n_pairs; i += nt) { t.pair_src[i] = P.pair_src[i]; t.pair_dst[i] = P.pair_dst[i]; }
  for (int i = tid; i <= P.n_pairs; i += nt) t.combo_off[i] = P.combo_off[i];
  for (int i = tid; i < P.n_ops; i += nt) t.op_param_mask[i] = P.op_param_mask[i];
  for (int i = tid; i < P.n_dev; i += nt) t.dev_kind[i] = P.dev_kind[i];
  for (int i = tid; i < P.n_dev * P.n_dev; i += nt) t.link_of[i] = P.link16[i];
}

__device__ inline void carve_warp(char *base, const DevProb &P, const Lay &L, W2 &w) {
  char *p = base;
  auto take = [&](size_t bytes) { char *r = p; p += al16(bytes); return r; };
  w.mapl = (int *)take(4 * P.n_ops);
  w.gmap = (int *)take(4 * P.n_ops);
  w.fbase = (int *)take(4 * (P.n_ops + 1));
  w.gbase = (int *)take(4 * (P.n_ops + 1));
  w.prow = (int *)take(4 * P.n_pairs);
  w.pcol = (int *)take(4 * P.n_pairs);
  w.asg = L.asg_global ? nullptr : (unsigned char *)take(P.n_slots);
  w.qclock = (double *)take(8 * P.n_queues);
  w.rs = (REnt *)take(sizeof(REnt) * P.cap);
  w.mem = (int *)take(4 * P.cap);
  w.exef = (double *)take(8 * P.n_ops);
  w.flags = (int *)take(16);
  w.wlane = (int *)take(128);
  w.cready = (double *)take(8 * L.SC);
  w.crem = (unsigned short *)take(2 * L.SC);
  w.cgrp = (unsigned char *)take(L.SC / 2);  // forward slots only: 2 Tf + G <= SC
  w.gmask = (unsigned long long *)take(8 * L.GC);
  w.srow = (int *)take(4 * L.RC);
  w.scol = (int *)take(4 * L.RC);
  w.oldasg = (unsigned char *)take(256);
  w.ph = (unsigned long long *)take(PH_BYTES);
  w.dc = (DeltaCtx *)take(sizeof(DeltaCtx));
  w.ran = (unsigned char *)take(2 * P.n_ops);
  w.rcap = P.cap;
  w.bq = nullptr;
  w.bmem = nullptr;
  w.bh = nullptr;
  w.bcap = 0;
  w.opmin = nullptr;
  w.tr = nullptr;
}

struct State {  // one candidate's dense counters (shared memory, or a global slice)
  double *ready;           // [0,Tf) forward, [Tf,2Tf) backward, [2Tf,2Tf+G) ring hop 0
  unsigned short *rem;
  unsigned char *grp;      // parameter shard of each forward slot
  unsigned long long *gmask;  // [G] ring devices per shard
  const int *rowoff, *coloff;  // staged (or global) overlap row / column offsets
  int Tf, G;
};

__host__ __device__ inline int overflow_cap(int n_slots) { return 4 * n_slots + 1024; }

__host__ __device__ inline size_t gscratch_bytes(int n_slots, int n_queues) {
  return al16((size_t)n_slots * 3 * 8) + al16((size_t)n_slots * 3 * 2) + al16((size_t)n_slots) +
         al16((size_t)n_slots * 8) + al16((size_t)n_queues * 16) + (size_t)overflow_cap(n_slots) * 44 + 256;
}

// one warp's global slice: scratch, plus its whole shared-memory layout in global mode
__host__ __device__ inline size_t gslice_bytes(const DevProb &P, const Lay &L) {
  return al16(gscratch_bytes(P.n_slots, P.n_queues)) + ((L.global_all || L.warp_global) ? L.warp_bytes : 0);
}

// The per-round state -- front ready set, member list, queue clocks, flags and
// winner lanes -- of a warp whose layout is otherwise in global memory
// (global_all): kept in shared memory when the launch provides hot_bytes per warp.
__host__ __device__ inline size_t hot_bytes_of(const DevProb &P) {
  return al16(32 * (size_t)P.cap) + al16(4 * (size_t)P.cap) + al16(8 * (size_t)P.n_queues) + 16 + 128;
}

__device__ inline void carve_hot(char *base, const DevProb &P, W2 &w) {
  char *p = base;
  auto take = [&](size_t bytes) { char *r = p; p += al16(bytes); return r; };
  w.rs = (REnt *)take(32 * (size_t)P.cap);
  w.mem = (int *)take(4 * (size_t)P.cap);
  w.qclock = (double *)take(8 * (size_t)P.n_queues);
  w.flags = (int *)take(16);
  w.wlane = (int *)take(128);
}

// prologue shared by the warp kernels: block tables and this warp's layout
__device__ inline void kernel_layout(const DevProb &P, const Lay &L, char *smem, char *gslice, int wib, Tab &T,
                                     W2 &w) {
  if (L.global_all) {
    tab_from_global(P, T);
    carve_warp(gslice + al16(gscratch_bytes(P.n_slots, P.n_queues)), P, L, w);
    if (L.hot_bytes) carve_hot(smem + (size_t)wib * L.hot_bytes, P, w);
  } else if (L.warp_global) {
    carve_tab(smem, P, T);
    load_tab(P, T);
    carve_warp(gslice + al16(gscratch_bytes(P.n_slots, P.n_queues)), P, L, w);
    carve_hot(smem + L.tab_bytes + (size_t)wib * L.hot_bytes, P, w);
  } else {
    carve_tab(smem, P, T);
    load_tab(P, T);
    carve_warp(smem + L.tab_bytes + wib * L.warp_bytes, P, L, w);
  }
}


// slow-path per-queue bid arrays (ready bits, origin key): tail of the warp's global slice
__device__ inline void bind_bids(const DevProb &P, char *gscratch, W2 &w) {
  char *g = gscratch + al16((size_t)P.n_slots * 3 * 8) + al16((size_t)P.n_slots * 3 * 2) + al16((size_t)P.n_slots) +
            al16((size_t)P.n_slots * 8);
  w.qready = (unsigned long long *)g;
  w.qbest = w.qready + P.n_queues;
  // the back ready set lives in the overflow slice
  char *b = g + al16((size_t)P.n_queues * 16);
  w.bcap = overflow_cap(P.n_slots);
  w.bq = (REnt *)b;
  w.bmem = (int *)(w.bq + w.bcap);
  w.bh = (unsigned long long *)(w.bmem + w.bcap);  // (36 bcap: 16-byte aligned, bcap = 4 n + 1024)
}

// Ready set in the warp's global slice (exact overflow path for wide candidates).
__device__ inline W2 with_global_ready_set(const DevProb &P, char *gscratch, W2 w) {
  char *g = gscratch + al16((size_t)P.n_slots * 3 * 8) + al16((size_t)P.n_slots * 3 * 2) + al16((size_t)P.n_slots) +
            al16((size_t)P.n_slots * 8) + al16((size_t)P.n_queues * 16);
  int c = overflow_cap(P.n_slots);
  w.rs = (REnt *)g;
  w.mem = (int *)(w.rs + c);
  w.rcap = c;
  w.bq = nullptr;  // (the front set now occupies the back set's slice)
  w.bmem = nullptr;
  w.bh = nullptr;
  w.bcap = 0;
  return w;
}

// simulator variants: SIM_TRACE records every task and dependency
// (k_simulate_trace), SIM_OPMIN keeps each op's earliest forward end (exhaustive
// search bounds); the MCMC kernel compiles neither
enum { SIM_TRACE = 1, SIM_OPMIN = 2, SIM_SIMPLE = 4, SIM_FULL = 8, SIM_FWD = 16, SIM_SNAP = 32, SIM_BACK = 64 };
template <int M>
__device__ SimOut warp_simulate2(const DevProb &P, const Tab &T, const W2 &w, const Lay &L, char *gscratch, int lane);

// First rounds of a delta simulation: the resumed strategy's below the resume
// round (those ops ran identically), unset above it.
__device__ inline void delta_first_rounds(const DevProb &P, const W2 &w, int lane) {
  DeltaCtx *dc = w.dc;
  __syncwarp();
  const int j = dc->restore_idx;
  const int *fs = dc->fsrc, *bs = dc->bsrc;
  int *fd = dc->frnd, *bd = dc->brnd;
  for (int i = lane; i < P.n_ops; i += 32) {
    int a = fs && j > 0 ? fs[i] : 0x7fffffff, b = bs && j > 0 ? bs[i] : 0x7fffffff;
    a = a <= j ? a : 0x7fffffff;
    b = b <= j ? b : 0x7fffffff;
    fd[i] = a;
    bd[i] = b;
    w.ran[i] = a <= j;
    w.ran[P.n_ops + i] = b <= j;
  }
  __syncwarp();
}

// Simulate; a candidate whose ready set outgrows shared memory is re-run with
// the ready set in global memory (same answer, slower).
template <int M>
__device__ inline SimOut simulate_any(const DevProb &P, const Tab &T, const W2 &w, const Lay &L, char *gscratch,
                                      int lane) {
  // one inlined copy of the simulator per call site (the code is large: keep it in the instruction cache)
  SimOut o;
  W2 wg = w;
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    if (M & SIM_SNAP) delta_first_rounds(P, w, lane);
    o = warp_simulate2<M>(P, T, wg, L, gscratch, lane);
    if (o.status != PS_STATUS_CAPACITY) break;
    wg = with_global_ready_set(P, gscratch, w);
  }
  return o;
}

// warp-wide lexicographic min of 64-bit (hi, lo) pairs; returns winning lane
__device__ __forceinline__ int warp_argmin128(unsigned long long hi, unsigned long long lo, int lane) {
  unsigned cand = FULLMASK, v, mn;
  v = (unsigned)(hi >> 32); mn = __reduce_min_sync(FULLMASK, v); cand = __ballot_sync(FULLMASK, v == mn);
  v = (cand >> lane & 1) ? (unsigned)hi : 0xffffffffu; mn = __reduce_min_sync(FULLMASK, v);
  cand &= __ballot_sync(FULLMASK, v == mn);
  v = (cand >> lane & 1) ? (unsigned)(lo >> 32) : 0xffffffffu; mn = __reduce_min_sync(FULLMASK, v);
  cand &= __ballot_sync(FULLMASK, v == mn);
  v = (cand >> lane & 1) ? (unsigned)lo : 0xffffffffu; mn = __reduce_min_sync(FULLMASK, v);
  cand &= __ballot_sync(FULLMASK, v == mn);
  return __ffs(cand) - 1;
}

__device__ __forceinline__ unsigned long long warp_min64(unsigned long long x, int lane) {
  unsigned v = (unsigned)(x >> 32), mn = __reduce_min_sync(FULLMASK, v);
  unsigned lo = v == mn ? (unsigned)x : 0xffffffffu;
  unsigned mlo = __reduce_min_sync(FULLMASK, lo);
  return ((unsigned long long)mn << 32) | mlo;
}

template <bool BACK>
__device__ __forceinline__ bool push2(bool want, double ready, unsigned long long key, double exe, int q, int &n,
                                      int &nb, unsigned long long &minb, const DevProb &P, const W2 &w, int lane) {
  unsigned bm = __ballot_sync(FULLMASK, want);
  if (!bm) return true;
  int total = __popc(bm);
  int room = w.rcap - n;
  if (!BACK && total > room) return false;  // (the caller re-runs with the ready set in global memory)
  if (BACK && total > room) {
    // the front set is full: the rest go to the back set (minb: their lower bound)
    int spill = total - room;  // (room >= 0: the front set never exceeds its capacity)
    if (nb + spill > w.bcap) return false;
    int pos = __popc(bm & ((1u << lane) - 1u));
    unsigned long long hb = (unsigned long long)__double_as_longlong(ready);
    if (want) {
      REnt r;
      r.h = hb; r.k = key; r.e = exe; r.q = q; r.pad = 0;
      if (pos < room) w.rs[n + pos] = r;
      else { w.bq[nb + pos - room] = r; w.bh[nb + pos - room] = hb; }
    }
    minb = min(minb, warp_min64(want && pos >= room ? hb : ~0ull, lane));
    n += room;
    nb += spill;
    return true;
  }
  if (want) {
    int pos = n + __popc(bm & ((1u << lane) - 1u));
    REnt r;
    r.h = (unsigned long long)__double_as_longlong(ready); r.k = key; r.e = exe; r.q = q; r.pad = 0;
    w.rs[pos] = r;
  }
  n += total;
  return true;
}

__device__ __forceinline__ int group_of2(const DevProb &P, int op, int g, int k, int pm) {
  int nd = P.op_ndim[op];
  int coords[PS_MAXDIM];
  for (int i = nd - 1; i >= 0; --i) {
    int dg = P.map_deg[g * PS_MAXDIM + i];
    coords[i] = k % dg;
    k /= dg;
  }
  int si = 0;
  for (int i = 0; i < nd; ++i)
    if (pm >> i & 1) si = si * P.map_deg[g * PS_MAXDIM + i] + coords[i];
  return si;
}

// Candidate setup: maps, dense bases, staged overlap offsets, state placement.
__device__ inline State setup_candidate(const DevProb &P, const Tab &T, const W2 &w, const Lay &L, char *gscratch,
                                        int lane) {
  int carry = 0, gcarry = 0;
  for (int base = 0; base < P.n_ops; base += 32) {
    int o = base + lane;
    int sz = 0, ng = 0;
    if (o < P.n_ops) {
      int g = T.op_map_off[o] + w.mapl[o];
      w.gmap[o] = g;
      sz = P.map_size[g];
      ng = T.op_param_mask[o] >= 0 ? P.map_ngroups[g] : 0;
      if (P.n_kinds == 1) w.exef[o] = P.exe_fwd[g];
    }
    int a = sz, b = ng;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      int ya = __shfl_up_sync(FULLMASK, a, off), yb = __shfl_up_sync(FULLMASK, b, off);
      if (lane >= off) { a += ya; b += yb; }
    }
    if (o < P.n_ops) { w.fbase[o] = carry + a - sz; w.gbase[o] = gcarry + b - ng; }
    carry += __shfl_sync(FULLMASK, a, 31);
    gcarry += __shfl_sync(FULLMASK, b, 31);
  }
  if (lane == 0) { w.fbase[P.n_ops] = carry; w.gbase[P.n_ops] = gcarry; }
  // per pair: global row/col base of the current combo and the staged layout
  int rcarry = 0, ccarry = 0;
  for (int base = 0; base < P.n_pairs; base += 32) {
    int p = base + lane;
    int nr = 0, nc = 0;
    if (p < P.n_pairs) {
      int s = T.pair_src[p], d = T.pair_dst[p];
      nr = P.map_size[w.gmap[s]] + 1;
      nc = P.full ? P.map_size[w.gmap[d]] + 1 : 0;
    }
    int a = nr, b = nc;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      int ya = __shfl_up_sync(FULLMASK, a, off), yb = __shfl_up_sync(FULLMASK, b, off);
      if (lane >= off) { a += ya; b += yb; }
    }
    if (p < P.n_pairs) {
      w.prow[p] = rcarry + a - nr;  // staged base (replaced by the global row if not staged)
      w.pcol[p] = ccarry + b - nc;
    }
    rcarry += __shfl_sync(FULLMASK, a, 31);
    ccarry += __shfl_sync(FULLMASK, b, 31);
  }
  __syncwarp();
  bool stage_r = rcarry <= L.RC, stage_c = ccarry <= L.RC;
  for (int p = lane; p < P.n_pairs; p += 32) {
    int s = T.pair_src[p], d = T.pair_dst[p];
    int nmd = T.op_map_off[d + 1] - T.op_map_off[d];
    int cc = T.combo_off[p] + w.mapl[s] * nmd + w.mapl[d];
    int grow = P.combo_row_off[cc], gcol = P.combo_col_off[cc];
    int nr = P.map_size[w.gmap[s]] + 1, nc = P.map_size[w.gmap[d]] + 1;
    if (stage_r) {
      int dst = w.prow[p];
      for (int k = 0; k < nr; ++k) w.srow[dst + k] = P.row_ent_off[grow + k];
    } else {
      w.prow[p] = grow;
    }
    if (P.full) {
      if (stage_c) {
        int dst = w.pcol[p];
        for (int k = 0; k < nc; ++k) w.scol[dst + k] = P.col_ent_off[gcol + k];
      } else {
        w.pcol[p] = gcol;
      }
    }
  }
  State st;
  st.Tf = carry;
  st.G = gcarry;
  st.rowoff = stage_r ? w.srow : P.row_ent_off;
  st.coloff = stage_c ? w.scol : P.col_ent_off;
  int need = P.full ? 2 * carry + gcarry : carry;
  if (need <= L.SC && gcarry <= L.GC) {
    st.ready = w.cready; st.rem = w.crem; st.grp = w.cgrp; st.gmask = w.gmask;
  } else {
    char *g = gscratch;
    st.ready = (double *)g; g += al16((size_t)P.n_slots * 3 * 8);
    st.rem = (unsigned short *)g; g += al16((size_t)P.n_slots * 3 * 2);
    st.grp = (unsigned char *)g; g += al16((size_t)P.n_slots);
    st.gmask = (unsigned long long *)g;
  }
  __syncwarp();
  return st;
}

// exe time / queue of a transfer between devices da -> db carrying nb bytes
// simple: the problem has one device kind, <= 2 link classes and a link between
// every pair of devices (a compile-time constant in the evaluation kernels'
// common variant, which drops the other paths and the missing-route checks)
__device__ __forceinline__ bool link_attrs(const DevProb &P, const Tab &T, int da, int db, double nb, int &q,
                                           double &exe, bool simple = false) {
  int lv = T.link_of[da * P.n_dev + db];
  if (!simple && lv < 0) return false;
  if (simple || P.n_cls) {
    q = P.n_dev + (lv & 0x3fff);
    exe = ((lv >> 14) ? P.cls_lat[1] : P.cls_lat[0]) + nb / ((lv >> 14) ? P.cls_bw[1] : P.cls_bw[0]);
  } else {
    q = P.n_dev + lv;
    exe = __ldg(&T.link_lat[lv]) + nb / __ldg(&T.link_bw[lv]);
  }
  return true;
}

__device__ __forceinline__ void op_attrs(const DevProb &P, const Tab &T, const W2 &w, unsigned kind, int a, int c,
                                         int &q, double &exe, bool simple = false) {
  int dev = w.asg[T.op_slot_off[a] + c];
  q = dev;
  if (simple || P.n_kinds == 1) exe = kind == KIND_OP ? w.exef[a] : __dmul_rn(w.exef[a], P.mult);
  else exe = (kind == KIND_OP ? P.exe_fwd : P.exe_bwd)[w.gmap[a] * P.n_kinds + T.dev_kind[dev]];
}

__device__ __forceinline__ bool sync_attrs(const DevProb &P, const Tab &T, const W2 &w, const State &st, int a, int si,
                                           int hop, int &q, double &exe, int &ea, int &eb, bool simple = false) {
  int gi = w.gbase[a] + si;
  unsigned long long msk = st.gmask[gi];
  int r = __popcll((long long)msk);
  int h0 = hop < r ? hop : hop - r, h1 = hop + 1 < r ? hop + 1 : hop + 1 - r;  // hop < 2 (r - 1)
  int da = nth_bit(msk, h0), db = nth_bit(msk, h1);
  // bytes per hop (taskgraph.py:245): computed when hop 0 becomes ready and
  // kept in the ring's counter slot, which is free from then on
  double *per = &st.ready[2 * st.Tf + gi];
  double nb;
  if (hop == 0) { nb = P.map_shard[w.gmap[a]] / (double)r; *per = nb; }
  else nb = *per;
  if (!link_attrs(P, T, da, db, nb, q, exe, simple)) { ea = da; eb = db; return false; }
  if (hop + 1 >= 2 * (r - 1)) q |= Q_SINK;
  return true;
}

// queue / time of the transfer an overlap record creates between da -> db
__device__ __forceinline__ bool link_attrs_ent(const DevProb &P, const Tab &T, int da, int db, const Ent32 &en,
                                               int &q, double &exe, bool simple = false) {
  if (!simple && !P.n_cls) return link_attrs(P, T, da, db, (double)en.bytes, q, exe);
  int lv = T.link_of[da * P.n_dev + db];
  if (!simple && lv < 0) return false;
  q = P.n_dev + (lv & 0x3fff);
  exe = (lv >> 14) ? en.exe[1] : en.exe[0];
  return true;
}

#ifdef PS_TCYC
// cycle timeline of one simulation of warp 0 of block 0 (debug builds)
__device__ long long g_tc[4096 * 16];
__device__ int g_tc_sim;
#define TC(i) do { if (tc_on && lane == 0 && tc_r < 4096) g_tc[tc_r * 16 + (i)] = clock64(); } while (0)
#else
#define TC(i)
#endif
#ifdef PS_PHASES
__device__ unsigned long long g_phase[PH_N];
#define PH_T(v) long long v = clock64()
#define PH_ADD(i, t0) do { if (lane == 0) w.ph[i] += (unsigned long long)(clock64() - (t0)); } while (0)
#define PH_CNT(i, x) do { if (lane == 0) w.ph[i] += (unsigned long long)(x); } while (0)
#else
#define PH_T(v)
#define PH_ADD(i, t0)
#define PH_CNT(i, x)
#endif

// Transfer bytes of an edge task from its key (trace mode only): row k of the
// pair's current combo, searched for column l.
__device__ inline double trace_nbytes(const DevProb &P, const Tab &T, const W2 &w, const State &st,
                                      unsigned long long key) {
  unsigned kind = key_kind(key);
  int a = key_a(key), b = key_b(key), c = key_c(key), d = key_d(key);
  if (kind == KIND_SYNC) {
    unsigned long long msk = st.gmask[w.gbase[a] + b];
    return P.map_shard[w.gmap[a]] / (double)__popcll((long long)msk);
  }
  if (kind != KIND_EDGE && kind != KIND_EDGE_BWD) return 0.0;
  for (int i = T.op_out_off[a]; i < T.op_out_off[a + 1]; ++i) {
    int p = T.op_out_pairs[i];
    if (T.pair_dst[p] != b) continue;
    int row = w.prow[p] + c;
    for (int e = st.rowoff[row]; e < st.rowoff[row + 1]; ++e)
      if ((int)P.ent_l[e] == d) return (double)P.ent_bytes[e];
  }
  return 0.0;
}

__device__ __forceinline__ void copy16(void *dst, const void *src, size_t bytes, int lane) {
  const int4 *s4 = (const int4 *)src;
  int4 *d4 = (int4 *)dst;
  int n = (int)((bytes + 15) >> 4);
  for (int i = lane; i < n; i += 32) d4[i] = s4[i];
}

// Snapshot of the simulation state at the start of round `round` (index i):
// vector copies of the dense layout, queue clocks, ready set and raw counters.
// A ready set larger than a snapshot holds marks the index unusable.
__device__ __forceinline__ void snap_write(const DevProb &P, const W2 &w, const State &st, int n, int nb,
                                           unsigned long long minb, int round, int i, double mk, bool full,
                                           int lane) {
  DeltaCtx *dc = w.dc;
  const SnapLay sl = snap_layout(P);
  char *dst = dc->snap + (2ull * (unsigned)i + ((dc->out_sel >> i) & 1u)) * dc->snap_bytes;
  const int nc = full ? 2 * st.Tf + st.G : st.Tf;
  bool ok = n <= P.cap && nb <= P.snap_b;
  unsigned long long mb = (unsigned long long)__double_as_longlong(mk);
  unsigned hi = __reduce_max_sync(FULLMASK, (unsigned)(mb >> 32));
  unsigned lo = __reduce_max_sync(FULLMASK, (unsigned)(mb >> 32) == hi ? (unsigned)mb : 0u);
  if (lane == 0) {
    SnapHdr h;
    h.round = round; h.n = n; h.Tf = st.Tf; h.G = st.G; h.valid = ok; h.epoch = dc->epoch;
    h.nb = nb; h.pad0_ = 0; h.minb = minb;
    h.makespan = __longlong_as_double((long long)(((unsigned long long)hi << 32) | lo));
    *(SnapHdr *)dst = h;
    dc->last = i;
    if (!ok) dc->bad |= 1u << i;
  }
  if (!ok) return;
  // ops seen to have run a task before this round: a task that ran has no
  // remaining count and is not in the ready set (ready-set op tasks are marked
  // with a count of 0xffff meanwhile; the raw copy below is taken before)
  copy16(dst + sl.rm, st.rem, 2 * (size_t)nc, lane);
  __syncwarp();
  for (int j = lane; j < n + nb; j += 32) {
    const unsigned long long k = j < n ? w.rs[j].k : w.bq[j - n].k;
    unsigned kd = key_kind(k);
    if (kd == KIND_OP || kd == KIND_OP_BWD) st.rem[(kd == KIND_OP ? 0 : st.Tf) + w.fbase[key_a(k)] + key_c(k)] = 0xffff;
  }
  __syncwarp();
  const int ndir = full ? 2 : 1;
  for (int x = lane; x < ndir * P.n_ops; x += 32) {
    if (w.ran[x]) continue;
    int o = x < P.n_ops ? x : x - P.n_ops;
    int base = (x < P.n_ops ? 0 : st.Tf) + w.fbase[o], sz = w.fbase[o + 1] - w.fbase[o];
    bool r = false;
    for (int k = 0; k < sz && !r; ++k) r = st.rem[base + k] == 0;
    if (r) {
      w.ran[x] = 1;
      (x < P.n_ops ? dc->frnd : dc->brnd)[o] = i;
    }
  }
  __syncwarp();
  for (int j = lane; j < n + nb; j += 32) {
    const unsigned long long k = j < n ? w.rs[j].k : w.bq[j - n].k;
    unsigned kd = key_kind(k);
    if (kd == KIND_OP || kd == KIND_OP_BWD) st.rem[(kd == KIND_OP ? 0 : st.Tf) + w.fbase[key_a(k)] + key_c(k)] = 0;
  }
  __syncwarp();
  copy16(dst + sl.fb, w.fbase, 4 * (size_t)(P.n_ops + 1), lane);
  if (full) copy16(dst + sl.gb, w.gbase, 4 * (size_t)(P.n_ops + 1), lane);
  copy16(dst + sl.qc, w.qclock, 8 * (size_t)P.n_queues, lane);
  copy16(dst + sl.rs, w.rs, 32 * (size_t)n, lane);
  if (nb) copy16(dst + sl.rb, w.bq, 32 * (size_t)nb, lane);
  copy16(dst + sl.rd, st.ready, 8 * (size_t)nc, lane);
}

// ---- two-level ready set helpers (warp_simulate2)

// LB over the back set: min over entries with successors of max(ready, clock) + exe
__device__ __forceinline__ unsigned long long back_lb(const W2 &w, int nb, int lane) {
  unsigned long long lb = INF_BITS;
  for (int i = lane; i < nb; i += 32) {
    REnt e = w.bq[i];
    if (!(e.q & Q_SINK)) {
      double r0 = __longlong_as_double((long long)e.h), ck = w.qclock[e.q & Q_MASK];
      unsigned long long eb = (unsigned long long)__double_as_longlong((r0 < ck ? ck : r0) + e.e);
      lb = eb < lb ? eb : lb;
    }
  }
  return warp_min64(lb, lane);
}

// Move every back entry ready before X (bits) to the front set, compacting the
// back set and recomputing its bound.  If they do not all fit, X drops to the
// largest of 32 evenly spaced boundaries between the back set's earliest ready
// time and X below which they do (refined twice more inside the first
// interval when even it overflows); the moved set stays downward closed, and
// holds at least the back set's earliest entry.  False (nothing moved) if no
// such boundary is found.
__device__ __forceinline__ bool back_refill(const W2 &w, int &n, int &nb, unsigned long long &minb,
                                            unsigned long long X, int lane) {
  // one pass over the ready times: the entries to move (their positions, in
  // order, while they fit), the minimum of those that stay, and the minimum
  const int room = w.rcap - n;
  int *idx = w.mem;  // (the slow path's member list: free between rounds; rcap ints)
  const unsigned lt = (1u << lane) - 1u;
  int cnt = 0;
  unsigned long long mn = ~0ull, mnk = ~0ull;
#pragma unroll 4
  for (int base = 0; base < nb; base += 32) {
    int i = base + lane;
    unsigned long long h = i < nb ? w.bh[i] : ~0ull;
    bool mv = h < X;
    unsigned bm = __ballot_sync(FULLMASK, mv);
    int pos = cnt + __popc(bm & lt);
    if (mv && pos < room) idx[pos] = i;
    cnt += __popc(bm);
    if (!mv) mnk = h < mnk ? h : mnk;
    mn = h < mn ? h : mn;
  }
  if (cnt <= room && cnt <= 1024) {
    // few to move (the usual case): copy them out, then fill the holes they
    // leave below the new end with the survivors of the tail, in order
    __syncwarp();
    for (int k = lane; k < cnt; k += 32) w.rs[n + k] = w.bq[idx[k]];
    const int nb2 = nb - cnt;
    unsigned *mask = (unsigned *)w.wlane;  // bit t: tail position nb2 + t moved (cnt <= room <= 1024)
    for (int k = lane; k < (cnt + 31) / 32; k += 32) mask[k] = 0u;
    __syncwarp();
    for (int k = lane; k < cnt; k += 32)
      if (idx[k] >= nb2) atomicOr(&mask[(idx[k] - nb2) >> 5], 1u << ((idx[k] - nb2) & 31));
    __syncwarp();
    int carry = 0;
    for (int tb = 0; tb < cnt; tb += 32) {
      int t = tb + lane;
      bool surv = t < cnt && !((mask[t >> 5] >> (t & 31)) & 1u);
      unsigned bs = __ballot_sync(FULLMASK, surv);
      if (surv) {  // (holes < nb2 <= survivors)
        const int d = idx[carry + __popc(bs & lt)];
        w.bq[d] = w.bq[nb2 + t];
        w.bh[d] = w.bh[nb2 + t];
      }
      carry += __popc(bs);
    }
    n += cnt;
    nb = nb2;
    minb = warp_min64(mnk, lane);
    __syncwarp();
    return true;
  }
  if (cnt > room) {
    if (X == ~0ull || room < 1) return false;
    mn = warp_min64(mn, lane);
    int *hist = w.wlane;  // (32 ints, free until the round picks its winners)
    unsigned long long hiX = X;
    bool found = false;
#pragma unroll 1
    for (int level = 0; level < 3 && !found; ++level) {
      // boundary j (lane j): mn + (hiX - mn) (j + 1) / 32, the last one hiX itself
      // (non-decreasing in the lane: monotone rounding, clamped to hiX)
      const double lo = __longlong_as_double((long long)mn), hi = __longlong_as_double((long long)hiX);
      unsigned long long bj = lane == 31 ? hiX
                                         : (unsigned long long)__double_as_longlong(
                                               lo + (hi - lo) * ((double)(lane + 1) * 0.03125));
      bj = bj < hiX ? bj : hiX;
      hist[lane] = 0;
      __syncwarp();
      for (int base = 0; base < nb; base += 32) {
        int i = base + lane;
        unsigned long long h = i < nb ? w.bh[i] : ~0ull;
        int b = 0;  // first boundary above h (when h < hiX)
#pragma unroll
        for (int st = 16; st >= 1; st >>= 1) {
          unsigned long long x = __shfl_sync(FULLMASK, bj, b + st - 1);
          if (!(h < x)) b += st;
        }
        if (h < hiX) atomicAdd(&hist[b], 1);
      }
      __syncwarp();
      int c = hist[lane];  // entries ready before boundary `lane`: inclusive scan
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        int y = __shfl_up_sync(FULLMASK, c, off);
        if (lane >= off) c += y;
      }
      unsigned ok = __ballot_sync(FULLMASK, c <= room);  // a leading run (c is non-decreasing)
      __syncwarp();
      const int jb = __popc(ok) - 1;
      const int cj = __shfl_sync(FULLMASK, c, max(jb, 0));
      if (jb >= 0 && cj > 0) {
        X = __shfl_sync(FULLMASK, bj, jb);
        found = true;
      } else {
        hiX = __shfl_sync(FULLMASK, bj, 0);  // refine inside the first interval
        if (hiX <= mn) break;
      }
    }
    if (!found) return false;
  }
  int kept = 0;
  unsigned long long mb = ~0ull;
  for (int base = 0; base < nb; base += 32) {
    int i = base + lane;
    bool v = i < nb;
    REnt e;
    if (v) e = w.bq[i];
    bool mv = v && e.h < X, kp = v && !mv;
    unsigned bm = __ballot_sync(FULLMASK, mv), bk = __ballot_sync(FULLMASK, kp);
    __syncwarp();  // (in-place compaction: every lane has read its entry)
    if (mv) w.rs[n + __popc(bm & lt)] = e;
    if (kp) {
      w.bq[kept + __popc(bk & lt)] = e;
      w.bh[kept + __popc(bk & lt)] = e.h;
      mb = e.h < mb ? e.h : mb;
    }
    n += __popc(bm);
    kept += __popc(bk);
  }
  nb = kept;
  minb = warp_min64(mb, lane);
  __syncwarp();
  return true;
}

// Keep about the 32 earliest front entries: T = the 33rd smallest ready time
// among the first 128 (bitonic sort, four per lane); entries ready at or after
// T move to the back set, whose bound becomes min(minb, T).  Any T is exact
// (only the split changes).
__device__ __forceinline__ bool front_trim(const W2 &w, int &n, int &nb, unsigned long long &minb, int lane,
                                           bool by_hist) {
  unsigned long long T;
  if (by_hist) {
  // threshold from a 32-bin histogram of the front's ready times between their
  // minimum and maximum: the largest boundary that keeps 1..48 entries (else the
  // first boundary that keeps any)
  unsigned long long lo = ~0ull, hi = 0ull;
  for (int i = lane; i < n; i += 32) {
    const unsigned long long h = w.rs[i].h;
    lo = h < lo ? h : lo;
    hi = h > hi ? h : hi;
  }
  lo = warp_min64(lo, lane);
  hi = ~warp_min64(~hi, lane);
  if (lo == hi) return true;  // (all tied: keep everything)
  unsigned long long bj;
  {
    const double dl = __longlong_as_double((long long)lo), dh = __longlong_as_double((long long)hi);
    bj = lane == 31 ? hi : (unsigned long long)__double_as_longlong(dl + (dh - dl) * ((double)(lane + 1) * 0.03125));
    bj = bj < hi ? bj : hi;
  }
  int *hist = w.wlane;  // (32 ints, free until the next round picks its winners)
  hist[lane] = 0;
  __syncwarp();
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    const unsigned long long h = i < n ? w.rs[i].h : ~0ull;
    int b = 0;  // first boundary above h (when h < hi)
#pragma unroll
    for (int st = 16; st >= 1; st >>= 1) {
      unsigned long long x = __shfl_sync(FULLMASK, bj, b + st - 1);
      if (!(h < x)) b += st;
    }
    if (h < hi) atomicAdd(&hist[b], 1);
  }
  __syncwarp();
  int c = hist[lane];
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    int y = __shfl_up_sync(FULLMASK, c, off);
    if (lane >= off) c += y;
  }
  const unsigned okm = __ballot_sync(FULLMASK, c >= 1 && c <= 48), anym = __ballot_sync(FULLMASK, c >= 1);
  const int jb = okm ? 31 - __clz(okm) : __ffs(anym) - 1;  // (anym != 0: lo < bj[31] = hi)
  T = __shfl_sync(FULLMASK, bj, jb);
  __syncwarp();
  } else {
  unsigned long long v[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    int i = j * 32 + lane;
    v[j] = i < n ? w.rs[i].h : ~0ull;
  }
#pragma unroll
  for (int k = 2; k <= 128; k <<= 1) {
#pragma unroll
    for (int sd = k >> 1; sd > 0; sd >>= 1) {
      if (sd >= 32) {
        const int js = sd >> 5;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (j & js) continue;
          const int j2 = j | js;
          const bool up = ((j * 32 + lane) & k) == 0;
          unsigned long long a = v[j], b = v[j2];
          if ((a > b) == up) { v[j] = b; v[j2] = a; }
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          unsigned long long o = __shfl_xor_sync(FULLMASK, v[j], sd);
          const bool up = ((j * 32 + lane) & k) == 0, lower = (lane & sd) == 0;
          v[j] = (lower == up) ? (v[j] < o ? v[j] : o) : (v[j] > o ? v[j] : o);
        }
      }
    }
  }
  T = __shfl_sync(FULLMASK, v[1], 0);
  const unsigned long long lo = __shfl_sync(FULLMASK, v[0], 0);
  if (T == lo) return true;  // (ties at the minimum: keep everything)
  }
  int evict = 0;
  for (int i = lane; i < n; i += 32) evict += w.rs[i].h >= T ? 1 : 0;
  evict = (int)__reduce_add_sync(FULLMASK, (unsigned)evict);
  if (nb + evict > w.bcap) return false;
  int kept = 0;
  const unsigned lt = (1u << lane) - 1u;
  for (int base = 0; base < n; base += 32) {
    int i = base + lane;
    bool v2 = i < n;
    REnt e;
    if (v2) e = w.rs[i];
    bool ev = v2 && e.h >= T, kp = v2 && !ev;
    unsigned be = __ballot_sync(FULLMASK, ev), bk = __ballot_sync(FULLMASK, kp);
    __syncwarp();
    if (ev) { w.bq[nb + __popc(be & lt)] = e; w.bh[nb + __popc(be & lt)] = e.h; }
    if (kp) w.rs[kept + __popc(bk & lt)] = e;
    nb += __popc(be);
    kept += __popc(bk);
  }
  n = kept;
  minb = T < minb ? T : minb;
  __syncwarp();
  return true;
}

// (warp_simulate2) the front set's LB (bits) is known: refill from the back set
// and restart the round when the back set could matter
#define BACK_CHECK(LBBITS)                                                                   \
  if (BACK && nb > 0 && !refilled && minb < (LBBITS)) {                                      \
    const unsigned long long X_ = (LBBITS) == INF_BITS ? ~0ull : (LBBITS);                   \
    if (!back_refill(w, n, nb, minb, X_, lane)) pend_bslow = true;                           \
    refilled = true;                                                                         \
    PH_CNT(21, 1);                                                                           \
    PH_ADD(32, t_sel);                                                                       \
    continue;                                                                                \
  }

template <int M>
__device__ SimOut warp_simulate2(const DevProb &P, const Tab &T, const W2 &w, const Lay &L, char *gscratch, int lane) {
  const bool trim_hist = !L.global_all;  // front-trim threshold method (see the trim at the end of a round)
  constexpr bool SIMPLE = (M & SIM_SIMPLE) != 0;  // one device kind, <= 2 link classes, full mesh
  constexpr bool SNAP = (M & SIM_SNAP) != 0;      // delta evaluation: snapshots, first rounds, resume
  constexpr bool BACK = (M & SIM_BACK) != 0;      // wide problems: two-level ready set (front + back)
  // mode known at compile time in the specialised variants (forward mode then
  // drops every backward / ring path)
  constexpr int MODE = (M & SIM_FULL) ? 1 : (M & SIM_FWD) ? 0 : -1;
  const bool FULL = MODE == 1 ? true : MODE == 0 ? false : (P.full != 0);
  SimOut out;
  out.makespan = 0.0;
  out.status = PS_STATUS_OK;
  out.err_a = out.err_b = -1;
#ifdef PS_TCYC
  bool tc_on = false;
  int tc_r = 0;
  if (threadIdx.x == 0 && blockIdx.x == 1) tc_on = atomicAdd(&g_tc_sim, 1) == 5;
#endif
  PH_T(t_setup);
  State st = setup_candidate(P, T, w, L, gscratch, lane);
  PH_ADD(0, t_setup);
  PH_CNT(8, 1);
  PH_CNT(9, st.rowoff == w.srow ? 1 : 0);
  const int Tf = st.Tf;
  PH_CNT(10, (FULL ? 2 * Tf + st.G : Tf) <= L.SC ? 1 : 0);
  const Ent32 *ent = (const Ent32 *)P.ent16;
  const Ent32 *cent = (const Ent32 *)P.cent16;
  const bool was_dirty = w.flags[0] != 0;
  for (int q = lane; q < P.n_queues; q += 32) {
    w.qclock[q] = 0.0;
    if (was_dirty) { w.qready[q] = ~0ull; w.qbest[q] = ~0ull; }
  }
  __syncwarp();
  if (lane == 0) w.flags[0] = 0;
  bool dirty = false;  // register copy of w.flags[0] for this simulation
  if (FULL)
    for (int s = lane; s < st.G; s += 32) st.gmask[s] = 0ull;
  __syncwarp();
  // ---- init: in-degrees, ring membership
  PH_T(t_init);
  for (int s = lane; s < Tf; s += 32) {
    int o = upper_bound(w.fbase, P.n_ops + 1, s) - 1;
    int k = s - w.fbase[o];
    int indeg = 0;
    for (int i = T.op_in_off[o]; i < T.op_in_off[o + 1]; ++i) {
      int col = w.pcol[T.op_in_pairs[i]] + k;
      if (FULL) indeg += st.coloff[col + 1] - st.coloff[col];
      else {  // forward mode: columns are not staged; count from the global index
        int p = T.op_in_pairs[i];
        int sp = T.pair_src[p];
        int nmd = T.op_map_off[o + 1] - T.op_map_off[o];
        int gc = P.combo_col_off[T.combo_off[p] + w.mapl[sp] * nmd + w.mapl[o]] + k;
        indeg += P.col_ent_off[gc + 1] - P.col_ent_off[gc];
      }
    }
    st.rem[s] = (unsigned short)indeg;
    st.ready[s] = 0.0;
#ifndef PS_DELTA_NOINDEG
    if (SNAP) w.dc->indeg[s] = (unsigned short)indeg;
#endif
    if (FULL) {
      int outd = 1;
      for (int i = T.op_out_off[o]; i < T.op_out_off[o + 1]; ++i) {
        int row = w.prow[T.op_out_pairs[i]] + k;
        outd += st.rowoff[row + 1] - st.rowoff[row];
      }
      st.rem[Tf + s] = (unsigned short)outd;
      st.ready[Tf + s] = 0.0;
#ifndef PS_DELTA_NOINDEG
      if (SNAP) w.dc->indeg[Tf + s] = (unsigned short)outd;
#endif
      int pm = T.op_param_mask[o];
      if (pm >= 0) {
        int g = w.gmap[o];
        int si = group_of2(P, o, g, k, pm);
        st.grp[s] = (unsigned char)si;
        atomicOr(&st.gmask[w.gbase[o] + si], 1ull << w.asg[T.op_slot_off[o] + k]);
        if (k < P.map_ngroups[g]) {
          int c = 2 * Tf + w.gbase[o] + k;
          st.rem[c] = (unsigned short)(P.map_size[g] / P.map_ngroups[g]);
          st.ready[c] = 0.0;
          if (SNAP) w.dc->indeg[c] = (unsigned short)(P.map_size[g] / P.map_ngroups[g]);
        }
      }
    }
  }
  __syncwarp();
  int n = 0;
  int nb = 0;                  // back ready set size
  bool refilled = false, pend_bslow = false;  // this round refilled / restarts as a combined slow round
  int last_fwd = 0;            // (SNAP) last round in which a forward operator task ran
  unsigned long long minb = ~0ull;  // lower bound of the back set's ready times (bits; ~0: empty)
  bool okc = true;
  int round = 0, next_snap = 0x7fffffff;  // (SNAP) round counter, round of the next snapshot
  PH_ADD(26, t_init);
  PH_T(t_rest);
  if (SNAP && w.dc->restore) {
    // resume: every counter some arrival had touched and that can still be
    // read (a task still waiting on predecessors; every ring: its slot keeps
    // the per-hop bytes once hop 0 is out) = new in-degree minus the arrivals at
    // the snapshot.  The changed op's counters start fresh; an op resized since
    // the snapshot had no arrivals then.  Tasks that ran or are in the ready set
    // are never counted again.
    const char *src = w.dc->restore;
    const SnapLay sl = snap_layout(P);
    const SnapHdr *hd = (const SnapHdr *)src;
    const int chg = w.dc->op, Tfo = hd->Tf, Go = hd->G;
    const unsigned short *rmo = (const unsigned short *)(src + sl.rm);
    const double *rdo = (const double *)(src + sl.rd);
    const unsigned short *ido = w.dc->indeg0 + (size_t)hd->epoch * w.dc->ep_stride;
    // the snapshot's layout, staged in the (still empty) ready-set area when it fits
    const int *fbo = (const int *)(src + sl.fb), *gbo = (const int *)(src + sl.gb);
    if ((size_t)(P.n_ops + 1) * 8 <= (size_t)w.rcap * sizeof(REnt)) {
      int *sf = (int *)w.rs, *sg = sf + (P.n_ops + 1);
      for (int j = lane; j <= P.n_ops; j += 32) { sf[j] = fbo[j]; if (FULL) sg[j] = gbo[j]; }
      fbo = sf; gbo = sg;
      __syncwarp();
    }
    const int nco = FULL ? 2 * Tfo : Tfo;
    for (int c8 = lane * 8; c8 < nco; c8 += 256) {  // 8 counters per lane per step
      uint4 rv = *(const uint4 *)(rmo + c8), iv = *(const uint4 *)(ido + c8);
      unsigned r2[4] = {rv.x, rv.y, rv.z, rv.w}, i2[4] = {iv.x, iv.y, iv.z, iv.w};
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        int os = c8 + u;
        unsigned re = (r2[u >> 1] >> ((u & 1) * 16)) & 0xffffu, ie = (i2[u >> 1] >> ((u & 1) * 16)) & 0xffffu;
        if (os < nco && re > 0 && re < ie) {
          int bw = os >= Tfo, x = bw ? os - Tfo : os;
          int o = upper_bound(fbo, P.n_ops + 1, x) - 1;
          int k = x - fbo[o];
          if (o != chg && k < w.fbase[o + 1] - w.fbase[o]) {
            int c = (bw ? Tf : 0) + w.fbase[o] + k;
            st.rem[c] -= (unsigned short)(ie - re);
            st.ready[c] = rdo[os];
          }
        }
      }
    }
    if (FULL)
      for (int og = lane; og < Go; og += 32) {
        int o = upper_bound(gbo, P.n_ops + 1, og) - 1;
        int si = og - gbo[o];
        if (o != chg && si < w.gbase[o + 1] - w.gbase[o]) {
          int c = 2 * Tf + w.gbase[o] + si, oc = 2 * Tfo + og;
          st.rem[c] -= (unsigned short)(ido[oc] - rmo[oc]);
          st.ready[c] = rdo[oc];
        }
      }
    __syncwarp();
    const double *qco = (const double *)(src + sl.qc);
    for (int q = lane; q < P.n_queues; q += 32) w.qclock[q] = qco[q];
    n = hd->n;
    const REnt *rso = (const REnt *)(src + sl.rs);
    const REnt *rbo = (const REnt *)(src + sl.rb);
    if (BACK) {
      nb = hd->nb;
      minb = hd->minb;
    }
    for (int i = lane; i < n + nb; i += 32) {
      REnt r = i < n ? rso[i] : rbo[i - n];
      if (i < n) w.rs[i] = r;
      else { w.bq[i - n] = r; w.bh[i - n] = r.h; }
      // a ready op task has no remaining count (the snapshots' "has run" test
      // reads it: ran = no remaining count and not in the ready set)
      unsigned kd = key_kind(r.k);
      if (kd == KIND_OP || (FULL && kd == KIND_OP_BWD))
        st.rem[(kd == KIND_OP ? 0 : Tf) + w.fbase[key_a(r.k)] + key_c(r.k)] = 0;
    }
    if (lane == 0) out.makespan = hd->makespan;
    round = hd->round;
    __syncwarp();
  } else {
    for (int base = 0; base < Tf; base += 32) {
      int s = base + lane;
      bool want = false;
      unsigned long long key = 0;
      int q = 0;
      double exe = 0.0;
      if (s < Tf && st.rem[s] == 0) {
        int o = upper_bound(w.fbase, P.n_ops + 1, s) - 1;
        key = pack_key(KIND_OP, o, 0, s - w.fbase[o], 0);
        op_attrs(P, T, w, KIND_OP, o, s - w.fbase[o], q, exe, SIMPLE);
        want = true;
      }
      okc &= push2<BACK>(want, 0.0, key, exe, q, n, nb, minb, P, w, lane);
    }
  }
  if (SNAP) {
    if (w.dc->snap && w.dc->restore_idx + 1 < w.dc->nsnap) next_snap = (w.dc->restore_idx + 1) * w.dc->stride;
    if (lane == 0) { w.dc->last = w.dc->restore_idx; w.dc->bad = 0; }
  }
  __syncwarp();
  PH_ADD(27, t_rest);
  PH_ADD(1, t_init);
  if (!okc) { out.status = PS_STATUS_CAPACITY; return out; }
  while (n > 0 || (BACK && nb > 0)) {
    if (SNAP && round == next_snap) {
      // (a state with a back set is not snapshotted: the index is marked unusable)
      PH_CNT(23, 1);
      PH_CNT(24, nb > P.snap_b ? 1 : 0);
      PH_CNT(25, n > P.cap ? 1 : 0);
      PH_T(t_snap);
      snap_write(P, w, st, n, nb, minb, round, round / w.dc->stride, out.makespan, FULL, lane);
      PH_ADD(28, t_snap);
      next_snap = round / w.dc->stride + 1 < w.dc->nsnap ? round + w.dc->stride : 0x7fffffff;
    }
    PH_T(t_sel);
    TC(0);
    PH_CNT(11, 1);
    PH_CNT(12, n);
    bool mine = false;
    int nw = 0;
    // (the winner's task: read only on winner lanes, or shuffled from them)
    unsigned long long mykey;
    double myready, myexe;
    int myq;
    int myrank = 0, maxrank = 0;  // position among this round's members on the same queue
    double end, mystart;  // set on winner lanes
    bool ran = false;  // fast path: rank-0 members already ran (their queue clock is the one read this round)
    // Medium path (33..64 ready tasks, two per lane): when the round's members
    // are at most 32, they are staged at [64, 64 + members) and the others
    // compacted to [0, rest); the fast path below then runs the members alone.
    // Two-level ready set.  With a back set, the round's members must also be
    // ready before every back entry (minb bounds them below), and the front
    // set alone must determine LB.  Each selection path below computes the
    // front set's LB; if the back set could hold a member or an earlier bound
    // (minb < that LB) its entries ready before that LB move to the front set
    // and the round restarts (at most one refill per round) -- or, if they do
    // not fit, the round restarts over both sets in the back set (bslow).  An
    // empty front set refills against the back set's own LB here.
    bool bslow = false;
    PH_T(t_rf);
    if (BACK && nb > 0 && (n == 0 || pend_bslow)) {
      bool moved = false;
      if (!pend_bslow) {
        unsigned long long X = back_lb(w, nb, lane);
        if (X == INF_BITS) X = ~0ull;  // no entry with successors: every entry is a member
        moved = back_refill(w, n, nb, minb, X, lane);
        refilled = true;
      }
      if (!moved) {
        if (nb + n > w.bcap) { out.status = PS_STATUS_CAPACITY; return out; }
        for (int i = lane; i < n; i += 32) { REnt r = w.rs[i]; w.bq[nb + i] = r; w.bh[nb + i] = r.h; }
        nb += n;
        n = 0;
        bslow = true;
        __syncwarp();
      }
      pend_bslow = false;
    }
    PH_ADD(33, t_rf);
    int sel_base = 0, sel_n = bslow ? 33 : n, rest = 0;
    bool forced = false;
    if (!bslow && n > 32 && n <= 64 && n + 32 <= w.rcap) {
      PH_CNT(22, 1);
      bool vA = true, vB = lane + 32 < n;
      unsigned long long hA = w.rs[lane].h, kA = w.rs[lane].k, hB = vB ? w.rs[lane + 32].h : ~0ull,
                         kB = vB ? w.rs[lane + 32].k : ~0ull;
      double eA = w.rs[lane].e, eB = vB ? w.rs[lane + 32].e : 0.0;
      int qA = w.rs[lane].q, qB = vB ? w.rs[lane + 32].q : 0;
      double rA = __longlong_as_double((long long)hA), rB = __longlong_as_double((long long)hB);
      double cA = w.qclock[qA & Q_MASK], cB = vB ? w.qclock[qB & Q_MASK] : 0.0;
      double lA = (rA < cA ? cA : rA) + eA, lB = (rB < cB ? cB : rB) + eB;
      unsigned long long bA = !(qA & Q_SINK) ? (unsigned long long)__double_as_longlong(lA) : INF_BITS;
      unsigned long long bB = (vB && !(qB & Q_SINK)) ? (unsigned long long)__double_as_longlong(lB) : INF_BITS;
      const unsigned long long lb2b = warp_min64(bA < bB ? bA : bB, lane);
      BACK_CHECK(lb2b);
      double LB2 = __longlong_as_double((long long)lb2b);
      bool mA = vA && rA < LB2 && (!BACK || hA < minb), mB = vB && rB < LB2 && (!BACK || hB < minb);
      unsigned gA = __ballot_sync(FULLMASK, mA), gB = __ballot_sync(FULLMASK, mB);
      int nm = __popc(gA) + __popc(gB);
      if (nm > 0 && nm <= 32) {
        unsigned lt = (1u << lane) - 1u;
        unsigned xA = __ballot_sync(FULLMASK, vA && !mA), xB = __ballot_sync(FULLMASK, vB && !mB);
        int pA = mA ? 64 + __popc(gA & lt) : __popc(xA & lt);
        int pB = mB ? 64 + __popc(gA) + __popc(gB & lt) : __popc(xA) + __popc(xB & lt);
        __syncwarp();
        w.rs[pA].h = hA; w.rs[pA].k = kA; w.rs[pA].e = eA; w.rs[pA].q = qA;
        if (vB) { w.rs[pB].h = hB; w.rs[pB].k = kB; w.rs[pB].e = eB; w.rs[pB].q = qB; }
        __syncwarp();
        sel_base = 64; sel_n = nm; rest = n - nm; forced = true;
      }
    }
    if (sel_n <= 32) {
      // ---- fast path: entry `lane` lives in this lane's registers for the round
      bool valid = lane < sel_n;
      int ix = sel_base + lane;
      REnt re = w.rs[valid ? ix : 0];  // unconditional load (entry 0 always exists), then mask
      unsigned long long h = valid ? re.h : ~0ull, k = valid ? re.k : ~0ull;
      double e = valid ? re.e : 0.0;
      int qr = valid ? re.q : 0;
      int q = qr & Q_MASK;
      double r = __longlong_as_double((long long)h);
      // LB = min over tasks with successors of max(ready, clock) + exe: no task
      // outside the ready set can become ready before LB (clocks only grow)
      double ck = valid ? w.qclock[q] : 0.0;
      double el = (r < ck ? ck : r) + e;
      TC(1);
      unsigned long long lbb = (valid && !(qr & Q_SINK)) ? (unsigned long long)__double_as_longlong(el) : INF_BITS;
      const unsigned long long lbw = warp_min64(lbb, lane);
      if (!forced) BACK_CHECK(lbw);
      double LB = __longlong_as_double((long long)lbw);
      PH_ADD(5, t_sel);
      TC(2);
      PH_T(t_cl);
      bool member = valid && (forced || (r < LB && (!BACK || h < minb)));
      if (!__any_sync(FULLMASK, member)) {
        // degenerate (zero or absorbed exe): the global minimum alone
        int wl = warp_argmin128(h, k, lane);
        member = lane == wl;
      }
      // every member runs this round; members sharing a queue run in (ready,
      // origin) order.  A 64-bin queue hash rules out shared queues in the
      // common case; otherwise the members of each shared queue rank themselves.
      TC(3);
      bool win = member;
      unsigned wb = __ballot_sync(FULLMASK, win);
      nw = __popc(wb);
      unsigned hlo = __reduce_or_sync(FULLMASK, (member && !(q & 32)) ? 1u << (q & 31) : 0u);
      unsigned hhi = __reduce_or_sync(FULLMASK, (member && (q & 32)) ? 1u << (q & 31) : 0u);
      TC(4);
      if (__popc(hlo) + __popc(hhi) < nw) {
        unsigned gm = __match_any_sync(FULLMASK, member ? q : (0x40000000 | lane));
        unsigned others = member ? (gm & ~(1u << lane)) : 0u;
        int cnt = __popc(others);
        maxrank = (int)__reduce_max_sync(FULLMASK, (unsigned)cnt);
        for (int j = 0; j < maxrank; ++j) {
          int src = others ? __ffs(others) - 1 : lane;
          others &= others - 1;
          unsigned long long hj = __shfl_sync(FULLMASK, h, src), kj = __shfl_sync(FULLMASK, k, src);
          if (j < cnt && (hj < h || (hj == h && kj < k))) ++myrank;
        }
      }
      TC(5);
      if (win && dirty) { w.qbest[q] = ~0ull; w.qready[q] = ~0ull; }  // bid left by a capped slow round
      bool keep = valid && !win;
      unsigned kb = __ballot_sync(FULLMASK, keep);
      if (keep) {
        int pos = __popc(kb & ((1u << lane) - 1u));
        REnt r2;
        r2.h = h; r2.k = k; r2.e = e; r2.q = qr; r2.pad = 0;
        w.rs[pos] = r2;
      }
      n = forced ? rest : __popc(kb);
      mine = win;
      if (win) w.wlane[__popc(wb & ((1u << lane) - 1u))] = lane;
      mykey = k; myready = r; myexe = e; myq = q;
      if (win && myrank == 0) {
        // the first member on its queue starts at max(ready, clock) with the
        // clock read above: end = el (simulate.py:92-94)
        mystart = r < ck ? ck : r;
        end = el;
        w.qclock[q] = end;
      }
      ran = true;
      TC(6);
      PH_ADD(15, t_cl);
    } else {
      // ---- slow path: the front set (more than 64 entries, or more than 32
      // members), or -- bslow -- front and back sets together in the back set
      REnt *S = bslow ? w.bq : w.rs;
      int *SM = bslow ? w.bmem : w.mem;
      int sn = bslow ? nb : n;
      const unsigned long long mbk = (!BACK || bslow) ? ~0ull : minb;  // members: ready below the back set too
      PH_T(t_slow);
      PH_CNT(16, 1);
      PH_CNT(17, sn);
      if (lane == 0) w.flags[0] = 1;
      dirty = true;
      // ---- scan 1: minimum key and LB = min(ready + exe)
      unsigned long long bh = ~0ull, bl = ~0ull, lb = INF_BITS;
      for (int i = lane; i < sn; i += 32) {
        unsigned long long h = S[i].h, l = S[i].k;
        if (h < bh || (h == bh && l < bl)) { bh = h; bl = l; }
        int qr = S[i].q;
        if (!(qr & Q_SINK)) {
          double r0 = __longlong_as_double((long long)h), ck = w.qclock[qr & Q_MASK];
          double e = (r0 < ck ? ck : r0) + S[i].e;
          unsigned long long eb = (unsigned long long)__double_as_longlong(e);
          if (eb < lb) lb = eb;
        }
      }
      int wl = warp_argmin128(bh, bl, lane);
      unsigned long long minkey = __shfl_sync(FULLMASK, bl, wl);
      const unsigned long long minready = __shfl_sync(FULLMASK, bh, wl);
      const unsigned long long lbs = warp_min64(lb, lane);
      if (!bslow) BACK_CHECK(lbs);
      double LB = __longlong_as_double((long long)lbs);
      // ---- scan 2: members (ready < LB, or the global minimum) -> member list,
      // and each bids its ready time for its queue
      int nm = 0;
      for (int base = 0; base < sn; base += 32) {
        int i = base + lane;
        bool mem = false;
        if (i < sn) {
          unsigned long long h2 = S[i].h;
          mem = (__longlong_as_double((long long)h2) < LB && h2 < mbk) || S[i].k == minkey;
          if (mem) atomicMin(&w.qready[S[i].q & Q_MASK], h2);
        }
        unsigned bm = __ballot_sync(FULLMASK, mem);
        if (mem) SM[nm + __popc(bm & ((1u << lane) - 1u))] = i;
        nm += __popc(bm);
      }
      __syncwarp();
      // ---- members tied on their queue's ready time bid their origin key
      for (int j = lane; j < nm; j += 32) {
        int i = SM[j];
        int q2 = S[i].q & Q_MASK;
        if (w.qready[q2] == S[i].h) atomicMin(&w.qbest[q2], S[i].k);
      }
      __syncwarp();
      // ---- winners: each queue's minimum (ready, origin); lane k holds winner k
      int mypos = -1;
      for (int base = 0; base < nm && nw < 32; base += 32) {
        int j = base + lane;
        bool win = false;
        int i = 0;
        if (j < nm) {
          i = SM[j];
          int q2 = S[i].q & Q_MASK;
          win = w.qbest[q2] == S[i].k && w.qready[q2] == S[i].h;
        }
        unsigned bm = __ballot_sync(FULLMASK, win);
        // lane nw + r takes the r-th winner of this chunk (winners past 32 wait)
        int r = lane - nw;
        int src = (r >= 0 && r < __popc(bm)) ? (int)__fns(bm, 0, r + 1) : 0;
        int i2 = __shfl_sync(FULLMASK, i, src);
        if (r >= 0 && r < __popc(bm)) mypos = i2;
        nw = min(32, nw + __popc(bm));
      }
      bool mine0 = lane < nw;
      if (mine0) {
        mykey = S[mypos].k;
        myready = __longlong_as_double((long long)S[mypos].h);
        myexe = S[mypos].e;
        myq = S[mypos].q & Q_MASK;
      }
      __syncwarp();
      if (mine0) { w.qbest[myq] = ~0ull; w.qready[myq] = ~0ull; S[mypos].h = ~0ull; }
      __syncwarp();
      // ---- remove the winners: refill holes below sn-nw with survivors from the tail
      {
        int tailpos = sn - nw + lane;
        bool survivor = lane < nw && S[tailpos].h != ~0ull;
        unsigned sm = __ballot_sync(FULLMASK, survivor);
        bool head_hole = mine0 && mypos < sn - nw;
        unsigned hm = __ballot_sync(FULLMASK, head_hole);
        int hrank = __popc(hm & ((1u << lane) - 1u));
        int src = -1;
        if (head_hole) src = sn - nw + (int)__fns(sm, 0, hrank + 1);
        unsigned long long h2 = 0, k2 = 0;
        double e2 = 0.0;
        int q2 = 0;
        if (head_hole) { h2 = S[src].h; k2 = S[src].k; e2 = S[src].e; q2 = S[src].q; }
        __syncwarp();
        if (head_hole) { S[mypos].h = h2; S[mypos].k = k2; S[mypos].e = e2; S[mypos].q = q2; }
        sn -= nw;
        __syncwarp();
      }
      mine = lane < nw;
      w.wlane[lane] = lane;
      if (bslow) {  // (minb: the earliest ready time before the round, a lower bound)
        nb = sn;
        minb = minready;
        for (int i = lane; i < nb; i += 32) w.bh[i] = w.bq[i].h;  // the keys of the rewritten back set
        __syncwarp();
      }
      else n = sn;
      PH_ADD(19, t_slow);
      PH_CNT(18, nw);
    }
    PH_T(t_run);
    // ---- run the winners: per queue in (ready, origin) order
#pragma unroll 1
    for (int lv = ran ? 1 : 0; lv <= maxrank; ++lv) {
      if (ran) __syncwarp();
      if (mine && myrank == lv) {
        double clk = w.qclock[myq];
        double start = myready < clk ? clk : myready;
        mystart = start;
        end = start + myexe;
        w.qclock[myq] = end;
      }
    }
    // (full-iteration snapshots only need to cover the forward part: every
    // resume point lies before the changed op's first forward task)
    if (SNAP && __any_sync(FULLMASK, mine && key_kind(mykey) == KIND_OP)) last_fwd = round;
    if (mine) {
      if (end > out.makespan) out.makespan = end;
      if ((M & SIM_OPMIN) && key_kind(mykey) == KIND_OP)
        atomicMin((unsigned long long *)&w.opmin[key_a(mykey)], (unsigned long long)__double_as_longlong(end));
    }
    int myrec = -1;
    if ((M & SIM_TRACE) && mine) {
      myrec = atomicAdd(w.tr->n_tasks, 1);
      if (myrec < w.tr->task_cap) {
        ps_trace_task rec;
        rec.key = mykey; rec.queue = myq; rec.aux = 0; rec.exe = myexe;
        rec.nbytes = trace_nbytes(P, T, w, st, mykey);
        rec.ready = myready; rec.start = mystart; rec.end = end;
        w.tr->tasks[myrec] = rec;
      }
    }
    PH_ADD(20, t_run);
    PH_ADD(2, t_sel);
    TC(7);
    PH_CNT(13, nw);
    PH_T(t_succ);
    // ---- successors: lane groups of G per winner, random access into each list.
    // A winner's successors are its overlap-list entries (forward op: row c of
    // each out-pair's current combo; backward op: column c of each in-pair's)
    // plus at most one fixed successor, taken last: forward -> its backward
    // task, backward -> its ring's hop 0, transfer -> the task it feeds, ring
    // hop -> the next hop.  Entries of both directions go through one code path
    // (taskgraph.py:199-221: same device -> dependency, else a transfer).
    int lg = 31 - __clz(nw);
    if ((1 << lg) < nw) ++lg;
    int G = 32 >> lg, lgG = 5 - lg;
    int wi = lane >> lgG, j0 = lane & (G - 1);
    bool act_lane = wi < nw;
    __syncwarp();
    int srcl = act_lane ? w.wlane[wi] : 0;
    unsigned long long wkey = __shfl_sync(FULLMASK, mykey, srcl);
    double wend = __shfl_sync(FULLMASK, end, srcl);
    int wrec = __shfl_sync(FULLMASK, myrec, srcl);
    int wq = __shfl_sync(FULLMASK, myq, srcl);  // an operator task's queue is its device
    unsigned kind = key_kind(wkey), a = key_a(wkey), b = key_b(wkey), c = key_c(wkey), d = key_d(wkey);
    if (MODE == 0) kind = kind == KIND_OP ? KIND_OP : KIND_EDGE;  // forward mode: no other kinds
    const bool fwd = kind == KIND_OP;
    TC(10);
    const int *poff = fwd ? T.op_out_off : T.op_in_off;
    const int *plist = fwd ? T.op_out_pairs : T.op_in_pairs;
    const int *pbase = fwd ? w.prow : w.pcol;
    const int *eoff = fwd ? st.rowoff : st.coloff;
    const Ent32 *etab = fwd ? ent : cent;
    int wdev = 0, L = 0;
    int fe = -1, fp = 0;  // this lane's first list entry (index j0) and its pair
    // fixed successor: fact 1 = arrive at counter fslot, 2 = push task fkey directly
    // (the f* values are only read where fact != 0: left uninitialised, no moves)
    int fact = 0, fslot, fq, fea = -1, feb = -1;
    unsigned long long fkey;
    double fexe;
    bool ferr = false;
    if (act_lane) {
      if (fwd || kind == KIND_OP_BWD) {
        wdev = wq;
        int r0 = j0;
        int i0 = poff[a], np = poff[a + 1] - i0;
        // the first four pairs: loads issued together (three dependent steps in all)
        int pp[4], ix[4], ea0[4], ea1[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) pp[j] = j < np ? plist[i0 + j] : 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) ix[j] = j < np ? pbase[pp[j]] + c : 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          ea0[j] = j < np ? eoff[ix[j]] : 0;
          ea1[j] = j < np ? eoff[ix[j] + 1] : 0;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          int len = ea1[j] - ea0[j];
          if (fe < 0 && r0 >= 0 && r0 < len) { fe = ea0[j] + r0; fp = pp[j]; }
          r0 -= len;
          L += len;
        }
        for (int i = i0 + 4; i < i0 + np; ++i) {
          int p = plist[i];
          int x = pbase[p] + c;
          int e0 = eoff[x], len = eoff[x + 1] - e0;
          if (fe < 0 && r0 >= 0 && r0 < len) { fe = e0 + r0; fp = p; }
          r0 -= len;
          L += len;
        }
        if (!fwd && T.op_param_mask[a] >= 0) {
          int si = st.grp[w.fbase[a] + c];
          if (__popcll((long long)st.gmask[w.gbase[a] + si]) >= 2) {
            fact = 1; fslot = 2 * Tf + w.gbase[a] + si; fkey = pack_key(KIND_SYNC, a, si, 0, 0);
          }
        }
      }
      if ((fwd && FULL) || kind == KIND_EDGE || kind == KIND_EDGE_BWD) {
        // forward -> its backward task; transfer -> the task it feeds
        bool tf = kind == KIND_EDGE;
        int xo = tf ? (int)b : (int)a, xb = tf ? (int)d : (int)c;
        fact = 1;
        fslot = (tf ? 0 : Tf) + w.fbase[xo] + xb;
        fkey = pack_key(tf ? KIND_OP : KIND_OP_BWD, xo, 0, xb, 0);
      } else if (kind == KIND_SYNC) {  // ring hop c -> c + 1 (none after the last)
        int r = __popcll((long long)st.gmask[w.gbase[a] + b]);
        if ((int)c + 1 < 2 * (r - 1)) {
          fact = 2; fkey = pack_key(KIND_SYNC, a, b, c + 1, 0);
          if (!sync_attrs(P, T, w, st, a, b, c + 1, fq, fexe, fea, feb, SIMPLE)) ferr = true;
        }
      }
    }
    Ent32 fen;
    // (read only by lanes with an entry: fe >= 0 whenever j0 < L)
    TC(11);
    if (fe >= 0) fen = etab[fe];
    int Lt = L + (fact ? 1 : 0);
    int iters = (Lt + G - 1) >> lgG;
    iters = (int)__reduce_max_sync(FULLMASK, (unsigned)(act_lane ? iters : 0));
    PH_ADD(3, t_succ);
    TC(8);
    PH_CNT(14, iters);
    PH_T(t_it);
    for (int t = 0; t < iters; ++t) {
      int idx = j0 + t * G;
      int act = 0;  // 1 arrive at counter `slot`, 2 push task `skey` directly
      int slot;               // read only when act == 1
      unsigned long long skey;  // stored only for lanes that push
      int pq;
      double pexe;
      bool err = false;
      int ea = -1, eb = -1;
      if (act_lane && idx < L) {
        Ent32 en = fen;
        int p = fp;
        if (t > 0) {
          int r = idx;
          for (int i = poff[a]; i < poff[a + 1]; ++i) {
            p = plist[i];
            int ix = pbase[p] + c;
            int e0 = eoff[ix], len = eoff[ix + 1] - e0;
            if (r < len) { en = etab[e0 + r]; break; }
            r -= len;
          }
        }
        // the entry's other end: forward -> consumer block l, backward -> producer block k
        int kk = en.kl & 0xffff, l = en.kl >> 16;
        int xo = fwd ? T.pair_dst[p] : T.pair_src[p];
        int xb = fwd ? l : kk;
        int xdev = w.asg[en.slot];
        if (xdev == wdev) {
          act = 1;
          slot = (fwd ? 0 : Tf) + w.fbase[xo] + xb;
          skey = pack_key(fwd ? KIND_OP : KIND_OP_BWD, xo, 0, xb, 0);
        } else {
          // transfer (producer op, consumer op, producer block, consumer block)
          act = 2;
          int so = fwd ? (int)a : xo, dop = fwd ? xo : (int)a, sb = fwd ? (int)c : kk, db = fwd ? l : (int)c;
          int sdv = fwd ? wdev : xdev, ddv = fwd ? xdev : wdev;
          skey = pack_key(fwd ? KIND_EDGE : KIND_EDGE_BWD, so, dop, sb, db);
          if (!link_attrs_ent(P, T, sdv, ddv, en, pq, pexe, SIMPLE)) { err = true; ea = sdv; eb = ddv; }
        }
      } else if (act_lane && idx == L && fact) {
        act = fact; slot = fslot; skey = fkey; pq = fq; pexe = fexe; err = ferr; ea = fea; eb = feb;
      }
      if (t == 0) TC(12);
      if ((M & SIM_TRACE) && act != 0 && wrec >= 0) {
        int e_ = atomicAdd(w.tr->n_edges, 1);
        if (e_ < w.tr->edge_cap) { w.tr->edge_pred[e_] = wrec; w.tr->edge_succ[e_] = skey; }
      }
      // arrivals.  The u16 counter is decremented through the 32-bit word that
      // holds it (no borrow: it stops at zero).  When no two lanes arrive at one
      // counter in this iteration (a 64-bin hash says so), each arriver folds
      // its end into the ready time itself: the last one keeps the maximum,
      // the others store it.  Otherwise every max lands (atomically) before
      // any count is taken, ordered by the warp barrier.
      bool arr = act == 1;
      unsigned alo = __reduce_or_sync(FULLMASK, (arr && !(slot & 32)) ? 1u << (slot & 31) : 0u);
      unsigned ahi = __reduce_or_sync(FULLMASK, (arr && (slot & 32)) ? 1u << (slot & 31) : 0u);
      bool shared_slot = __popc(alo) + __popc(ahi) < __popc(__ballot_sync(FULLMASK, arr));
      if (shared_slot) {
        if (arr) atomicMax((unsigned long long *)&st.ready[slot], (unsigned long long)__double_as_longlong(wend));
        __syncwarp();
      }
      if (t == 0) TC(13);
      bool want = false;
      double pready = 0.0;
      if (arr) {
        unsigned sh = (slot & 1) * 16;
        unsigned old = atomicSub((unsigned *)(st.rem + (slot & ~1)), 1u << sh);
        bool last = ((old >> sh) & 0xffffu) == 1u;
        double cur = st.ready[slot];
        if (!shared_slot) {
          if (wend > cur) cur = wend;
          if (!last) st.ready[slot] = cur;
        }
        if (last) {
          want = true;
          pready = cur;
          unsigned sk = MODE == 0 ? (unsigned)KIND_OP : key_kind(skey);  // forward: arrivals feed forward ops
          if (sk == KIND_SYNC) {
            if (!sync_attrs(P, T, w, st, key_a(skey), key_b(skey), 0, pq, pexe, ea, eb, SIMPLE)) err = true;
          } else {
            op_attrs(P, T, w, sk, key_a(skey), key_c(skey), pq, pexe, SIMPLE);
          }
        }
      } else if (act == 2) {
        want = true;
        pready = wend;
      }
      if (t == 0) TC(14);
      if (!SIMPLE) {  // (a full mesh has a route for every transfer)
        unsigned bad = __ballot_sync(FULLMASK, err);
        if (bad) {
          int s3 = __ffs(bad) - 1;
          out.status = PS_STATUS_NO_ROUTE;
          out.err_a = __shfl_sync(FULLMASK, ea, s3);
          out.err_b = __shfl_sync(FULLMASK, eb, s3);
          return out;
        }
      }
      if (!push2<BACK>(want, pready, skey, pexe, pq, n, nb, minb, P, w, lane)) { out.status = PS_STATUS_CAPACITY; return out; }
      __syncwarp();
    }
    PH_ADD(4, t_it);
    TC(9);
#ifdef PS_TCYC
    ++tc_r;
#endif
    if (SNAP) ++round;
    refilled = false;
    // keep the front set small: past 64 entries, the later ones move to the back set
    if (BACK && n > 64 && w.bcap) {
      PH_T(t_trim);
      // threshold: a histogram of the front's ready times where the tables sit on
      // chip (NMT-40 +8 %, random-1k +5 %), the 33rd smallest by a bitonic sort in
      // the all-global layout (random-10k: the histogram's smaller fronts refill
      // more often, -8 %); PS_TRIM_HIST=0/1 at build time forces one
#ifdef PS_TRIM_HIST
      const bool by_hist = PS_TRIM_HIST != 0;
#else
      const bool by_hist = trim_hist;
#endif
      if (!front_trim(w, n, nb, minb, lane, by_hist)) { out.status = PS_STATUS_CAPACITY; return out; }
      PH_ADD(30, t_trim);
      PH_CNT(31, 1);
    }
    // (no barrier here: every path above ends with one after its last shared store)
  }
  if (SNAP && lane == 0) { w.dc->rounds = round; w.dc->rounds_fwd = last_fwd + 1; }
  // makespan: max over lanes
  unsigned long long mb = (unsigned long long)__double_as_longlong(out.makespan);
  unsigned hi = __reduce_max_sync(FULLMASK, (unsigned)(mb >> 32));
  unsigned lo = __reduce_max_sync(FULLMASK, (unsigned)(mb >> 32) == hi ? (unsigned)mb : 0u);
  out.makespan = __longlong_as_double((long long)(((unsigned long long)hi << 32) | lo));
  return out;
}

template <int S>
__global__ void PS_BOUNDS(S)
k_simulate_batch(DevProb P, Lay lay, const int *__restrict__ maps, const unsigned char *__restrict__ asgs, int n,
                 double *makespan, int *status, char *gscratch, double *opmin, int *next) {
  extern __shared__ __align__(16) char smem[];
  int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  int gw = blockIdx.x * wpb + wib;
  char *gs = gscratch + (size_t)gw * gslice_bytes(P, lay);
  Tab T;
  W2 w;
  kernel_layout(P, lay, smem, gs, wib, T, w);
  __syncthreads();
  bind_bids(P, gs, w);
  if (lane == 0) w.flags[0] = 1;  // the global bid arrays start uninitialised
  __syncwarp();
  // candidates are taken from a work queue: a slow one (e.g. a wide data-parallel
  // strategy) holds up only its own warp
  for (int cand = __shfl_sync(FULLMASK, lane == 0 ? atomicAdd(next, 1) : 0, 0); cand < n;
       cand = __shfl_sync(FULLMASK, lane == 0 ? atomicAdd(next, 1) : 0, 0)) {
    const int *m = maps + (size_t)cand * P.n_ops;
    const unsigned char *a = asgs + (size_t)cand * P.n_slots;
    for (int i = lane; i < P.n_ops; i += 32) w.mapl[i] = m[i];
    if (lay.asg_global) w.asg = const_cast<unsigned char *>(a);
    else
      for (int i = lane; i < P.n_slots; i += 32) w.asg[i] = a[i];
    if (opmin) {
      w.opmin = opmin + (size_t)cand * P.n_ops;
      for (int i = lane; i < P.n_ops; i += 32) w.opmin[i] = __longlong_as_double(0x7ff0000000000000ll);
    }
    __syncwarp();
    SimOut o = opmin ? simulate_any<SIM_OPMIN | S>(P, T, w, lay, gs, lane) : simulate_any<S>(P, T, w, lay, gs, lane);
    if (lane == 0) {
      makespan[cand] = o.status == PS_STATUS_OK ? o.makespan : -1.0;
      status[cand] = o.status;
    }
    __syncwarp();
  }
}

__global__ void __launch_bounds__(32)
k_simulate_trace(DevProb P, Lay lay, const int *map, const unsigned char *asg, char *gscratch, TraceSink tr,
                 double *makespan, int *status, int *err) {
  extern __shared__ __align__(16) char smem[];
  int lane = threadIdx.x & 31;
  Tab T;
  W2 w;
  kernel_layout(P, lay, smem, gscratch, 0, T, w);
  __syncthreads();
  bind_bids(P, gscratch, w);
  if (lane == 0) w.flags[0] = 1;
  for (int i = lane; i < P.n_ops; i += 32) w.mapl[i] = map[i];
  if (lay.asg_global) w.asg = const_cast<unsigned char *>(asg);
  else
    for (int i = lane; i < P.n_slots; i += 32) w.asg[i] = asg[i];
  w.tr = &tr;
  __syncwarp();
  SimOut o = warp_simulate2<SIM_TRACE>(P, T, w, lay, gscratch, lane);
  if (o.status == PS_STATUS_CAPACITY) {  // wide ready set: rerun in global memory, fresh trace
    if (lane == 0) { *tr.n_tasks = 0; *tr.n_edges = 0; }
    __syncwarp();
    o = warp_simulate2<SIM_TRACE>(P, T, with_global_ready_set(P, gscratch, w), lay, gscratch, lane);
  }
  if (lane == 0) {
    *makespan = o.makespan;
    *status = o.status;
    err[0] = o.err_a;
    err[1] = o.err_b;
  }
}

__global__ void __launch_bounds__(32)
k_simulate_explicit(int n_tasks, int n_queues, const int *__restrict__ queue, const double *__restrict__ exe,
                    const unsigned long long *__restrict__ rank, const int *__restrict__ succ_off,
                    const int *__restrict__ succ, const int *__restrict__ indeg, double *ready, double *start,
                    double *end, int *order, int *rem, double *qclock, unsigned long long *rhi,
                    unsigned long long *rlo, int *raux, int *status, double *makespan) {
  int lane = threadIdx.x;
  for (int q = lane; q < n_queues; q += 32) qclock[q] = 0.0;
  WarpSmem w;
  w.qclock = qclock; w.rhi = rhi; w.rlo = rlo; w.raux = raux;
  int n = 0;
  for (int base = 0; base < n_tasks; base += 32) {
    int t = base + lane;
    bool want = false;
    if (t < n_tasks) {
      rem[t] = indeg[t];
      ready[t] = 0.0;
      want = indeg[t] == 0;
    }
    warp_push(want, 0.0, t < n_tasks ? rank[t] : 0ull, t, n, n_tasks, w, lane);
  }
  __syncwarp();
  double mk = 0.0;
  int popped = 0;
  while (n > 0) {
    unsigned long long bh = ~0ull, bl = ~0ull;
    int bp = 0;
    for (int i = lane; i < n; i += 32) {
      unsigned long long h = rhi[i], l = rlo[i];
      if (h < bh || (h == bh && l < bl)) { bh = h; bl = l; bp = i; }
    }
    for (int off = 16; off > 0; off >>= 1) {
      unsigned long long oh = __shfl_xor_sync(FULLMASK, bh, off), ol = __shfl_xor_sync(FULLMASK, bl, off);
      int op = __shfl_xor_sync(FULLMASK, bp, off);
      if (oh < bh || (oh == bh && ol < bl)) { bh = oh; bl = ol; bp = op; }
    }
    int t = raux[bp];
    double r = __longlong_as_double((long long)bh);
    __syncwarp();
    if (lane == 0) { rhi[bp] = rhi[n - 1]; rlo[bp] = rlo[n - 1]; raux[bp] = raux[n - 1]; }
    --n;
    __syncwarp();
    int q = queue[t];
    double clk = qclock[q];
    double st = r < clk ? clk : r;
    double en = st + exe[t];
    __syncwarp();
    if (lane == 0) { qclock[q] = en; ready[t] = r; start[t] = st; end[t] = en; order[popped] = t; }
    ++popped;
    if (en > mk) mk = en;
    for (int jb = succ_off[t]; jb < succ_off[t + 1]; jb += 32) {
      int j = jb + lane;
      bool want = false;
      double sr = 0.0;
      int v = 0;
      if (j < succ_off[t + 1]) {
        v = succ[j];
        sr = ready[v];
        if (en > sr) { sr = en; ready[v] = sr; }
        want = --rem[v] == 0;
      }
      warp_push(want, sr, want ? rank[v] : 0ull, v, n, n_tasks, w, lane);
    }
    __syncwarp();
  }
  if (lane == 0) {
    *status = popped == n_tasks ? PS_STATUS_OK : 3;
    *makespan = mk;
  }
}

// ---------------------------------------------------------------- MCMC
struct ChainState {
  double cost, best, beta, initial;
  long long proposals, accepted;
  unsigned long long key, ctr;  // Philox
  int bpos, mti;                // Philox buffer position / MT index
  int status, err_a, err_b, started;
  int last_op, pad_;
};

__device__ __forceinline__ void philox_block(unsigned long long ctr, unsigned long long key, unsigned out[4]) {
  unsigned c0 = (unsigned)ctr, c1 = (unsigned)(ctr >> 32), c2 = 0u, c3 = 0u;
  unsigned k0 = (unsigned)key, k1 = (unsigned)(key >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    unsigned hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    unsigned hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    c0 = hi1 ^ c1 ^ k0; c1 = lo1; c2 = hi0 ^ c3 ^ k1; c3 = lo0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

// Warp-uniform RNG: every lane holds the same state and gets the same word.
struct WarpRng {
  int mode;
  unsigned long long key, ctr;
  unsigned buf[4];
  int bpos;
  unsigned *mt;  // global [624]
  int mti;
  int lane;

  __device__ unsigned next() {
    if (mode == PS_RNG_PHILOX) {
      if (bpos == 4) { philox_block(ctr++, key, buf); bpos = 0; }
      return buf[bpos++];
    }
    if (mti >= 624) twist();
    unsigned y = mt[mti++];
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= y >> 18;
    return y;
  }
  // MT19937 regeneration in three dependency-free phases
  __device__ void twist_range(int lo, int hi) {
    for (int base = lo; base < hi; base += 32) {
      int i = base + lane;
      unsigned nv = 0;
      if (i < hi) {
        unsigned y = (mt[i] & 0x80000000u) | (mt[i + 1 < 624 ? i + 1 : 0] & 0x7fffffffu);
        int j = i + 397 < 624 ? i + 397 : i + 397 - 624;
        nv = mt[j] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
      }
      __syncwarp();
      if (i < hi) mt[i] = nv;
      __syncwarp();
    }
  }
  __device__ void twist() {
    twist_range(0, 227);
    twist_range(227, 454);
    twist_range(454, 623);
    twist_range(623, 624);
    mti = 0;
  }
  __device__ unsigned below(unsigned n) {
    int k = 32 - __clz(n);
    unsigned v = next() >> (32 - k);
    while (v >= n) v = next() >> (32 - k);
    return v;
  }
  __device__ double random() {
    unsigned a = next() >> 5, b = next() >> 6;
    return ((double)a * 67108864.0 + (double)b) * (1.0 / 9007199254740992.0);
  }
};

// Per-chain delta buffers of an MCMC handle (global memory)
struct DeltaBufs {
  ChainDelta *cd;          // [n]
  char *snaps;             // [n][nsnap][2] snapshot slots
  int *frb;                // [n][2 copies][forward, backward][n_ops] first rounds
  unsigned short *indeg;   // [n][nsnap + 1 epochs][snap_counters_pad] in-degrees per simulation
  unsigned long long snap_bytes;
  int nsnap;
  int exp;                 // experiments (PS_DELTA_EXP): 1 no snapshots, 2 snapshots but no resume
  int *dbg;                // PS_DELTA_TRACE: [n][dbg_cap][8] per proposal (o, j, R, rounds, nvalid, stride, ...)
  int dbg_cap;
};

// Resume point of a proposal that changes op o:
// R_o = the first round in which a task with an o-dependent successor list ran
// -- a forward task of o or of one of its producers, or (full-iteration) a
// backward task of o or of one of its consumers; a source op resumes nowhere.
// Returns the last usable snapshot index at or before R_o (0: from scratch) and
// points the warp's delta context at it.
__device__ inline int delta_prepare(const DevProb &P, const Tab &T, const W2 &w, const DeltaBufs &db, int chain,
                                    int o, double cost, bool full, bool from_scratch, int lane) {
  DeltaCtx *dc = w.dc;
  const ChainDelta &ch = dc->ch;  // (shared memory: read in place)
  int *fb0 = db.frb + (size_t)chain * 4 * P.n_ops;
  const int *fcur = fb0 + (size_t)(ch.fsel * 2) * P.n_ops, *bcur = fcur + P.n_ops;
  int *fnew = fb0 + (size_t)((ch.fsel ^ 1) * 2) * P.n_ops, *bnew = fnew + P.n_ops;
  int j = 0;
  if (!from_scratch && db.exp != 2 && ch.stride > 0 && ch.nvalid > 1 && P.min_exe > __dmul_rn(cost, 0x1p-50)) {
    // (first snapshot index at which a task with an o-dependent successor list had run) - 1
    int i0 = T.op_in_off[o], i1 = T.op_in_off[o + 1];
    int R = i0 == i1 ? 0 : fcur[o];
    if (full) R = min(R, bcur[o]);
    for (int i = i0 + lane; i < i1; i += 32) R = min(R, fcur[T.pair_src[T.op_in_pairs[i]]]);
    if (full)
      for (int i = T.op_out_off[o] + lane; i < T.op_out_off[o + 1]; i += 32)
        R = min(R, bcur[T.pair_dst[T.op_out_pairs[i]]]);
    R = __reduce_min_sync(FULLMASK, R);
    j = max(0, min(R - 1, ch.nvalid - 1));
    while (j > 0 && ((ch.bad >> j) & 1u)) --j;
  }
  __syncwarp();
  // an epoch buffer no live snapshot of the current strategy refers to
  unsigned used = 0;
  for (int i = 1; i < ch.nvalid; ++i) used |= 1u << ch.ep[i];
  const int epoch = __ffs(~used) - 1;  // nsnap + 1 buffers, at most nsnap - 1 in use
  if (lane == 0) {
    const unsigned long long eps = snap_counters_pad(P);
    dc->indeg0 = db.indeg + (size_t)chain * (db.nsnap + 1) * eps;
    dc->ep_stride = eps;
    dc->epoch = epoch;
    dc->snap = ch.stride > 0 && db.exp != 1 ? db.snaps + (size_t)chain * 2 * db.nsnap * db.snap_bytes : nullptr;
    dc->restore = j > 0 ? dc->snap + (2ull * j + ((ch.cur >> j) & 1u)) * db.snap_bytes : nullptr;
    dc->frnd = fnew; dc->brnd = bnew;
    dc->fsrc = fcur; dc->bsrc = bcur;
    dc->indeg = db.indeg + ((size_t)chain * (db.nsnap + 1) + epoch) * eps;
    dc->snap_bytes = db.snap_bytes;
    dc->stride = ch.stride;
    dc->nsnap = db.nsnap;
    dc->out_sel = ~ch.cur;
    dc->op = o;
    dc->restore_idx = j;
    dc->r0 = j * ch.stride;
  }
  __syncwarp();
  return j;
}

// After an accepted delta simulation: its snapshots past the resume point and
// its first rounds become the chain's current ones.
__device__ inline void delta_commit(DeltaCtx *dc, int j, int lane) {
  __syncwarp();
  if (lane == 0) {
    ChainDelta &ch = dc->ch;
    if (ch.stride > 0) {
      int last = dc->last;
      unsigned upto = last >= 31 ? 0xffffffffu : ((1u << (last + 1)) - 1u);
      unsigned mask = upto & ~((1u << (j + 1)) - 1u);
      ch.cur ^= mask;
      ch.bad = (ch.bad & ~mask) | (dc->bad & mask);
      ch.nvalid = last + 1;
      for (int i = j + 1; i <= last; ++i) ch.ep[i] = (unsigned char)dc->epoch;
    }
    ch.fsel ^= 1;
  }
  __syncwarp();
}

// Given single-op changes (ps_delta_batch): chain i's op[i] takes local map
// map[i] and devices asg[i * stride + k]; commit[i] keeps it (else rolled back);
// the new makespan / status go to mk[i] / status[i].  op == nullptr: the chains
// draw their own proposals (MCMC).
struct Given {
  const int *op, *map;
  const unsigned char *asg, *commit;
  int stride;
  double *mk;
  int *status;
};

// One chain's segment of the MCMC (k_mcmc runs the chains of a warp one after another).
template <int S>
__device__ __forceinline__ void mcmc_chain(const DevProb &P, const Lay &lay, const Tab &T, W2 &w, int lane, int chain,
                                           int proposals, int rng_mode, int beta_given, double beta_param,
                                           double ln10, int *maps, unsigned char *asgs, int *best_maps,
                                           unsigned char *best_asgs, ChainState *st, unsigned *mt_all,
                                           double *trace_cand, unsigned char *trace_ok, int trace_cap, char *gs,
                                           unsigned long long budget_ns, const DeltaBufs &db, const Given &gv) {
  constexpr bool DELTA = (S & SIM_SNAP) != 0;
  int *gmapl = maps + (size_t)chain * P.n_ops;
  unsigned char *gasg = asgs + (size_t)chain * P.n_slots;
  ChainState cs = st[chain];
  if (gv.op) {
    if (gv.op[chain] < 0) return;  // no change for this chain
    if (cs.status != PS_STATUS_OK) {
      if (lane == 0) { gv.mk[chain] = cs.cost; gv.status[chain] = cs.status; }
      return;
    }
  }
  if (cs.status != PS_STATUS_OK) return;
  if (DELTA) {
    if (lane == 0) w.dc->ch = db.cd[chain];
    __syncwarp();
  }
  for (int i = lane; i < P.n_ops; i += 32) w.mapl[i] = gmapl[i];
  if (lay.asg_global) w.asg = gasg;
  else
    for (int i = lane; i < P.n_slots; i += 32) w.asg[i] = gasg[i];
  __syncwarp();
  WarpRng rng;
  rng.mode = rng_mode;
  rng.key = cs.key;
  rng.ctr = cs.ctr;
  rng.bpos = cs.bpos;
  rng.lane = lane;
  rng.mt = mt_all ? mt_all + (size_t)chain * 624 : nullptr;
  rng.mti = cs.mti;
  if (rng_mode == PS_RNG_PHILOX && rng.bpos < 4) philox_block(rng.ctr - 1, rng.key, rng.buf);
  int *bmap = best_maps + (size_t)chain * P.n_ops;
  unsigned char *basg = best_asgs + (size_t)chain * P.n_slots;
  unsigned long long t0 = globaltimer_ns();
#ifdef PS_PHASES
  for (int i = lane; i < PH_N; i += 32) w.ph[i] = 0;
  __syncwarp();
#endif
  PH_T(t_loop);
  int n_it = 0;
  // iteration -1 scores the chain's initial strategy (first launch only); the
  // simulator has a single call site so the kernel holds one copy of it
  for (int it = cs.started ? 0 : -1; it < proposals; ++it) {
    int o = 0, m = 0, base = 0, old_m = 0, old_size = 0;
    bool same = false;
    if (it >= 0) {
      ++n_it;
      if (budget_ns) {
        // time-boxed segment: stop between proposals when the next one (at
        // this chain's mean proposal time so far) would end past the budget,
        // so the segment ends close to the budget instead of waiting for the
        // slowest chain's overshoot
        unsigned long long now = __shfl_sync(FULLMASK, globaltimer_ns(), 0);
        unsigned long long spent = now - t0, mean = n_it > 1 ? spent / (unsigned long long)(n_it - 1) : 0ull;
        if (spent + mean >= budget_ns) break;
      }
      // _propose_change (search.py:101-115): op, degree map, one device per task
      // (or the caller's change: update_task_graph's op and config)
      o = gv.op ? gv.op[chain] : (int)rng.below((unsigned)P.n_ops);
      m = gv.op ? gv.map[chain] : (int)rng.below((unsigned)P.op_nmaps_enum[o]);
      cs.last_op = o;
      int g = T.op_map_off[o] + m;
      int size = P.map_size[g];
      base = T.op_slot_off[o];
      old_m = w.mapl[o];
      old_size = P.map_size[T.op_map_off[o] + old_m];
      same = (m == old_m);
      for (int i = lane; i < old_size; i += 32) w.oldasg[i] = w.asg[base + i];
      __syncwarp();
      for (int k = 0; k < size; ++k) {
        unsigned dv = gv.op ? gv.asg[(size_t)chain * gv.stride + k] : rng.below((unsigned)P.n_dev);
        same = same && (k < old_size && w.oldasg[k] == (unsigned char)dv);
        __syncwarp();
        if (lane == 0) w.asg[base + k] = (unsigned char)dv;
      }
      if (lane == 0) w.mapl[o] = m;
      __syncwarp();
    }
    double cand;
    int dj = 0;  // resumed snapshot index of this proposal's delta simulation
    if (same) {
      cand = cs.cost;
    } else {
      SimOut so;
      // the initial scoring of a delta chain runs twice: once to learn the
      // round count (the snapshot spacing), once to take its snapshots
      const int npass = (DELTA && it < 0) ? 2 : 1;
#pragma unroll 1
      for (int pass = 0; pass < npass; ++pass) {
        if (DELTA) {
          const bool full = (S & SIM_FULL) ? true : (S & SIM_FWD) ? false : P.full != 0;
          PH_T(t_prep);
          dj = delta_prepare(P, T, w, db, chain, o, cs.cost, full, it < 0, lane);
          PH_ADD(29, t_prep);
        }
        so = simulate_any<S>(P, T, w, lay, gs, lane);
        if (so.status != PS_STATUS_OK) break;
        if (DELTA && db.dbg && lane == 0 && it >= 0 && cs.proposals < db.dbg_cap) {
          int *d = db.dbg + ((size_t)chain * db.dbg_cap + cs.proposals) * 8;
          d[0] = o; d[1] = dj; d[2] = w.dc->ch.nvalid; d[3] = w.dc->rounds; d[4] = w.dc->ch.stride;
          d[5] = w.dc->last; d[6] = (int)w.dc->ch.bad; d[7] = w.dc->ch.fsel;
        }
        if (DELTA) {
          if (lane == 0) {
            ChainDelta &ch = w.dc->ch;
            if (it < 0 && pass == 0) {
              // snapshots spread over the rounds that can be resumed from: the
              // forward part in full-iteration mode (see delta_prepare), all in forward mode
              const bool fullm = (S & SIM_FULL) ? true : (S & SIM_FWD) ? false : P.full != 0;
              int r = fullm ? w.dc->rounds_fwd : w.dc->rounds;
              ch.stride = max(4, (r + db.nsnap - 1) / db.nsnap);
            } else {
              ch.rounds_reused += w.dc->r0;
              ch.rounds_run += w.dc->rounds - w.dc->r0;
            }
          }
          __syncwarp();
          if (it < 0) delta_commit(w.dc, 0, lane);
        }
      }
      if (so.status != PS_STATUS_OK) {
        cs.status = so.status; cs.err_a = so.err_a; cs.err_b = so.err_b;
        if (gv.op && lane == 0) { gv.mk[chain] = __longlong_as_double(0x7ff0000000000000ll); gv.status[chain] = so.status; }
        if (it < 0) {
          cs.started = 1;
          cs.initial = cs.best = cs.cost = __longlong_as_double(0x7ff0000000000000ll);
          if (lane == 0) st[chain] = cs;
          if (DELTA && lane == 0) db.cd[chain] = w.dc->ch;
          return;
        }
        break;
      }
      cand = so.makespan;
    }
    if (it < 0) {
      cs.started = 1;
      cs.cost = cs.best = cs.initial = cand;
      cs.beta = beta_given ? beta_param : (cand > 0.0 ? __ddiv_rn(ln10, __dmul_rn(0.05, cand)) : 1.0);
      for (int i = lane; i < P.n_ops; i += 32) bmap[i] = w.mapl[i];
      for (int i = lane; i < P.n_slots; i += 32) basg[i] = w.asg[i];
      __syncwarp();
      continue;  // (the budget covers the initial scoring too: all chains end together)
    }
    long long idx = cs.proposals++;
    bool ok;
    if (gv.op) {
      ok = gv.commit ? gv.commit[chain] != 0 : true;
      if (lane == 0) { gv.mk[chain] = cand; gv.status[chain] = PS_STATUS_OK; }
    } else if (cand <= cs.cost) ok = true;
    else {
      double pr = exp(__dmul_rn(cs.beta, __dsub_rn(cs.cost, cand)));
      ok = pr >= 1.0 ? true : rng.random() < pr;
    }
    if (trace_cap > 0 && lane == 0) {
      // a ring of trace_cap proposals per chain: the host reads it back at least
      // every trace_cap proposals (time-boxed searches read it after each segment)
      size_t slot = (size_t)chain * trace_cap + (size_t)(idx % trace_cap);
      trace_cand[slot] = cand;
      trace_ok[slot] = ok;
    }
    if (cand < cs.best) {
      cs.best = cand;
      for (int i = lane; i < P.n_ops; i += 32) bmap[i] = w.mapl[i];
      for (int i = lane; i < P.n_slots; i += 32) basg[i] = w.asg[i];
    }
    if (ok) {
      cs.cost = cand;
      cs.accepted++;
      if (DELTA && !same) delta_commit(w.dc, dj, lane);
    } else {
      for (int i = lane; i < old_size; i += 32) w.asg[base + i] = w.oldasg[i];
      if (lane == 0) w.mapl[o] = old_m;
    }
    __syncwarp();
  }
  PH_ADD(6, t_loop);
  PH_CNT(7, n_it);
#ifdef PS_PHASES
  __syncwarp();
  for (int i = lane; i < PH_N; i += 32) atomicAdd(&g_phase[i], w.ph[i]);
#endif
  for (int i = lane; i < P.n_ops; i += 32) gmapl[i] = w.mapl[i];
  if (!lay.asg_global)
    for (int i = lane; i < P.n_slots; i += 32) gasg[i] = w.asg[i];
  cs.key = rng.key;
  cs.ctr = rng.ctr;
  cs.bpos = rng.bpos;
  cs.mti = rng.mti;
  if (lane == 0) st[chain] = cs;
  if (DELTA && lane == 0) db.cd[chain] = w.dc->ch;
}

template <int S>
__global__ void PS_BOUNDS(S)
k_mcmc(DevProb P, Lay lay, int n_chains, int proposals, int rng_mode, int beta_given, double beta_param, double ln10,
       int *maps, unsigned char *asgs, int *best_maps, unsigned char *best_asgs, ChainState *st, unsigned *mt_all,
       double *trace_cand, unsigned char *trace_ok, int trace_cap, char *gscratch, unsigned long long budget_ns,
       DeltaBufs db, Given gv) {
  extern __shared__ __align__(16) char smem[];
  int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  const int gw = blockIdx.x * wpb + wib, nw = gridDim.x * wpb;
  char *gs = gscratch + (size_t)(gw < n_chains ? gw : 0) * gslice_bytes(P, lay);
  Tab T;
  W2 w;
  kernel_layout(P, lay, smem, gs, wib, T, w);
  __syncthreads();
  if (gw >= n_chains) return;
  bind_bids(P, gs, w);
  if (lane == 0) w.flags[0] = 1;
  __syncwarp();
  // chains gw, gw + nw, ...: a warp runs its chains one after another when there
  // are more chains than resident warps (no second wave waiting for the first);
  // a time-boxed segment is split evenly among them
  const int m = (n_chains - gw + nw - 1) / nw;
  const unsigned long long slice = budget_ns ? (budget_ns / (unsigned long long)m > 0 ? budget_ns / m : 1ull) : 0ull;
#pragma unroll 1
  for (int chain = gw; chain < n_chains; chain += nw)
    mcmc_chain<S>(P, lay, T, w, lane, chain, proposals, rng_mode, beta_given, beta_param, ln10, maps, asgs, best_maps,
                  best_asgs, st, mt_all, trace_cand, trace_ok, trace_cap, gs, slice, db, gv);
}

__global__ void k_best(const ChainState *st, int n, double *best_cost, int *best_chain) {
  // single block argmin by (best, chain) -- earliest chain wins ties (search.py:256)
  __shared__ double sb[1024];
  __shared__ int si[1024];
  double b = __longlong_as_double(0x7ff0000000000000ll);
  int bi = -1;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double v = st[i].best;
    bool live = st[i].started && st[i].initial < __longlong_as_double(0x7ff0000000000000ll);
    if (live && (bi < 0 || v < b)) { b = v; bi = i; }
  }
  sb[threadIdx.x] = b;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      double ob = sb[threadIdx.x + s];
      int oi = si[threadIdx.x + s];
      if (oi >= 0 && (si[threadIdx.x] < 0 || ob < sb[threadIdx.x] || (ob == sb[threadIdx.x] && oi < si[threadIdx.x]))) {
        sb[threadIdx.x] = ob;
        si[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { *best_cost = sb[0]; *best_chain = si[0]; }
}

template <class T>
int upload(std::vector<void *> &owned, const T *host, size_t n, const T **dev) {
  if (n == 0) { *dev = nullptr; return PS_OK; }
  void *p = nullptr;
  CK(cudaMalloc(&p, n * sizeof(T)));
  owned.push_back(p);
  CK(cudaMemcpy(p, host, n * sizeof(T), cudaMemcpyHostToDevice));
  *dev = (const T *)p;
  return PS_OK;
}

}  // namespace

// kernel variant pickers: v = 0 generic, 1 simple full-iteration, 2 simple forward
typedef void (*BatchKernel)(DevProb, Lay, const int *, const unsigned char *, int, double *, int *, char *, double *,
                            int *);
static BatchKernel batch_kernel(int v, bool wide) {
  if (wide)
    return v == 0 ? k_simulate_batch<SIM_BACK> : v == 1 ? k_simulate_batch<SIM_BACK | SIM_SIMPLE | SIM_FULL>
                                                        : k_simulate_batch<SIM_BACK | SIM_SIMPLE | SIM_FWD>;
  return v == 0 ? k_simulate_batch<0> : v == 1 ? k_simulate_batch<SIM_SIMPLE | SIM_FULL>
                                               : k_simulate_batch<SIM_SIMPLE | SIM_FWD>;
}
typedef void (*McmcKernel)(DevProb, Lay, int, int, int, int, double, double, int *, unsigned char *, int *,
                           unsigned char *, ChainState *, unsigned *, double *, unsigned char *, int, char *,
                           unsigned long long, DeltaBufs, Given);
static McmcKernel mcmc_kernel(int v, bool snap, bool wide) {
  constexpr int B = SIM_BACK, S = SIM_SNAP, F = SIM_SIMPLE | SIM_FULL, W = SIM_SIMPLE | SIM_FWD;
  if (wide) {
    if (snap) return v == 0 ? k_mcmc<B | S> : v == 1 ? k_mcmc<B | S | F> : k_mcmc<B | S | W>;
    return v == 0 ? k_mcmc<B> : v == 1 ? k_mcmc<B | F> : k_mcmc<B | W>;
  }
  if (snap) return v == 0 ? k_mcmc<S> : v == 1 ? k_mcmc<S | F> : k_mcmc<S | W>;
  return v == 0 ? k_mcmc<0> : v == 1 ? k_mcmc<F> : k_mcmc<W>;
}

struct ps_problem {
  int device;
  DevProb P;
  std::vector<void *> owned;
  long long n_entries, n_combos, n_rows, n_cols;
  size_t smem_per_block;  // v2 kernels: tab + wpb * warp slice
  int blocks_per_sm, sm_count, wpb;
  Lay lay;
  char *scratch = nullptr;  // batch scratch (grid-sized)
  size_t scratch_warps = 0;
  int *d_map = nullptr;
  unsigned char *d_asg = nullptr;
  double *d_mk = nullptr;
  int *d_st = nullptr;
  int *d_next = nullptr;  // batch work queue: next candidate to take
  bool simple = false;    // kernels' SIM_SIMPLE variant applies (one kind, <= 2 link classes, full mesh)
  bool wide = false;      // SIM_BACK variants: two-level ready set (many task slots, or PS_FORCE_WIDE)
  char *mcmc_scratch = nullptr;  // chain scratch kept from the last destroyed MCMC handle
  size_t mcmc_scratch_bytes = 0;
  // chain buffers kept from the last destroyed MCMC handle (create/run/destroy
  // cycles, as in an end-to-end loop, then allocate nothing)
  struct {
    int n = 0;
    int *maps = nullptr, *best_maps = nullptr;
    unsigned char *asgs = nullptr, *best_asgs = nullptr;
    void *st = nullptr;
    double *d_best = nullptr;
    int *d_bestc = nullptr;
  } spare;
  struct {  // delta buffers kept from the last destroyed MCMC handle (same chain and snapshot counts)
    int n = 0, ns = 0;
    ChainDelta *cd = nullptr;
    char *snaps = nullptr;
    int *frb = nullptr;
    unsigned short *indeg = nullptr;
  } spare_delta;
  size_t io_cap = 0;
  long long device_bytes = 0;
  std::vector<int> h_map_off, h_map_size;  // host copies: argument checks of ps_delta_batch
  size_t total_mem = 0;                    // device memory (snapshot budget), queried once
};

struct ps_mcmc {
  ps_problem *prob;
  int n;
  ps_mcmc_params params;
  int *maps, *best_maps;
  unsigned char *asgs, *best_asgs;
  ChainState *st;
  unsigned *mt;
  double *trace_cand;
  unsigned char *trace_ok;
  char *scratch;
  size_t scratch_bytes = 0;
  double *d_best;
  int *d_bestc;
  int cap_n;  // chains the buffers above were sized for
  DeltaBufs db;  // delta-evaluation state (db.cd == nullptr: every proposal simulates from scratch)
  char *given = nullptr;  // ps_delta_batch staging (host-pointer calls)
  size_t given_bytes = 0;
  int max_blocks = 0;     // PS_MCMC_MUX: resident blocks of the handle's k_mcmc variant (0: not yet known)
};

static int ensure_io(ps_problem *pr, size_t n) {
  if (n <= pr->io_cap) return PS_OK;
  cudaFree(pr->d_map); cudaFree(pr->d_asg); cudaFree(pr->d_mk); cudaFree(pr->d_st);
  CK(cudaMalloc(&pr->d_map, n * pr->P.n_ops * sizeof(int)));
  CK(cudaMalloc(&pr->d_asg, n * (size_t)pr->P.n_slots));
  CK(cudaMalloc(&pr->d_mk, n * sizeof(double)));
  CK(cudaMalloc(&pr->d_st, n * sizeof(int)));
  pr->io_cap = n;
  return PS_OK;
}

extern "C" {

const char *ps_last_error(void) { return g_err.c_str(); }
int ps_abi_version(void) { return PS_ABI_VERSION; }

namespace {
// frees temporary device buffers on every exit path of problem_build
struct TmpBufs {
  std::vector<void *> p;
  ~TmpBufs() { for (void *x : p) cudaFree(x); }
};
int problem_build(const ps_problem_desc *d, int device, ps_problem *pr);
}  // namespace

int ps_problem_create(const ps_problem_desc *d, int device, ps_problem **out) {
  if (!d || !out) return fail(PS_ERR_INVALID, "null argument");
  if (d->abi_version != PS_ABI_VERSION) return fail(PS_ERR_INVALID, "ABI version mismatch");
  if (d->n_devices > 64) return fail(PS_ERR_INVALID, "at most 64 devices per topology are supported");
  if (d->n_ops >= 65536) return fail(PS_ERR_INVALID, "at most 65535 operations are supported");
  CK(cudaSetDevice(device));
  ps_problem *pr = new ps_problem();
  pr->device = device;
  int rc = problem_build(d, device, pr);
  if (rc != PS_OK) {
    std::string msg = g_err;
    ps_problem_destroy(pr);  // every buffer allocated so far is owned by pr
    g_err = msg;
    return rc;
  }
  *out = pr;
  return PS_OK;
}

}  // extern "C"

namespace {
int problem_build(const ps_problem_desc *d, int device, ps_problem *pr) {
  DevProb &P = pr->P;
  P.n_ops = d->n_ops; P.n_dev = d->n_devices; P.n_kinds = d->n_kinds; P.n_links = d->n_links;
  P.n_pairs = d->n_pairs; P.n_maps = d->n_maps; P.full = d->mode_full; P.n_slots = d->n_slots;
  P.n_queues = d->n_devices + d->n_links;
  P.cap = d->ready_capacity > 0 ? d->ready_capacity : 128;
  if (const char *e = getenv("PS_READY_CAP")) P.cap = std::max(2, atoi(e));  // (experiments)
  P.mult = d->backward_multiplier;
  pr->h_map_off.assign(d->op_map_off, d->op_map_off + P.n_ops + 1);
  pr->h_map_size.assign(d->map_size, d->map_size + P.n_maps);
  std::vector<void *> &ow = pr->owned;
  int n_combos = 0;
  n_combos = d->combo_off[d->n_pairs];
  int n_rows = d->combo_row_off[n_combos], n_cols = d->combo_col_off[n_combos];
  int n_need = d->pair_need_off[d->n_pairs];
  int rc = PS_OK;
#define UP(field, count) \
  if ((rc = upload(ow, d->field, (size_t)(count), &P.field)) != PS_OK) return rc;
  UP(dev_kind, P.n_dev);
  UP(link_of, (size_t)P.n_dev * P.n_dev);
  UP(link_bw, P.n_links);
  UP(link_lat, P.n_links);
  UP(op_ndim, P.n_ops);
  if ((rc = upload(ow, (const long long *)d->op_dim, (size_t)P.n_ops * PS_MAXDIM, &P.op_dim)) != PS_OK) return rc;
  UP(op_esize, P.n_ops);
  UP(op_param_mask, P.n_ops);
  UP(op_map_off, P.n_ops + 1);
  UP(op_nmaps_enum, P.n_ops);
  UP(op_slot_off, P.n_ops + 1);
  UP(slot_op, P.n_slots);
  UP(op_in_off, P.n_ops + 1);
  UP(op_in_pairs, d->op_in_off[P.n_ops]);
  UP(op_out_off, P.n_ops + 1);
  UP(op_out_pairs, d->op_out_off[P.n_ops]);
  UP(map_deg, (size_t)P.n_maps * PS_MAXDIM);
  UP(map_size, P.n_maps);
  UP(exe_fwd, (size_t)P.n_maps * P.n_kinds);
  UP(exe_bwd, (size_t)P.n_maps * P.n_kinds);
  UP(map_shard, P.n_maps);
  UP(map_ngroups, P.n_maps);
  UP(pair_src, P.n_pairs);
  UP(pair_dst, P.n_pairs);
  UP(pair_need_off, P.n_pairs + 1);
  UP(need, (size_t)n_need * PS_MAXDIM * PS_NEED_STRIDE);
  UP(combo_off, P.n_pairs + 1);
  UP(combo_row_off, n_combos + 1);
  UP(combo_col_off, n_combos + 1);
#undef UP
  pr->n_combos = n_combos; pr->n_rows = n_rows; pr->n_cols = n_cols;
  {
    // link classes: distinct (latency, bandwidth) bit patterns, if at most two
    std::vector<int> cls(P.n_links, 0);
    int ncls = 0;
    for (int li = 0; li < P.n_links && ncls <= 2; ++li) {
      int c = 0;
      while (c < ncls && !(memcmp(&P.cls_lat[c], &d->link_lat[li], 8) == 0 &&
                           memcmp(&P.cls_bw[c], &d->link_bw[li], 8) == 0)) ++c;
      if (c == ncls) {
        if (ncls == 2) { ncls = 3; break; }
        P.cls_lat[c] = d->link_lat[li]; P.cls_bw[c] = d->link_bw[li]; ++ncls;
      }
      cls[li] = c;
    }
    P.n_cls = (ncls <= 2 && P.n_links < 16384) ? ncls : 0;
    bool mesh = true;
    for (int i = 0; i < P.n_dev && mesh; ++i)
      for (int j = 0; j < P.n_dev; ++j)
        if (i != j && d->link_of[i * P.n_dev + j] < 0) { mesh = false; break; }
    pr->simple = mesh && P.n_cls > 0 && P.n_kinds == 1;
    pr->wide = P.n_slots >= 4096 || getenv("PS_FORCE_WIDE") != nullptr;
    // delta snapshots of wide problems also hold the back ready set (up to 1024 entries)
    {
      int sbc = 1024;
      if (const char *e = getenv("PS_SNAP_BACK")) sbc = std::max(0, atoi(e));
      P.snap_b = pr->wide ? std::min(overflow_cap(P.n_slots), sbc) : 0;
    }
    std::vector<short> l16((size_t)P.n_dev * P.n_dev);
    for (size_t i = 0; i < l16.size(); ++i) {
      int li = d->link_of[i];
      l16[i] = (short)(li < 0 ? -1 : (P.n_cls ? (li | cls[li] << 14) : li));
    }
    if ((rc = upload(ow, l16.data(), l16.size(), &P.link16)) != PS_OK) return rc;
  }
  {
    // delta evaluation: dense ring-counter bound, and a lower bound of every
    // task time (op tasks from the tables; transfers >= 1 byte; ring hops
    // >= the smallest shard over 64 devices)
    P.n_rings = 0;
    double mn = INFINITY, min_shard = INFINITY;
    for (int o = 0; o < P.n_ops; ++o) {
      int mg = 0;
      for (int g = d->op_map_off[o]; g < d->op_map_off[o + 1]; ++g) {
        mg = std::max(mg, d->map_ngroups[g]);
        if (d->op_param_mask[o] >= 0 && d->map_shard[g] < min_shard) min_shard = d->map_shard[g];
      }
      if (d->op_param_mask[o] >= 0) P.n_rings += mg;
    }
    for (int i = 0; i < P.n_maps * P.n_kinds; ++i) mn = std::min(mn, std::min(d->exe_fwd[i], d->exe_bwd[i]));
    for (int l = 0; l < P.n_links; ++l) {
      mn = std::min(mn, d->link_lat[l] + 1.0 / d->link_bw[l]);
      if (min_shard < INFINITY) mn = std::min(mn, d->link_lat[l] + (min_shard / 64.0) / d->link_bw[l]);
    }
    P.min_exe = (mn > 0.0 && mn < INFINITY) ? mn : 0.0;
  }
  // ---- overlap tables: count rows -> scan -> fill, then the column index
  int *cnt = nullptr, *off = nullptr, *ccnt = nullptr, *coff = nullptr;
  void *tmp = nullptr;
  size_t tmp_bytes = 0, t2 = 0;
  TmpBufs tb_;
  CK(cudaMalloc(&cnt, (n_rows + 1) * sizeof(int)));
  tb_.p.push_back(cnt);
  CK(cudaMalloc(&off, (n_rows + 1) * sizeof(int)));
  ow.push_back(off);
  CK(cudaMalloc(&ccnt, (n_cols + 1) * sizeof(int)));
  tb_.p.push_back(ccnt);
  CK(cudaMalloc(&coff, (n_cols + 1) * sizeof(int)));
  ow.push_back(coff);
  CK(cudaMemset(cnt, 0, (n_rows + 1) * sizeof(int)));
  CK(cudaMemset(ccnt, 0, (n_cols + 1) * sizeof(int)));
  if (n_rows) k_rows<<<(n_rows + 127) / 128, 128>>>(P, n_rows, n_combos, cnt, nullptr);
  CK(cudaGetLastError());
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, off, n_rows + 1);
  cub::DeviceScan::ExclusiveSum(nullptr, t2, ccnt, coff, n_cols + 1);
  tmp_bytes = std::max(tmp_bytes, t2);
  CK(cudaMalloc(&tmp, tmp_bytes));
  tb_.p.push_back(tmp);
  CK(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, off, n_rows + 1));
  int n_ent = 0;
  CK(cudaMemcpy(&n_ent, off + n_rows, sizeof(int), cudaMemcpyDeviceToHost));
  pr->n_entries = n_ent;
  unsigned short *ek = nullptr, *el = nullptr;
  long long *eb = nullptr;
  int *cent = nullptr;
  CK(cudaMalloc(&ek, (n_ent + 1) * sizeof(unsigned short)));
  ow.push_back(ek);
  CK(cudaMalloc(&el, (n_ent + 1) * sizeof(unsigned short)));
  ow.push_back(el);
  CK(cudaMalloc(&eb, (n_ent + 1) * sizeof(long long)));
  ow.push_back(eb);
  CK(cudaMalloc(&cent, (n_ent + 1) * sizeof(int)));
  ow.push_back(cent);
  P.ent_k = ek; P.ent_l = el; P.ent_bytes = eb; P.col_ent = cent; P.row_ent_off = off;
  if (n_rows) k_rows<<<(n_rows + 127) / 128, 128>>>(P, n_rows, n_combos, nullptr, off);
  CK(cudaGetLastError());
  if (n_cols) k_cols<<<(n_cols + 127) / 128, 128>>>(P, n_cols, n_combos, ccnt, nullptr);
  CK(cudaGetLastError());
  CK(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, ccnt, coff, n_cols + 1));
  P.col_ent_off = coff;
  if (n_cols) k_cols<<<(n_cols + 127) / 128, 128>>>(P, n_cols, n_combos, nullptr, coff);
  CK(cudaGetLastError());
  void *e16 = nullptr, *c16 = nullptr;
  CK(cudaMalloc(&e16, (size_t)(n_ent + 1) * sizeof(Ent32)));
  ow.push_back(e16);
  CK(cudaMalloc(&c16, (size_t)(n_ent + 1) * sizeof(Ent32)));
  ow.push_back(c16);
  P.ent16 = e16; P.cent16 = c16;
  if (n_ent) k_pack<<<(n_ent + 127) / 128, 128>>>(P, n_ent, (int)n_rows, (int)n_combos, e16, c16);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  // ---- launch geometry: largest shared-state capacity S that still keeps
  // >= 8 resident warps (candidates) per SM; warps per block in {4, 2, 1}
  CK(cudaDeviceGetAttribute(&pr->sm_count, cudaDevAttrMultiProcessorCount, device));
  int optin = 0, per_sm = 0;
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  CK(cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device));
  {
    // Shared-memory budget per resident warp: counters for SC tasks, GC parameter
    // shards and RC staged overlap offsets.  Pick the largest capacities that keep
    // `target` resident warps per SM (default 8: 1024 chains on 148 SMs).
    size_t tb = al16(tab_bytes_of(P));
    int target = 7;  // 7 x 148 SMs = 1036 resident chains >= the 1024-chain workload
    if (const char *e = getenv("PS_TARGET_WARPS_PER_SM")) target = std::max(1, atoi(e));
    int bestSC = -1, bestW = 0, bestWarps = 0, bestRC = 0, bestGC = 0, bestAG = 0;
    std::vector<int> caps;
    for (int c = 4096; c >= 128; c -= 32) caps.push_back(c);
    caps.push_back(0);
    int ag0 = getenv("PS_FORCE_ASG_GLOBAL") ? 1 : 0;  // test hook: exercise the in-place path
    int rc_frac = 11;  // staged row / column offsets per 16 counters (0: read in place)
    if (const char *e = getenv("PS_RC_FRAC")) rc_frac = std::max(0, atoi(e));
    // resident warps per SM the evaluation kernels' registers allow
    int reg_warps = 64;
    const int max_wpb = (pr->wide ? PS_WIDE_THREADS : PS_MAX_THREADS) / 32;
    {
      cudaFuncAttributes fa;
      if (cudaFuncGetAttributes(&fa, mcmc_kernel(1, true, pr->wide)) == cudaSuccess && fa.numRegs > 0) {
        int per_warp = ((fa.numRegs * 32 + 255) / 256) * 256;
        reg_warps = 65536 / per_warp;
      }
    }
    for (int ag = ag0; ag < 2 && bestWarps < target; ++ag) {
      for (int ci = 0; ci < (int)caps.size(); ++ci) {
        // ring shards and staged rows / columns sized in proportion to the task
        // counters (typical full-iteration candidates: G ~ 0.19, rows ~ 0.69 of 2 Tf + G)
        int SC = caps[ci];
        int GC = std::max(16, (SC * 5 + 23) / 24);
        int RC = rc_frac ? std::max(64, SC * rc_frac / 16) : 0;
        size_t wb = al16(warp_bytes_of(P, SC, GC, RC, ag));
        int cw = 0, cwp = 0;
        for (int wp : {12, 11, 10, 9, 8, 7, 6, 5, 4, 3, 2, 1}) {
          if (wp > max_wpb) continue;
          size_t blk = tb + wp * wb;
          if (blk > (size_t)optin) continue;
          int blocks = std::min(32, (int)(per_sm / (blk + 1024)));
          int warps = std::min(reg_warps / wp * wp, blocks * wp);
          if (warps > cw) { cw = warps; cwp = wp; }
        }
        if (cw > bestWarps || (cw >= target && bestWarps < target)) {
          bestWarps = cw; bestSC = SC; bestW = cwp; bestRC = RC; bestGC = GC; bestAG = ag;
        }
        if (cw >= target) break;
      }
    }
    if (getenv("PS_FORCE_GLOBAL_ALL")) bestSC = -1;  // test hook: exercise the global layout
    if (bestSC < 0) {
      // nothing fits on chip: block tables and warp slices move to global memory
      pr->lay.global_all = 1;
      pr->lay.warp_global = 0;
      pr->lay.asg_global = 1;
      pr->lay.SC = 3 * P.n_slots + 64;
      pr->lay.GC = P.n_slots + 16;
      pr->lay.RC = 0;
      pr->lay.tab_bytes = 0;
      pr->lay.warp_bytes = al16(warp_bytes_of(P, pr->lay.SC, pr->lay.GC, pr->lay.RC, 1));
      pr->wpb = std::min(8, max_wpb);
      pr->lay.hot_bytes = (int)al16(hot_bytes_of(P));
      if ((size_t)pr->wpb * pr->lay.hot_bytes > (size_t)optin || getenv("PS_NO_HOT")) pr->lay.hot_bytes = 0;
      pr->smem_per_block = (size_t)pr->wpb * pr->lay.hot_bytes;
      bestW = pr->wpb; bestWarps = std::min(reg_warps, 32); bestSC = pr->lay.SC;
    } else {
      pr->lay.global_all = 0;
      pr->lay.hot_bytes = 0;
      pr->lay.warp_global = 0;
    pr->lay.tab_bytes = tb;
    pr->lay.SC = bestSC;
    pr->lay.GC = bestGC;
    pr->lay.RC = bestRC;
    pr->lay.asg_global = bestAG;
    pr->lay.warp_bytes = al16(warp_bytes_of(P, bestSC, bestGC, bestRC, bestAG));
    pr->wpb = bestW;
    pr->smem_per_block = tb + bestW * pr->lay.warp_bytes;
    // Wide problems whose warp slices keep few warps resident: the slices move
    // to global memory and only the per-round state stays on chip, when that at
    // least doubles the resident warps (as many as the registers allow)
    const bool force_wg = getenv("PS_FORCE_WARP_GLOBAL") != nullptr;  // test hook
    if (pr->wide && (bestWarps < target || force_wg) && !getenv("PS_NO_WARP_GLOBAL")) {
      size_t hot = al16(hot_bytes_of(P));
      int cw = 0, cwp = 0;
      for (int wp : {8, 4, 2}) {
        size_t blk = tb + wp * hot;
        if (blk > (size_t)optin || wp > max_wpb) continue;
        int blocks = std::min(32, (int)(per_sm / (blk + 1024)));
        int warps = std::min(reg_warps / wp * wp, blocks * wp);
        if (warps > cw) { cw = warps; cwp = wp; }
      }
      if (cw >= 2 * bestWarps || (force_wg && cw > 0)) {
        pr->lay.warp_global = 1;
        pr->lay.asg_global = 1;
        pr->lay.SC = 3 * P.n_slots + 64;
        pr->lay.GC = P.n_slots + 16;
        pr->lay.RC = 0;
        pr->lay.hot_bytes = (int)hot;
        pr->lay.warp_bytes = al16(warp_bytes_of(P, pr->lay.SC, pr->lay.GC, pr->lay.RC, 1));
        pr->wpb = cwp;
        pr->smem_per_block = tb + (size_t)cwp * hot;
        bestW = cwp; bestWarps = cw; bestSC = pr->lay.SC;
      }
    }
    }
    pr->blocks_per_sm = std::max(1, bestWarps / bestW);
  }
  // the attribute is per kernel, not per problem: allow the device maximum so
  // problems with different layouts can coexist
  for (int wide = 0; wide < 2; ++wide)
    for (int v = 0; v < 3; ++v) {
      CK(cudaFuncSetAttribute(batch_kernel(v, wide), cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
      for (int snap = 0; snap < 2; ++snap)
        CK(cudaFuncSetAttribute(mcmc_kernel(v, snap, wide), cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    }
  CK(cudaFuncSetAttribute(k_simulate_trace, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, mcmc_kernel(pr->simple ? (P.full ? 1 : 2) : 0, true, pr->wide),
                                                   pr->wpb * 32, pr->smem_per_block));
  if (getenv("PS_DEBUG"))
    fprintf(stderr, "[parasim] tab=%zu warp=%zu SC=%d GC=%d RC=%d wpb=%d smem/block=%zu occ=%d optin=%d per_sm=%d\n",
            pr->lay.tab_bytes, pr->lay.warp_bytes, pr->lay.SC, pr->lay.GC, pr->lay.RC, pr->wpb, pr->smem_per_block, occ,
            optin, per_sm);
  if (occ < 1) return fail(PS_ERR_CAPACITY, "kernel does not fit on an SM");
  pr->blocks_per_sm = occ;
  pr->device_bytes = 0;
  return PS_OK;
}
}  // namespace

extern "C" {

void ps_problem_destroy(ps_problem *pr) {
  if (!pr) return;
  cudaSetDevice(pr->device);
  for (void *p : pr->owned) cudaFree(p);
  cudaFree(pr->scratch);
  cudaFree(pr->d_map); cudaFree(pr->d_asg); cudaFree(pr->d_mk); cudaFree(pr->d_st); cudaFree(pr->d_next);
  cudaFree(pr->mcmc_scratch);
  cudaFree(pr->spare.maps); cudaFree(pr->spare.best_maps); cudaFree(pr->spare.asgs); cudaFree(pr->spare.best_asgs);
  cudaFree(pr->spare.st); cudaFree(pr->spare.d_best); cudaFree(pr->spare.d_bestc);
  cudaFree(pr->spare_delta.cd); cudaFree(pr->spare_delta.snaps); cudaFree(pr->spare_delta.frb);
  cudaFree(pr->spare_delta.indeg);
  delete pr;
}

int ps_problem_info_get(const ps_problem *pr, ps_problem_info *o) {
  if (!pr || !o) return fail(PS_ERR_INVALID, "null argument");
  o->n_entries = pr->n_entries;
  o->n_combos = pr->n_combos;
  o->n_queues = pr->P.n_queues;
  o->n_slots = pr->P.n_slots;
  o->ready_capacity = pr->P.cap;
  o->warps_per_block = pr->wpb;
  o->device_bytes = pr->device_bytes;
  o->shared_counters = pr->lay.SC;
  o->resident_warps_per_sm = pr->blocks_per_sm * pr->wpb;
  o->smem_per_block = (int32_t)pr->smem_per_block;
  return PS_OK;
}

int ps_combo_entries(ps_problem *pr, int pair, int src_map, int dst_map, int cap, int32_t *k_out,
                     int32_t *l_out, int64_t *bytes_out, int *n_out) {
  CK(cudaSetDevice(pr->device));
  // host copies of the small offset tables are not kept; fetch what we need
  int co[2];
  CK(cudaMemcpy(co, pr->P.combo_off + pair, sizeof(int), cudaMemcpyDeviceToHost));
  int dst = 0, md[2];
  CK(cudaMemcpy(&dst, pr->P.pair_dst + pair, sizeof(int), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(md, pr->P.op_map_off + dst, 2 * sizeof(int), cudaMemcpyDeviceToHost));
  int c = co[0] + src_map * (md[1] - md[0]) + dst_map;
  int ro[2];
  CK(cudaMemcpy(ro, pr->P.combo_row_off + c, 2 * sizeof(int), cudaMemcpyDeviceToHost));
  int e[2];
  CK(cudaMemcpy(&e[0], pr->P.row_ent_off + ro[0], sizeof(int), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&e[1], pr->P.row_ent_off + ro[1], sizeof(int), cudaMemcpyDeviceToHost));
  int n = e[1] - e[0];
  *n_out = n;
  if (n > cap) return fail(PS_ERR_INVALID, "buffer too small");
  std::vector<unsigned short> k(n), l(n);
  std::vector<long long> b(n);
  if (n) {
    CK(cudaMemcpy(k.data(), pr->P.ent_k + e[0], n * 2, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(l.data(), pr->P.ent_l + e[0], n * 2, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(b.data(), pr->P.ent_bytes + e[0], n * 8, cudaMemcpyDeviceToHost));
  }
  for (int i = 0; i < n; ++i) { k_out[i] = k[i]; l_out[i] = l[i]; bytes_out[i] = b[i]; }
  return PS_OK;
}

int ps_simulate_batch_ex(ps_problem *pr, const int32_t *map_local, const uint8_t *assign, int n, double *makespan_out,
                         int32_t *status_out, double *op_min_end_out, int flags, void *stream) {
  if (!pr || n < 0) return fail(PS_ERR_INVALID, "bad arguments");
  if (n == 0) return PS_OK;
  CK(cudaSetDevice(pr->device));
  cudaStream_t s = (cudaStream_t)stream;
  const int *dm = map_local;
  const unsigned char *da = assign;
  double *dk = makespan_out;
  int *ds = status_out;
  if (flags != PS_DEVICE_PTRS) {
    int rc = ensure_io(pr, n);
    if (rc) return rc;
    CK(cudaMemcpyAsync(pr->d_map, map_local, (size_t)n * pr->P.n_ops * sizeof(int), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(pr->d_asg, assign, (size_t)n * pr->P.n_slots, cudaMemcpyHostToDevice, s));
    dm = pr->d_map; da = pr->d_asg; dk = pr->d_mk; ds = pr->d_st;
  }
  int wpb = pr->wpb;
  int blocks = std::min((n + wpb - 1) / wpb, pr->sm_count * pr->blocks_per_sm);
  size_t warps = (size_t)blocks * wpb;
  if (warps > pr->scratch_warps) {
    cudaFree(pr->scratch);
    size_t want = (size_t)pr->sm_count * pr->blocks_per_sm * wpb;
    CK(cudaMalloc(&pr->scratch, want * gslice_bytes(pr->P, pr->lay)));
    pr->scratch_warps = want;
  }
  double *dop = nullptr;
  if (op_min_end_out) {
    if (flags == PS_DEVICE_PTRS) dop = op_min_end_out;
    else CK(cudaMalloc(&dop, (size_t)n * pr->P.n_ops * sizeof(double)));
  }
  if (!pr->d_next) CK(cudaMalloc(&pr->d_next, sizeof(int)));
  CK(cudaMemsetAsync(pr->d_next, 0, sizeof(int), s));
  auto kb = batch_kernel(!pr->simple ? 0 : pr->P.full ? 1 : 2, pr->wide);
  kb<<<blocks, wpb * 32, pr->smem_per_block, s>>>(pr->P, pr->lay, dm, da, n, dk, ds, pr->scratch, dop,
                                                                 pr->d_next);
  CK(cudaGetLastError());
  if (flags != PS_DEVICE_PTRS) {
    CK(cudaMemcpyAsync(makespan_out, dk, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(status_out, ds, n * sizeof(int), cudaMemcpyDeviceToHost, s));
    if (dop) CK(cudaMemcpyAsync(op_min_end_out, dop, (size_t)n * pr->P.n_ops * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (dop) cudaFree(dop);
  }
  return PS_OK;
}

int ps_simulate_batch(ps_problem *pr, const int32_t *map_local, const uint8_t *assign, int n, double *makespan_out,
                      int32_t *status_out, int flags, void *stream) {
  return ps_simulate_batch_ex(pr, map_local, assign, n, makespan_out, status_out, nullptr, flags, stream);
}

int ps_simulate_trace(ps_problem *pr, const int32_t *map_local, const uint8_t *assign, int task_cap,
                      ps_trace_task *tasks, int *n_tasks, int edge_cap, int32_t *edge_pred, uint64_t *edge_succ_key,
                      int *n_edges, double *makespan, int32_t *status, int32_t *err_devices) {
  CK(cudaSetDevice(pr->device));
  int rc = ensure_io(pr, 1);
  if (rc) return rc;
  char *scr = nullptr;
  ps_trace_task *dt = nullptr;
  int32_t *dep = nullptr;
  unsigned long long *des = nullptr;
  int *cnts = nullptr, *err = nullptr;
  double *dmk = nullptr;
  CK(cudaMalloc(&scr, gslice_bytes(pr->P, pr->lay)));
  CK(cudaMalloc(&dt, sizeof(ps_trace_task) * (size_t)std::max(task_cap, 1)));
  CK(cudaMalloc(&dep, sizeof(int32_t) * (size_t)std::max(edge_cap, 1)));
  CK(cudaMalloc(&des, sizeof(unsigned long long) * (size_t)std::max(edge_cap, 1)));
  CK(cudaMalloc(&cnts, 2 * sizeof(int)));
  CK(cudaMalloc(&err, 3 * sizeof(int)));
  CK(cudaMalloc(&dmk, sizeof(double)));
  CK(cudaMemset(cnts, 0, 2 * sizeof(int)));
  CK(cudaMemcpy(pr->d_map, map_local, pr->P.n_ops * sizeof(int), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(pr->d_asg, assign, pr->P.n_slots, cudaMemcpyHostToDevice));
  TraceSink tr;
  tr.tasks = dt; tr.task_cap = task_cap; tr.n_tasks = cnts; tr.edge_pred = dep; tr.edge_succ = des;
  tr.edge_cap = edge_cap; tr.n_edges = cnts + 1;
  size_t smem = pr->lay.global_all    ? pr->lay.hot_bytes
                : pr->lay.warp_global ? pr->lay.tab_bytes + pr->lay.hot_bytes
                                      : pr->lay.tab_bytes + pr->lay.warp_bytes;
  k_simulate_trace<<<1, 32, smem>>>(pr->P, pr->lay, pr->d_map, pr->d_asg, scr, tr, dmk, err + 2, err);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  int h[2], he[3];
  CK(cudaMemcpy(h, cnts, 2 * sizeof(int), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(he, err, 3 * sizeof(int), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(makespan, dmk, sizeof(double), cudaMemcpyDeviceToHost));
  *n_tasks = h[0];
  *n_edges = h[1];
  *status = he[2];
  err_devices[0] = he[0];
  err_devices[1] = he[1];
  if (h[0] <= task_cap && h[0] > 0) CK(cudaMemcpy(tasks, dt, sizeof(ps_trace_task) * h[0], cudaMemcpyDeviceToHost));
  if (h[1] <= edge_cap && h[1] > 0) {
    CK(cudaMemcpy(edge_pred, dep, sizeof(int32_t) * h[1], cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(edge_succ_key, des, sizeof(uint64_t) * h[1], cudaMemcpyDeviceToHost));
  }
  cudaFree(scr); cudaFree(dt); cudaFree(dep); cudaFree(des); cudaFree(cnts); cudaFree(err); cudaFree(dmk);
  if (h[0] > task_cap || h[1] > edge_cap) return fail(PS_ERR_CAPACITY, "trace buffers too small");
  return PS_OK;
}


int ps_simulate_explicit(int n_tasks, int n_queues, const int32_t *queue, const double *exe, const uint64_t *rank,
                         const int32_t *succ_off, const int32_t *succ, double *ready, double *start, double *end,
                         int32_t *order, double *makespan, int32_t *status, int device) {
  if (n_tasks < 0 || n_queues < 0) return fail(PS_ERR_INVALID, "bad arguments");
  CK(cudaSetDevice(device));
  int n = n_tasks > 0 ? n_tasks : 1, nq = n_queues > 0 ? n_queues : 1;
  int n_edges = n_tasks > 0 ? succ_off[n_tasks] : 0;
  std::vector<int> indeg(n, 0);
  for (int e = 0; e < n_edges; ++e) {
    if (succ[e] < 0 || succ[e] >= n_tasks) return fail(PS_ERR_INVALID, "successor out of range");
    indeg[succ[e]]++;
  }
  for (int t = 0; t < n_tasks; ++t)
    if (queue[t] < 0 || queue[t] >= n_queues) return fail(PS_ERR_INVALID, "queue out of range");
  std::vector<void *> tmp;
  auto alloc = [&](size_t bytes) -> void * { void *p = nullptr; if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr; tmp.push_back(p); return p; };
  int *dq = (int *)alloc(n * 4), *dso = (int *)alloc((n + 1) * 4), *ds = (int *)alloc((n_edges + 1) * 4);
  int *dind = (int *)alloc(n * 4), *drem = (int *)alloc(n * 4), *dord = (int *)alloc(n * 4), *draux = (int *)alloc(n * 4);
  double *dexe = (double *)alloc(n * 8), *drd = (double *)alloc(n * 8), *dst = (double *)alloc(n * 8),
         *den = (double *)alloc(n * 8), *dqc = (double *)alloc(nq * 8), *dmk = (double *)alloc(8);
  unsigned long long *drank = (unsigned long long *)alloc(n * 8), *drhi = (unsigned long long *)alloc(n * 8),
                     *drlo = (unsigned long long *)alloc(n * 8);
  int *dstat = (int *)alloc(4);
  for (void *p : tmp) if (!p) { for (void *q : tmp) cudaFree(q); return fail(PS_ERR_CUDA, "cudaMalloc failed"); }
  int rc = PS_OK;
  do {
    if (n_tasks) {
      if (cudaMemcpy(dq, queue, n_tasks * 4, cudaMemcpyHostToDevice) ||
          cudaMemcpy(dso, succ_off, (n_tasks + 1) * 4, cudaMemcpyHostToDevice) ||
          (n_edges && cudaMemcpy(ds, succ, n_edges * 4, cudaMemcpyHostToDevice)) ||
          cudaMemcpy(dind, indeg.data(), n_tasks * 4, cudaMemcpyHostToDevice) ||
          cudaMemcpy(dexe, exe, n_tasks * 8, cudaMemcpyHostToDevice) ||
          cudaMemcpy(drank, rank, n_tasks * 8, cudaMemcpyHostToDevice)) { rc = fail(PS_ERR_CUDA, "copy failed"); break; }
    }
    k_simulate_explicit<<<1, 32>>>(n_tasks, nq, dq, dexe, drank, dso, ds, dind, drd, dst, den, dord, drem, dqc, drhi,
                                   drlo, draux, dstat, dmk);
    if (cudaDeviceSynchronize() != cudaSuccess) { rc = fail(PS_ERR_CUDA, cudaGetErrorString(cudaGetLastError())); break; }
    if (n_tasks && (cudaMemcpy(ready, drd, n_tasks * 8, cudaMemcpyDeviceToHost) ||
                    cudaMemcpy(start, dst, n_tasks * 8, cudaMemcpyDeviceToHost) ||
                    cudaMemcpy(end, den, n_tasks * 8, cudaMemcpyDeviceToHost) ||
                    cudaMemcpy(order, dord, n_tasks * 4, cudaMemcpyDeviceToHost))) { rc = fail(PS_ERR_CUDA, "copy back failed"); break; }
    cudaMemcpy(makespan, dmk, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(status, dstat, 4, cudaMemcpyDeviceToHost);
  } while (0);
  for (void *p : tmp) cudaFree(p);
  return rc;
}

int ps_mcmc_create(ps_problem *pr, const ps_mcmc_params *params, int n, const int32_t *init_map,
                   const uint8_t *init_assign, const uint64_t *seeds, const uint32_t *mt_state, ps_mcmc **out) {
  if (!pr || !params || n <= 0 || !out) return fail(PS_ERR_INVALID, "bad arguments");
  if (params->rng_mode == PS_RNG_MT19937 && !mt_state) return fail(PS_ERR_INVALID, "MT19937 mode needs mt_state");
  CK(cudaSetDevice(pr->device));
  ps_mcmc *m = new ps_mcmc();
  memset(m, 0, sizeof(*m));
  m->prob = pr;
  m->n = n;
  m->params = *params;
  const DevProb &P = pr->P;
  if (pr->spare.maps && pr->spare.n >= n) {
    m->maps = pr->spare.maps; m->best_maps = pr->spare.best_maps; m->asgs = pr->spare.asgs;
    m->best_asgs = pr->spare.best_asgs; m->st = (ChainState *)pr->spare.st; m->d_best = pr->spare.d_best;
    m->d_bestc = pr->spare.d_bestc; m->cap_n = pr->spare.n;
    pr->spare.maps = nullptr; pr->spare.n = 0;
  } else {
    CK(cudaMalloc(&m->maps, (size_t)n * P.n_ops * sizeof(int)));
    CK(cudaMalloc(&m->best_maps, (size_t)n * P.n_ops * sizeof(int)));
    CK(cudaMalloc(&m->asgs, (size_t)n * P.n_slots));
    CK(cudaMalloc(&m->best_asgs, (size_t)n * P.n_slots));
    CK(cudaMalloc(&m->st, (size_t)n * sizeof(ChainState)));
    CK(cudaMalloc(&m->d_best, sizeof(double)));
    CK(cudaMalloc(&m->d_bestc, sizeof(int)));
    m->cap_n = n;
  }
  {
    size_t want = (size_t)n * gslice_bytes(P, pr->lay);
    if (pr->mcmc_scratch && pr->mcmc_scratch_bytes >= want) {  // reuse: repeated create/run/destroy cycles
      m->scratch = pr->mcmc_scratch;
      pr->mcmc_scratch = nullptr;
      m->scratch_bytes = pr->mcmc_scratch_bytes;
    } else {
      CK(cudaMalloc(&m->scratch, want));
      m->scratch_bytes = want;
    }
  }
  CK(cudaMemcpy(m->maps, init_map, (size_t)n * P.n_ops * sizeof(int), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(m->asgs, init_assign, (size_t)n * P.n_slots, cudaMemcpyHostToDevice));
  std::vector<ChainState> st(n);
  for (int i = 0; i < n; ++i) {
    ChainState &c = st[i];
    memset(&c, 0, sizeof c);
    c.key = seeds[i];
    c.ctr = 0;
    c.bpos = 4;
    c.mti = params->rng_mode == PS_RNG_MT19937 ? (int)mt_state[(size_t)i * 625 + 624] : 624;
  }
  CK(cudaMemcpy(m->st, st.data(), (size_t)n * sizeof(ChainState), cudaMemcpyHostToDevice));
  if (params->rng_mode == PS_RNG_MT19937) {
    std::vector<unsigned> words((size_t)n * 624);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < 624; ++j) words[(size_t)i * 624 + j] = mt_state[(size_t)i * 625 + j];
    CK(cudaMalloc(&m->mt, words.size() * sizeof(unsigned)));
    CK(cudaMemcpy(m->mt, words.data(), words.size() * sizeof(unsigned), cudaMemcpyHostToDevice));
  }
  if (params->record_trace && params->trace_capacity > 0) {
    CK(cudaMalloc(&m->trace_cand, (size_t)n * params->trace_capacity * sizeof(double)));
    CK(cudaMalloc(&m->trace_ok, (size_t)n * params->trace_capacity));
  }
  {
    // delta evaluation: snapshots per chain (two copies per index), first
    // rounds, in-degrees.  Off when some task can take zero time, when asked
    // (params->delta == 0 / PS_NO_DELTA), or when fewer than 4 snapshot indices
    // fit in a quarter of the device memory.
    size_t sb = snap_layout(P).total;
    if (!pr->total_mem) {
      size_t free_b = 0;
      CK(cudaMemGetInfo(&free_b, &pr->total_mem));
    }
    const size_t total_b = pr->total_mem;
    size_t budget = total_b / 4;
    if (const char *e = getenv("PS_SNAP_BUDGET_GB")) budget = std::min(total_b / 3, (size_t)atof(e) * ((size_t)1 << 30));
    // snapshot indices per chain: more resume points vs more snapshot writes per
    // simulation (measured on Inception-v3 4x4: full-iteration 8 > 12 > 24,
    // forward 12 > 8 > 24)
    size_t want_ns = P.full ? 8 : 12;
    if (const char *e = getenv("PS_NSNAP")) want_ns = (size_t)std::max(4, std::min(31, atoi(e)));
    int ns = (int)std::min<size_t>(want_ns, budget / ((size_t)n * 2 * sb));
    bool on = params->delta != 0 && P.min_exe > 0.0 && ns >= 4 && !getenv("PS_NO_DELTA");
    if (on) {
      m->db.nsnap = ns;
      if (const char *e = getenv("PS_DELTA_EXP")) m->db.exp = atoi(e);
      if (const char *e = getenv("PS_DELTA_TRACE")) {
        m->db.dbg_cap = atoi(e);
        CK(cudaMalloc(&m->db.dbg, (size_t)n * m->db.dbg_cap * 8 * sizeof(int)));
        CK(cudaMemset(m->db.dbg, 0xff, (size_t)n * m->db.dbg_cap * 8 * sizeof(int)));
      }
      m->db.snap_bytes = sb;
      if (pr->spare_delta.cd && pr->spare_delta.n == n && pr->spare_delta.ns == ns) {
        // reuse (create / run / destroy cycles allocate nothing)
        m->db.cd = pr->spare_delta.cd; m->db.snaps = pr->spare_delta.snaps; m->db.frb = pr->spare_delta.frb;
        m->db.indeg = pr->spare_delta.indeg;
        pr->spare_delta.cd = nullptr; pr->spare_delta.n = 0;
      } else {
        CK(cudaMalloc(&m->db.cd, (size_t)n * sizeof(ChainDelta)));
        CK(cudaMalloc(&m->db.snaps, (size_t)n * 2 * ns * sb));
        CK(cudaMalloc(&m->db.frb, (size_t)n * 4 * P.n_ops * sizeof(int)));
        CK(cudaMalloc(&m->db.indeg, (size_t)n * (ns + 1) * snap_counters_pad(P) * sizeof(unsigned short)));
      }
      CK(cudaMemset(m->db.cd, 0, (size_t)n * sizeof(ChainDelta)));
      CK(cudaMemset(m->db.frb, 0x7f, (size_t)n * 4 * P.n_ops * sizeof(int)));  // "never ran"
      CK(cudaMemset(m->db.indeg, 0, (size_t)n * (ns + 1) * snap_counters_pad(P) * sizeof(unsigned short)));
    }
  }
  *out = m;
  return PS_OK;
}

static int mcmc_launch(ps_mcmc *m, int proposals, unsigned long long budget_ns, void *stream, Given gv = Given{}) {
  if (!m || proposals < 0) return fail(PS_ERR_INVALID, "bad arguments");
  ps_problem *pr = m->prob;
  CK(cudaSetDevice(pr->device));
  int wpb = pr->wpb;
  int blocks = (m->n + wpb - 1) / wpb;
  size_t smem = pr->smem_per_block;
  auto km = mcmc_kernel(!pr->simple ? 0 : pr->P.full ? 1 : 2, m->db.cd != nullptr, pr->wide);
  // One warp per chain: chains beyond one resident wave wait for a block to
  // finish (the block scheduler balances fast and slow chains).  PS_MCMC_MUX caps
  // the grid at one resident wave instead, each warp running its chains in turn
  // with the time box split among them -- measured slower on wide problems
  // (NMT-40, 4096 chains: 10k vs 42k proposals per 300 ms step), where a warp
  // with slow chains holds the whole launch.
  if (getenv("PS_MCMC_MUX")) {
    if (m->max_blocks <= 0) {
      int occ = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, km, wpb * 32, smem));
      m->max_blocks = std::max(1, occ) * pr->sm_count;
    }
    blocks = std::min(blocks, m->max_blocks);
  }
  km<<<blocks, wpb * 32, smem, (cudaStream_t)stream>>>(
      pr->P, pr->lay, m->n, proposals, m->params.rng_mode, m->params.beta_given, m->params.beta, m->params.ln10, m->maps,
      m->asgs, m->best_maps, m->best_asgs, m->st, m->mt, m->trace_cand, m->trace_ok,
      m->params.record_trace && !gv.op ? m->params.trace_capacity : 0, m->scratch, budget_ns, m->db, gv);
  CK(cudaGetLastError());
  return PS_OK;
}

int ps_mcmc_run(ps_mcmc *m, int proposals, void *stream) { return mcmc_launch(m, proposals, 0ull, stream); }

int ps_mcmc_run_budget(ps_mcmc *m, int max_proposals, uint64_t budget_ns, void *stream) {
  return mcmc_launch(m, max_proposals, (unsigned long long)budget_ns, stream);
}

int ps_delta_batch(ps_mcmc *m, const int32_t *op, const int32_t *map_local, const uint8_t *assign, int assign_stride,
                   const uint8_t *commit, double *makespan_out, int32_t *status_out, int flags, void *stream) {
  if (!m || !op || !map_local || !assign || assign_stride <= 0 || !makespan_out || !status_out)
    return fail(PS_ERR_INVALID, "bad arguments");
  ps_problem *pr = m->prob;
  const DevProb &P = pr->P;
  CK(cudaSetDevice(pr->device));
  const int n = m->n;
  Given gv{};
  if (flags == PS_DEVICE_PTRS) {
    gv = Given{op, map_local, assign, commit, assign_stride, makespan_out, status_out};
    return mcmc_launch(m, 1, 0ull, stream, gv);
  }
  // host arguments: validate, stage in the handle's buffers, launch, read back
  for (int i = 0; i < n; ++i) {
    if (op[i] < 0) continue;
    const int nm = op[i] < P.n_ops ? pr->h_map_off[op[i] + 1] - pr->h_map_off[op[i]] : 0;
    if (op[i] >= P.n_ops || map_local[i] < 0 || map_local[i] >= nm)
      return fail(PS_ERR_INVALID, "op or map index out of range");
    const int size = pr->h_map_size[pr->h_map_off[op[i]] + map_local[i]];
    if (size > assign_stride) return fail(PS_ERR_INVALID, "assign_stride is smaller than the map's task count");
    for (int k = 0; k < size; ++k)
      if (assign[(size_t)i * assign_stride + k] >= P.n_dev) return fail(PS_ERR_INVALID, "device index out of range");
  }
  size_t need = (size_t)n * (4 + 4 + 1 + 8 + 4) + (size_t)n * assign_stride + 64;
  if (need > m->given_bytes) {
    cudaFree(m->given);
    m->given = nullptr;
    CK(cudaMalloc(&m->given, need));
    m->given_bytes = need;
  }
  char *b = m->given;
  double *dmk = (double *)b; b += 8 * (size_t)n;
  int *dop = (int *)b; b += 4 * (size_t)n;
  int *dmap = (int *)b; b += 4 * (size_t)n;
  int *dst = (int *)b; b += 4 * (size_t)n;
  unsigned char *dcm = (unsigned char *)b; b += n;
  unsigned char *dasg = (unsigned char *)b;
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaMemcpyAsync(dop, op, 4 * (size_t)n, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(dmap, map_local, 4 * (size_t)n, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(dasg, assign, (size_t)n * assign_stride, cudaMemcpyHostToDevice, s));
  if (commit) CK(cudaMemcpyAsync(dcm, commit, (size_t)n, cudaMemcpyHostToDevice, s));
  gv = Given{dop, dmap, dasg, commit ? dcm : nullptr, assign_stride, dmk, dst};
  int rc = mcmc_launch(m, 1, 0ull, stream, gv);
  if (rc != PS_OK) return rc;
  CK(cudaMemcpyAsync(makespan_out, dmk, 8 * (size_t)n, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(status_out, dst, 4 * (size_t)n, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  for (int i = 0; i < n; ++i)
    if (op[i] < 0) { makespan_out[i] = 0.0; status_out[i] = PS_STATUS_OK; }
  return PS_OK;
}

int ps_mcmc_read(ps_mcmc *m, ps_chain_summary *summary, int32_t *best_map, uint8_t *best_assign, double *trace_cand,
                 uint8_t *trace_ok) {
  ps_problem *pr = m->prob;
  CK(cudaSetDevice(pr->device));
  CK(cudaDeviceSynchronize());
  std::vector<ChainState> st(m->n);
  CK(cudaMemcpy(st.data(), m->st, (size_t)m->n * sizeof(ChainState), cudaMemcpyDeviceToHost));
  if (summary) {
    for (int i = 0; i < m->n; ++i) {
      ps_chain_summary &s = summary[i];
      s.initial_cost = st[i].initial; s.best_cost = st[i].best; s.cost = st[i].cost; s.beta = st[i].beta;
      s.proposals = st[i].proposals; s.accepted = st[i].accepted; s.status = st[i].status;
      s.err_a = st[i].err_a; s.err_b = st[i].err_b; s.last_op = st[i].last_op;
      s.rounds_run = s.rounds_reused = 0;
    }
    if (m->db.cd) {
      std::vector<ChainDelta> cd(m->n);
      CK(cudaMemcpy(cd.data(), m->db.cd, (size_t)m->n * sizeof(ChainDelta), cudaMemcpyDeviceToHost));
      for (int i = 0; i < m->n; ++i) {
        summary[i].rounds_run = cd[i].rounds_run;
        summary[i].rounds_reused = cd[i].rounds_reused;
      }
    }
  }
  if (best_map) CK(cudaMemcpy(best_map, m->best_maps, (size_t)m->n * pr->P.n_ops * sizeof(int), cudaMemcpyDeviceToHost));
  if (best_assign) CK(cudaMemcpy(best_assign, m->best_asgs, (size_t)m->n * pr->P.n_slots, cudaMemcpyDeviceToHost));
  size_t tc = (size_t)m->n * m->params.trace_capacity;
  if (trace_cand && m->trace_cand) CK(cudaMemcpy(trace_cand, m->trace_cand, tc * sizeof(double), cudaMemcpyDeviceToHost));
  if (trace_ok && m->trace_ok) CK(cudaMemcpy(trace_ok, m->trace_ok, tc, cudaMemcpyDeviceToHost));
  return PS_OK;
}


int ps_mcmc_stop(ps_mcmc *m, const uint8_t *stop) {
  if (!m || !stop) return fail(PS_ERR_INVALID, "bad arguments");
  CK(cudaSetDevice(m->prob->device));
  CK(cudaDeviceSynchronize());
  std::vector<ChainState> st(m->n);
  CK(cudaMemcpy(st.data(), m->st, (size_t)m->n * sizeof(ChainState), cudaMemcpyDeviceToHost));
  for (int i = 0; i < m->n; ++i)
    if (stop[i] && st[i].status == PS_STATUS_OK) st[i].status = PS_STATUS_STOPPED;
  CK(cudaMemcpy(m->st, st.data(), (size_t)m->n * sizeof(ChainState), cudaMemcpyHostToDevice));
  return PS_OK;
}


int ps_mcmc_chains(const ps_mcmc *m) { return m ? m->n : 0; }

// debug: raw per-chain delta bookkeeping (stride, nvalid, cur, bad, fsel, pad,
// rounds_run, rounds_reused) -- 40 bytes per chain; PS_ERR_INVALID when delta is off
int ps_debug_delta_state(ps_mcmc *m, void *out) {
  if (!m || !m->db.cd) return fail(PS_ERR_INVALID, "delta evaluation is off for this handle");
  CK(cudaSetDevice(m->prob->device));
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(out, m->db.cd, (size_t)m->n * sizeof(ChainDelta), cudaMemcpyDeviceToHost));
  return PS_OK;
}

// debug (PS_DELTA_TRACE=cap): per chain and proposal (op, resume index, nvalid, rounds, stride, last, bad, fsel),
// then the chain's first-index buffers [2][2][n_ops]
int ps_debug_delta_trace(ps_mcmc *m, int32_t *out, int32_t *frb) {
  if (!m || !m->db.dbg) return fail(PS_ERR_INVALID, "PS_DELTA_TRACE was not set");
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(out, m->db.dbg, (size_t)m->n * m->db.dbg_cap * 8 * sizeof(int), cudaMemcpyDeviceToHost));
  if (frb) CK(cudaMemcpy(frb, m->db.frb, (size_t)m->n * 4 * m->prob->P.n_ops * sizeof(int), cudaMemcpyDeviceToHost));
  return PS_OK;
}

int ps_debug_tcyc(long long *out) {
#ifdef PS_TCYC
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpyFromSymbol(out, g_tc, sizeof(long long) * 4096 * 16));
  int ns = 0;
  CK(cudaMemcpyFromSymbol(&ns, g_tc_sim, sizeof(int)));
  fprintf(stderr, "[parasim] tcyc: %d simulations on warp 0\n", ns);
  return PS_OK;
#else
  (void)out;
  return fail(PS_ERR_INVALID, "built without PS_TCYC");
#endif
}

int ps_debug_phases(unsigned long long *out, int reset) {
#ifdef PS_PHASES
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpyFromSymbol(out, g_phase, sizeof(unsigned long long) * PH_N));
  if (reset) {
    unsigned long long z[PH_N] = {0};
    CK(cudaMemcpyToSymbol(g_phase, z, sizeof z));
  }
  return PS_OK;
#else
  (void)out; (void)reset;
  return fail(PS_ERR_INVALID, "built without PS_PHASES");
#endif
}

int ps_mcmc_read_state(ps_mcmc *m, int32_t *maps, uint8_t *assign) {
  if (!m) return fail(PS_ERR_INVALID, "bad arguments");
  ps_problem *pr = m->prob;
  CK(cudaSetDevice(pr->device));
  CK(cudaDeviceSynchronize());
  if (maps) CK(cudaMemcpy(maps, m->maps, (size_t)m->n * pr->P.n_ops * sizeof(int), cudaMemcpyDeviceToHost));
  if (assign) CK(cudaMemcpy(assign, m->asgs, (size_t)m->n * pr->P.n_slots, cudaMemcpyDeviceToHost));
  return PS_OK;
}

int ps_mcmc_best(ps_mcmc *m, double *best_cost, int32_t *best_chain) {
  CK(cudaSetDevice(m->prob->device));
  k_best<<<1, 1024>>>(m->st, m->n, m->d_best, m->d_bestc);
  CK(cudaGetLastError());
  CK(cudaMemcpy(best_cost, m->d_best, sizeof(double), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(best_chain, m->d_bestc, sizeof(int), cudaMemcpyDeviceToHost));
  return PS_OK;
}

void ps_mcmc_destroy(ps_mcmc *m) {
  if (!m) return;
  cudaSetDevice(m->prob->device);
  ps_problem *pr = m->prob;
  cudaDeviceSynchronize();  // kept buffers must be idle before a later handle reuses them (cudaFree would sync too)
  if (!pr->spare.maps) {  // keep the chain buffers for the problem's next handle
    pr->spare.n = m->cap_n; pr->spare.maps = m->maps; pr->spare.best_maps = m->best_maps; pr->spare.asgs = m->asgs;
    pr->spare.best_asgs = m->best_asgs; pr->spare.st = m->st; pr->spare.d_best = m->d_best;
    pr->spare.d_bestc = m->d_bestc;
  } else {
    cudaFree(m->maps); cudaFree(m->best_maps); cudaFree(m->asgs); cudaFree(m->best_asgs); cudaFree(m->st);
    cudaFree(m->d_best); cudaFree(m->d_bestc);
  }
  cudaFree(m->mt); cudaFree(m->trace_cand); cudaFree(m->trace_ok); cudaFree(m->given);
  cudaFree(m->db.dbg);
  if (m->db.cd && !pr->spare_delta.cd) {  // keep the delta buffers for the problem's next handle
    pr->spare_delta.n = m->n; pr->spare_delta.ns = m->db.nsnap; pr->spare_delta.cd = m->db.cd;
    pr->spare_delta.snaps = m->db.snaps; pr->spare_delta.frb = m->db.frb; pr->spare_delta.indeg = m->db.indeg;
  } else {
    cudaFree(m->db.cd); cudaFree(m->db.snaps); cudaFree(m->db.frb); cudaFree(m->db.indeg);
  }
  if (m->scratch) {  // keep the largest chain scratch for the problem's next handle
    if (m->scratch_bytes >= m->prob->mcmc_scratch_bytes) {
      cudaFree(m->prob->mcmc_scratch);
      m->prob->mcmc_scratch = m->scratch;
      m->prob->mcmc_scratch_bytes = m->scratch_bytes;
    } else {
      cudaFree(m->scratch);
    }
  }
  delete m;
}

}  // extern "C"
