/*
 * parasim.h -- C ABI of libparasim_cuda.so, the B200 strategy-evaluation path.
 *
 * The reference (pkg/src/parasim, pure Python) has no FFI; its boundary is the
 * Python API.  These entry points are what that API binds (via ctypes, see
 * INTEGRATION.md); each names the reference interface it replaces:
 *
 *   ps_problem_create      lowering of (OperatorGraph, DeviceTopology, CostProfile, mode)
 *                          into device tables, incl. the region-overlap tables
 *                          _wire_pair derives per task pair
 *                          (reference taskgraph.py:154-222, partition.py:117-211,
 *                           cost.py:105-130)
 *   ps_simulate_batch      build_task_graph + full_simulate, batched over strategies
 *                          (reference taskgraph.py:276-292, simulate.py:68-117)
 *   ps_simulate_trace      the same for one strategy, returning every task
 *                          (origin key, queue, exe, bytes, ready/start/end) and every
 *                          dependency edge -- what TaskGraph/timeline_table expose
 *                          (reference taskgraph.py:57-110,424-443)
 *   ps_mcmc_create/run     mcmc_search's per-chain loop with polish=False, one warp
 *                          per chain (reference search.py:89-115,170-271)
 *
 * Conventions: every call returns PS_OK or a PS_ERR_* code and records a
 * message for ps_last_error() (thread-local).  Host pointers unless the
 * PS_DEVICE_PTRS flag says otherwise.  All times are IEEE fp64 seconds and
 * reproduce the reference bit for bit ("Exactness").
 * One ps_problem per (GPU, host thread); calls on one handle are not
 * concurrent; work is ordered on the given stream (NULL = legacy stream).
 */
#ifndef PARASIM_H
#define PARASIM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PS_ABI_VERSION 3
#define PS_MAXDIM 5

enum {
  PS_OK = 0,
  PS_ERR_INVALID = 1,   /* bad descriptor / arguments (ValueError in the reference) */
  PS_ERR_NO_ROUTE = 2,  /* a transfer needs a missing link (NoRouteError, taskgraph.py:148-152) */
  PS_ERR_CYCLE = 3,     /* a task never became ready (SimulationError, simulate.py:108-112) */
  PS_ERR_CAPACITY = 4,  /* ready set exceeded the configured capacity */
  PS_ERR_CUDA = 5
};

/* per-candidate status words written by the batch calls */
#define PS_STATUS_OK 0
#define PS_STATUS_NO_ROUTE 2
#define PS_STATUS_CAPACITY 4
#define PS_STATUS_STOPPED 9 /* chain halted by ps_mcmc_stop (stagnation / budget) */

enum { PS_HOST_PTRS = 0, PS_DEVICE_PTRS = 1 };
enum { PS_RNG_PHILOX = 0, PS_RNG_MT19937 = 1 };

/* need-descriptor modes: how a source dim's needed range follows the dst block
 * (partition.py:162-211) */
enum { PS_NEED_FULL = 0, PS_NEED_IDENT = 1, PS_NEED_WINDOW = 2, PS_NEED_CONCAT = 3 };
#define PS_NEED_STRIDE 8 /* ints per (edge, src dim): mode,out_dim,extent,kernel,stride,pad,offset,0 */

typedef struct ps_problem_desc {
  int32_t abi_version;
  int32_t n_ops, n_devices, n_kinds, n_links, n_pairs, n_maps, mode_full;
  int32_t n_slots;         /* sum over ops of the largest map size ("NF") */
  int32_t ready_capacity;  /* ready-set entries per simulating warp (0 = default) */
  /* devices (sorted by id) and links */
  const int32_t *dev_kind; /* [n_devices] device-kind index */
  const int32_t *link_of;  /* [n_devices^2] link index, -1 = no connection */
  const double *link_bw;   /* [n_links] bytes/s */
  const double *link_lat;  /* [n_links] s */
  /* ops in sorted-id order (index == rank in the origin ordering) */
  const int32_t *op_ndim;       /* [n_ops] */
  const int64_t *op_dim;        /* [n_ops*5] output extents */
  const int32_t *op_esize;      /* [n_ops] output element size */
  const int32_t *op_param_mask; /* [n_ops] bit i: output dim i is a parameter dim; -1: no sync */
  const int32_t *op_map_off;    /* [n_ops+1] */
  const int32_t *op_nmaps_enum; /* [n_ops] leading maps that proposals draw from */
  const int32_t *op_slot_off;   /* [n_ops+1] first slot per op */
  const int32_t *slot_op;       /* [n_slots] owning op */
  const int32_t *op_in_off, *op_in_pairs;   /* CSR: pairs whose dst is the op */
  const int32_t *op_out_off, *op_out_pairs; /* CSR: pairs whose src is the op */
  /* degree maps */
  const int32_t *map_deg;  /* [n_maps*5] degree per output dim (1 beyond ndim) */
  const int32_t *map_size; /* [n_maps] tasks */
  const double *exe_fwd;   /* [n_maps*n_kinds] cost-table lookups */
  const double *exe_bwd;   /* [n_maps*n_kinds] exe_fwd * backward_multiplier */
  const double *map_shard; /* [n_maps] parameter bytes per shard (0 without sync) */
  const int32_t *map_ngroups; /* [n_maps] parameter shards */
  /* op pairs (distinct (src,dst) in tensor order) */
  const int32_t *pair_src, *pair_dst; /* [n_pairs] */
  const int32_t *pair_need_off;       /* [n_pairs+1] tensor edges per pair */
  const int32_t *need;                /* [n_edges*5*PS_NEED_STRIDE] */
  const int32_t *combo_off;           /* [n_pairs+1] (src map, dst map) combos per pair */
  const int32_t *combo_row_off;       /* [n_combos+1] prefix of src map sizes */
  const int32_t *combo_col_off;       /* [n_combos+1] prefix of dst map sizes */
  double backward_multiplier;         /* exe_bwd == exe_fwd * this (cost.py:111) */
} ps_problem_desc;

typedef struct ps_problem_info {
  int64_t n_entries;   /* (k,l) overlap entries over all combos */
  int64_t n_combos;
  int32_t n_queues;    /* devices + links */
  int32_t n_slots;
  int32_t ready_capacity;
  int32_t warps_per_block;
  int64_t device_bytes; /* resident static tables */
  int32_t shared_counters;       /* per-warp task counters kept in shared memory */
  int32_t resident_warps_per_sm; /* candidates / chains resident per SM */
  int32_t smem_per_block;
  int32_t reserved_;
} ps_problem_info;

typedef struct ps_problem ps_problem;

int ps_problem_create(const ps_problem_desc *desc, int device, ps_problem **out);
void ps_problem_destroy(ps_problem *prob);
int ps_problem_info_get(const ps_problem *prob, ps_problem_info *out);

/* Overlap entries of one (pair, src map, dst map) combo, sorted by (k, l):
 * the transfer volumes _wire_pair computes (taskgraph.py:168-195). */
int ps_combo_entries(ps_problem *prob, int pair, int src_map, int dst_map, int cap,
                     int32_t *k_out, int32_t *l_out, int64_t *bytes_out, int *n_out);

/* Full evaluation of n strategies.  map_local: [n][n_ops] local map index;
 * assign: [n][n_slots] device index per task slot (op_slot_off layout).
 * makespan_out/status_out: [n].  flags: PS_HOST_PTRS or PS_DEVICE_PTRS. */
int ps_simulate_batch(ps_problem *prob, const int32_t *map_local, const uint8_t *assign, int n,
                      double *makespan_out, int32_t *status_out, int flags, void *stream);

/* As ps_simulate_batch, plus op_min_end_out [n][n_ops]: the earliest end of each
 * op's forward tasks (the bound exhaustive_optimal prunes with, search.py:380-381). */
int ps_simulate_batch_ex(ps_problem *prob, const int32_t *map_local, const uint8_t *assign, int n,
                         double *makespan_out, int32_t *status_out, double *op_min_end_out, int flags,
                         void *stream);

/* One strategy with the full timeline.  Tasks are reported in pop order. */
typedef struct ps_trace_task {
  uint64_t key;   /* packed origin: kind<<61 | a<<45 | b<<29 | c<<14 | d */
  int32_t queue;  /* device index, or n_devices + link index */
  int32_t aux;
  double exe, nbytes, ready, start, end;
} ps_trace_task;

int ps_simulate_trace(ps_problem *prob, const int32_t *map_local, const uint8_t *assign,
                      int task_cap, ps_trace_task *tasks, int *n_tasks, int edge_cap,
                      int32_t *edge_pred, uint64_t *edge_succ_key, int *n_edges, double *makespan,
                      int32_t *status, int32_t *err_devices /* [2] */);


/* Explicit task graph (hand-built TaskGraphs; the oracle_simulate path):
 * n_tasks tasks with queue, exe and a total order rank of their origins, CSR
 * successors.  Outputs per task ready/start/end and the pop order.  status:
 * PS_STATUS_OK, or 3 when some task never became ready (a cycle). */
int ps_simulate_explicit(int n_tasks, int n_queues, const int32_t *queue, const double *exe, const uint64_t *rank,
                         const int32_t *succ_off, const int32_t *succ, double *ready, double *start, double *end,
                         int32_t *order, double *makespan, int32_t *status, int device);

/* MCMC (search.py:170-271 with polish=False), one warp per chain. */
typedef struct ps_mcmc_params {
  int32_t rng_mode;       /* PS_RNG_PHILOX or PS_RNG_MT19937 */
  int32_t beta_given;     /* 0: ln10 / (0.05 * initial cost) per chain */
  double beta;
  double ln10;            /* math.log(10.0) of the host */
  int32_t record_trace;   /* keep (cand, accepted) per proposal */
  int32_t trace_capacity; /* ring of proposals recorded per chain: proposal i lands in slot i % capacity */
  int32_t delta;          /* 1: checkpointed delta evaluation of proposals (update_task_graph +
                             delta_simulate, taskgraph.py:309-418, simulate.py:120-210); 0: each
                             proposal re-simulates from time zero.  Same results either way. */
  int32_t reserved_;
} ps_mcmc_params;

typedef struct ps_chain_summary {
  double initial_cost, best_cost, cost, beta;
  int64_t proposals, accepted;
  int32_t status;         /* PS_STATUS_* of the chain */
  int32_t err_a, err_b;   /* device pair of a no-route failure */
  int32_t last_op;        /* op of the most recent proposal */
  int64_t rounds_run;     /* simulation rounds executed (delta evaluation) */
  int64_t rounds_reused;  /* rounds skipped by resuming from a snapshot */
} ps_chain_summary;

typedef struct ps_mcmc ps_mcmc;

/* init_map: [n][n_ops], init_assign: [n][n_slots], seeds: [n] (random.Random seed per
 * chain), mt_state: [n][625] CPython MT19937 state words + position (MT mode, else NULL). */
int ps_mcmc_create(ps_problem *prob, const ps_mcmc_params *params, int n_chains,
                   const int32_t *init_map, const uint8_t *init_assign, const uint64_t *seeds,
                   const uint32_t *mt_state, ps_mcmc **out);
/* Advance every live chain by `proposals` proposals (first call also scores
 * the initial strategies).  Device-resident; asynchronous on `stream`. */
int ps_mcmc_run(ps_mcmc *m, int proposals, void *stream);
/* Time-boxed segment: every chain proposes until `max_proposals` or until
 * budget_ns of device time (%globaltimer) has passed since the launch began,
 * checked between proposals -- no warp idles behind a slow chain. */
int ps_mcmc_run_budget(ps_mcmc *m, int max_proposals, uint64_t budget_ns, void *stream);
/* Delta evaluation of given single-op changes on resident strategies: the
 * B200 form of update_task_graph + delta_simulate (reference taskgraph.py:309-418,
 * simulate.py:120-210; SURVEY 8b "ps_delta_batch").  The handle's chains hold
 * the current strategies (ps_mcmc_create's initial ones, or the last committed
 * change); for chain i, op op[i] takes local map map_local[i] and the devices
 * assign[i * assign_stride + k], k < that map's task count.  The changed strategy
 * is simulated from the chain's last snapshot before the change's first
 * dependent round (bit-identical to a full simulation) and its makespan written
 * to makespan_out[i], with status_out[i] = PS_STATUS_*.  commit[i] != 0 (or
 * commit == NULL) keeps the change -- the chain's strategy, cost and snapshots
 * move to it -- else the previous strategy is restored.  op[i] < 0 leaves chain
 * i alone (makespan 0).  A chain whose change fails (no route) stays failed.
 * The first call on a handle also scores the initial strategies.  flags:
 * PS_HOST_PTRS (arguments checked, synchronous) or PS_DEVICE_PTRS (asynchronous
 * on `stream`, unchecked). */
int ps_delta_batch(ps_mcmc *m, const int32_t *op, const int32_t *map_local, const uint8_t *assign,
                   int assign_stride, const uint8_t *commit, double *makespan_out, int32_t *status_out,
                   int flags, void *stream);
int ps_mcmc_read(ps_mcmc *m, ps_chain_summary *summary, int32_t *best_map, uint8_t *best_assign,
                 double *trace_cand, uint8_t *trace_ok);
/* Number of chains, and their live (current) strategies. */
int ps_mcmc_chains(const ps_mcmc *m);
int ps_mcmc_read_state(ps_mcmc *m, int32_t *maps, uint8_t *assign);
/* Halt chains with stop[i] != 0 (host-side stagnation / budget rules). */
int ps_mcmc_stop(ps_mcmc *m, const uint8_t *stop);
void ps_mcmc_destroy(ps_mcmc *m);

/* Best chain by (best_cost, chain index) -- the reference's strict-< earliest-chain
 * rule (search.py:256), reduced on the device. */
int ps_mcmc_best(ps_mcmc *m, double *best_cost, int32_t *best_chain);

const char *ps_last_error(void);
int ps_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif
