/*
 * tessel_b200 — C ABI of the B200-native schedule-search path.
 *
 * Drop-in boundary for the reference's decide-kernel seam
 *   repsched._core.decide   (/root/reference/pkg/src/repsched/_core/__init__.py:23-28,
 *                            kernel_c.pyx:23-37)
 * plus the batched repetend-search engine the reference has no equivalent of
 * (it evaluates one candidate per Python call: completion.py:318-349,
 * repetend.py:253-328).  Plain pointers and sizes only; no torch types.
 *
 * Status codes follow the reference: TSL_UNSAT=0, TSL_SAT=1, TSL_TIMEOUT=2.
 * Functions returning int use 0 for success and a negative TSL_E* code on
 * error (message via tsl_last_error(), thread-local).  The library never
 * falls back to CPU computation: without a CUDA device every compute entry
 * point fails with TSL_ENODEV.
 */
#ifndef TESSEL_B200_H
#define TESSEL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSL_UNSAT 0
#define TSL_SAT 1
#define TSL_TIMEOUT 2

#define TSL_OK 0
#define TSL_EINVAL -1  /* malformed arguments / value out of kernel range */
#define TSL_ENODEV -2  /* no CUDA device / driver */
#define TSL_ECUDA -3   /* CUDA runtime error */
#define TSL_ERANGE -4  /* size beyond the compiled limits */

/* Maximum items per decide problem, devices per placement, stages per
 * placement handled by the batched repetend engine. */
#define TSL_MAX_ITEMS 2048
#define TSL_MAX_DEVICES 64
#define TSL_MAX_STAGES 64

const char *tsl_last_error(void);
int tsl_version(void);
/* Number of visible CUDA devices (0 when none). */
int tsl_device_count(void);
/* Bind the calling thread to a CUDA device. */
int tsl_set_device(int device);

/* ----------------------------------------------------------------------
 * Single decide problem — replaces repsched._core.decide
 * (kernel_c.pyx:23-37): lex-first feasible start vector in `order` within
 * [lo, hi] under difference edges s[dst] >= s[src] + lag (edges: m rows of
 * (src, dst, lag), row-major), exclusivity between items with intersecting
 * device masks, per-device running memory <= cap (cap < 0: unconstrained),
 * node cap `node_budget` (0 = none) and a wall budget `budget_secs`
 * (<= 0 = none; replaces the absolute `deadline`).  Node counts equal the
 * reference's.  Writes out_starts[n] on SAT and *out_nodes always.
 * Returns the status (>= 0) or a negative error code.
 * ---------------------------------------------------------------------- */
int tsl_decide(int n, const int64_t *dur, const uint64_t *devmask, const int64_t *mem,
               const int64_t *edges, int m, const int64_t *order, const int64_t *lo,
               const int64_t *hi, int ndev, const int64_t *init_mem, int64_t cap,
               int64_t node_budget, double budget_secs, int64_t *out_starts,
               int64_t *out_nodes);

/* Batched form: `count` independent problems evaluated concurrently on the
 * GPU (one per CUDA thread group).  Each problem uses the fields below with
 * the same meaning as tsl_decide.  status[i], nodes[i] and
 * starts[i*stride .. +n_i) are written per problem. */
typedef struct tsl_problem {
  int n, m, ndev;
  const int64_t *dur, *mem, *edges, *order, *lo, *hi, *init_mem;
  const uint64_t *devmask;
  int64_t cap, node_budget;
} tsl_problem;

int tsl_decide_batch(int count, const tsl_problem *probs, double budget_secs, int32_t *status,
                     int64_t *nodes, int64_t *starts, int stride);

/* ----------------------------------------------------------------------
 * Batched repetend-search engine (replaces the per-candidate loop of
 * completion.search + repetend.solve_repetend: completion.py:318-349,
 * repetend.py:65-90, 93-105, 108-190, 253-302).
 * A placement is K stages on D devices: per-stage time, memory delta and
 * device mask, plus the dependency pairs (i, j) sorted ascending.
 * ---------------------------------------------------------------------- */
typedef struct tsl_engine tsl_engine;

typedef struct tsl_level_stats {
  int64_t probes;        /* (candidate, period) probes run at this level   */
  int64_t root_refuted;  /* refuted by root propagation / root checks      */
  int64_t nodes;         /* DFS nodes (reference node accounting)          */
  int64_t capped;        /* probes that hit the node cap (TIMEOUT)         */
  int64_t sat;           /* probes that returned SAT                       */
  int64_t deferred;      /* probes over the small budget, sent to resolve   */
  int64_t dj_refuted;    /* deferred probes proven infeasible by DJ         */
  int64_t dj_nodes;      /* DJ branching nodes                              */
} tsl_level_stats;

tsl_engine *tsl_engine_open(int K, int D, const int32_t *dur, const int32_t *mem,
                            const uint64_t *devmask, int n_deps, const int32_t *deps,
                            int device);
void tsl_engine_close(tsl_engine *e);

/* Number of enumerated candidates at n_r (repetend.py:65-90 order, with the
 * min-index-0 filter).  Fails with TSL_ERANGE beyond 2^63. */
int tsl_engine_count(tsl_engine *e, int n_r, uint64_t *out_count);
/* Host-side unranking (global lexicographic rank -> per-stage indices). */
int tsl_engine_unrank(tsl_engine *e, int n_r, uint64_t rank, int32_t *out_assignment);

/* Stage a window of ranks [r0, r1) at n_r on the device: unrank, entry
 * memory, memory gate (cap < 0: none).  Returns the number of candidates
 * that pass the gate in *out_active and, if gate_out is non-NULL, one byte
 * per rank (1 = passes, 0 = "infeasible"). */
int tsl_engine_stage(tsl_engine *e, int n_r, uint64_t r0, uint64_t r1, int64_t cap,
                     int64_t *out_active, uint8_t *gate_out);

/* Probe every still-active candidate of the staged window at `period`.
 * `node_budget` is the reference's per-probe node cap (0 = none:
 * repetend.py:289-292).  Each probe first runs the reference-exact DFS with
 * `small_budget` nodes; probes that exhaust it below the reference cap are
 * DEFERRED (see tsl_engine_resolve).  Candidates whose window index exceeds
 * `widx_limit` are retired without probing.  SAT candidates leave the
 * active set and are reported as (window index, starts[K]) rows in
 * ascending window-index order, up to max_sat rows (*out_nsat is the true
 * count).  *out_active / *out_deferred receive the remaining counts. */
int tsl_engine_probe(tsl_engine *e, int period, int64_t node_budget, int64_t small_budget,
                     int64_t cap, int64_t widx_limit, double budget_secs, int64_t max_sat,
                     int64_t *out_nsat, int64_t *sat_widx, int32_t *sat_starts,
                     int64_t *out_active, int64_t *out_deferred, tsl_level_stats *stats);

/* One stage of settling the deferred probes of the last level whose window
 * index is <= widx_limit (the others are retired and dropped): when
 * dj_budget > 0, a complete disjunctive solver first (an infeasibility proof
 * = "not SAT", the same conclusion the reference draws from its UNSAT or its
 * node-capped TIMEOUT); then the reference-exact DFS with
 * min(stage_budget, node_budget) nodes (stage_budget 0 = the reference cap).
 * Probes exhausting a stage budget below the cap stay deferred for the next
 * stage.  SAT rows are merged into the level's SAT list (returned sorted as
 * in tsl_engine_probe); settled non-SAT probes rejoin the active set. */
int tsl_engine_resolve(tsl_engine *e, int period, int64_t node_budget, int64_t stage_budget,
                       int64_t dj_budget, int64_t cap, int64_t widx_limit, double budget_secs,
                       int64_t max_sat, int64_t *out_nsat, int64_t *sat_widx,
                       int32_t *sat_starts, int64_t *out_active, int64_t *out_deferred,
                       tsl_level_stats *stats);

/* Speculation support (see engine.py): take the deferred entries of the last
 * stage with window index <= widx_limit to the host (ascending; they leave
 * the device lists unsettled), and append window indices to the active list
 * (probed again at the next period). */
int tsl_engine_take_deferred(tsl_engine *e, int64_t widx_limit, int64_t max_out,
                             int64_t *widx_out, int64_t *out_count);
int tsl_engine_add_active(tsl_engine *e, int64_t count, const int64_t *widx);

/* Reference-exact repetend probes for explicit (window index, period) pairs
 * of the staged window, each under its own node cap (0 = none), run
 * concurrently (one warp per pair).  Writes status, node count and, on SAT,
 * starts[i*K .. +K).  A SAT (w, P) speculatively retires every pair (w2, P2)
 * with w2 > w and P2 >= P: such pairs stop early with status 3 (aborted, not
 * a reference status); the caller re-runs them unless that SAT's completion
 * check passes. */
/* Asynchronous verification (engine.py pipelines windows): stash the
 * assignments of `count` window indices of the staged window into slot
 * 0..TSL_VERIFY_SLOTS-1 (rows = positions 0..count-1), launch the
 * verification of (row position, window index, period, cap) quadruples of
 * that slot on the slot's own stream — it runs while later windows are
 * staged and scanned, concurrently with the other slots — and wait for /
 * read its results (same meaning as tsl_engine_verify). */
#define TSL_VERIFY_SLOTS 8
int tsl_engine_verify_stash(tsl_engine *e, int slot, int64_t count, const int64_t *widx);
int tsl_engine_verify_launch(tsl_engine *e, int slot, int64_t count, const int64_t *pos,
                             const int64_t *widx, const int32_t *period,
                             const int64_t *node_budget, int64_t cap);
int tsl_engine_verify_wait(tsl_engine *e, int slot, int32_t *status_out, int64_t *nodes_out,
                           int32_t *starts_out);

/* Diagnostic: the disjunctive filter (DJ) on explicit (assignment[K],
 * period) pairs — status 0 = proven infeasible, 1 = feasible, 2 = undecided
 * within `budget` orientation nodes.  mode 1 = warp filter, 0 = one-lane
 * filter.  The search uses DJ only to refute (never to accept). */
int tsl_engine_dj(tsl_engine *e, int64_t count, const int32_t *assignments,
                  const int32_t *period, int64_t cap, int64_t budget, int mode,
                  int32_t *status_out, int64_t *nodes_out);

int tsl_engine_verify(tsl_engine *e, int64_t count, const int64_t *widx, const int32_t *period,
                      const int64_t *node_budget, int64_t cap, int32_t *status_out,
                      int64_t *nodes_out, int32_t *starts_out);

/* Rows [first, first+count) of the last probe's SAT list (ascending window
 * index): window indices and starts[count*K].  Rows stay on the device until
 * the next tsl_engine_probe / tsl_engine_stage call. */
/* Ordered walk of the last level's SAT list on the device: the SAT with the
 * smallest window index above `after` (-1: the first) and its starts[K];
 * *widx_out = -1 when there is none.  Replaces the host sort of
 * completion.py:351-382's in-order scan (north_star kernel 3). */
int tsl_engine_sat_next(tsl_engine *e, int64_t after, int64_t *widx_out, int32_t *starts_out);
int tsl_engine_sat_rows(tsl_engine *e, int64_t first, int64_t count, int64_t *widx_out,
                        int32_t *starts_out);

/* Process-wide counters since load: kernel launches issued by this library
 * and bytes copied host->device / device->host (bench accounting). */
void tsl_counters(int64_t *launches, int64_t *h2d_bytes, int64_t *d2h_bytes);

/* Device time (ms) of the kernels of the last tsl_engine_stage/probe call,
 * measured with CUDA events on the engine's stream. */
float tsl_engine_last_kernel_ms(tsl_engine *e);
/* Device time (CUDA events) of the root-filter kernel inside the last
 * tsl_engine_probe call (part of tsl_engine_last_kernel_ms). */
float tsl_engine_last_root_ms(tsl_engine *e);

/* Schedule validation on the device — the checks of the reference's
 * validate_schedule (schedule.py:77-168) for an N-micro-batch schedule:
 * starts[st * N + n]; deps as sorted (a, b) pairs.  P = next power of two
 * >= max over devices of (#stages on the device) * N.  Writes the number of
 * violations (overlaps + memory group ends + dependencies + negative starts)
 * to *out_count and, only when it is > 0, per device d the sorted event keys
 * ((start ^ 0x80000000) << 32 | position, position = stage-slot * N + mb,
 * stage slots ascending) and, at sorted position p, overlap / memory flags
 * and the running memory after p (D*P each), dependency flags [n_deps*N] and
 * negative-start flags [K*N].  The caller formats the violation list. */
int tsl_validate(int K, int D, const int32_t *dur, const int32_t *mem, const uint64_t *devmask,
                 int n_deps, const int32_t *deps, int N, const int32_t *starts,
                 const int64_t *init_mem, int64_t cap, int64_t P, int64_t *out_count,
                 uint64_t *sorted_keys, uint8_t *overlap_flags, uint8_t *memory_flags,
                 int64_t *runs, uint8_t *dep_flags, uint8_t *neg_flags);

/* Process-wide counters of the subtree-parallel decide: solves, rounds,
 * tasks, replays, nested sub-solves, master nodes, master wall ms, task wall
 * ms, donated pieces, tasks re-run undivided, nodes explored by task
 * launches, sticky-set epochs (out[12]). */
void tsl_sp_stats(double *out);

#ifdef __cplusplus
}
#endif
#endif
