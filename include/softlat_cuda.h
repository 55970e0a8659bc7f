/*
 * softlat_cuda.h -- C ABI of the B200 spring-mass step library
 * (paper_1911_10274_b200/libsoftlat_cuda.so).
 *
 * This is the drop-in boundary for the reference's hot path.  The reference
 * (Python + numba, /root/reference/pkg/src/softlat) dispatches a step through
 * engine.spring_pass / engine.mass_pass / engine.step (engine.py:158-264) into
 * numba kernels that take flat store arrays, mutate them in place and report
 * through out-parameters (kernels.py:28-32, 250-253; counters[3] at
 * kernels.py:84-86; err_slot at kernels.py:374-376).  Each entry point below
 * names the reference interface it replaces.
 *
 * Conventions
 *   - plain pointers + sizes, no torch / CUDA types; host arrays are in the
 *     reference store layout: vectors double[n][3] C-contiguous, indices
 *     int64, flags one byte (numpy bool), generations int64
 *     (store.py:123-151).
 *   - every call returns an int status (SL_OK = 0).  No exception crosses the
 *     ABI.  sl_last_error(ctx) holds a message for the last failure.
 *   - one context = one device + one CUDA stream; a context is not
 *     thread-safe (the reference's controller already serialises every call
 *     under its condition lock, control.py:628-643).  Distinct contexts may
 *     be driven from distinct threads.
 *   - the host store is authoritative while paused, the device while a run
 *     is in progress (store.lock_for_run, store.py:206-224).
 */
#ifndef SOFTLAT_CUDA_H
#define SOFTLAT_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (engine.py:251-255 NumericalAbort maps to SL_ENUMERIC) */
#define SL_OK 0
#define SL_EINVAL 1       /* bad argument (InvalidValueError)            */
#define SL_ECUDA 2        /* CUDA runtime failure                         */
#define SL_ENUMERIC 3     /* non-finite state; err_slot = slot + 1        */
#define SL_ESTATE 4       /* call illegal in the context's current state  */
#define SL_EUNSUPPORTED 5 /* feature not available on this build/device   */

/* arithmetic of the state and of the spring force (hard part 3) */
#define SL_PREC_FP64 0  /* double everywhere; parity mode (bit-exact gather) */
#define SL_PREC_FP32 1  /* float spring math; compensated float positions   */
#define SL_PREC_MIXED 2 /* double mass state, float spring parameters/math  */

/* force accumulation (StepConfig.accumulation, engine.py:40,49):
 *   GATHER = deterministic per-mass CSR gather in ascending spring-slot order
 *            (== reference "slotted" == serial, engine.py:105-118)
 *   ATOMIC = one thread per spring, vector atomics into f_ext
 *            (reference "linearizable": order-dependent rounding)         */
#define SL_ACC_GATHER 0
#define SL_ACC_ATOMIC 1
#define SL_ACC_AUTO 2   /* gather unless hub masses (widest list > 128) */

typedef struct sl_ctx sl_ctx;

typedef struct sl_stats {
  int64_t masses;          /* mass slots resident (high-water m_n)          */
  int64_t springs;         /* spring slots resident (high-water s_n)        */
  int64_t alive_springs;   /* springs alive at the last layout build        */
  int64_t entries;         /* incidence entries incl. padding               */
  int64_t slices;          /* 32-mass slices of the incidence layout        */
  int64_t layout_builds;   /* number of device layout (re)builds            */
  int64_t device_bytes;    /* device memory owned by the context            */
  int64_t kernel_launches; /* kernels launched by the context so far        */
  int32_t precision;
  int32_t device;
  int32_t step_path;   /* fused gather kernel in use: SL_PATH_*             */
  int32_t split_batch; /* gather batch U of the split TMA kernel (0 = n/a) */
  int64_t fused_groups;   /* body groups of the multi-step fused kernel
                             (0: the context runs per-step kernels only)  */
  int64_t fused_launches; /* multi-step fused launches so far             */
  int64_t fused_aborts;   /* of which re-run through per-step kernels     */
  int32_t win_tile_slices; /* window kernel: slices per tile = consumer
                              warps (the k_win_tma<P, T> instantiation)   */
  int32_t win_stages;      /* window kernel: tile stages in the ring      */
  int64_t inplace_edits;   /* spring record writes applied to the live
                              layout in place (sl_write_springs: O(edits),
                              no re-index)                                 */
} sl_stats;

/* sl_stats.step_path */
#define SL_PATH_NONE 0        /* no incidence layout built yet              */
#define SL_PATH_EXACT 1       /* exact layout, one thread per mass          */
#define SL_PATH_EXACT_TMA 2   /* exact layout, TMA-pipelined (k_gather_tma) */
#define SL_PATH_SPLIT 3       /* split layout, one thread per mass          */
#define SL_PATH_SPLIT_TMA 4   /* split layout, TMA-pipelined (k_split_tma)  */
#define SL_PATH_WINDOW_TMA 5  /* split layout, tiled windows (k_win_tma)     */
#define SL_PATH_EXACT_WINDOW 6 /* exact layout, tiled windows (fp64 k_win_tma) */

/* ---------------------------------------------------------------- lifecycle */
int sl_abi_version(void);
int sl_device_count(int *count);
/* one context per store per device (engine._StoreCache, engine.py:71-102) */
int sl_create(int device, int precision, sl_ctx **out);
int sl_destroy(sl_ctx *ctx);
const char *sl_last_error(const sl_ctx *ctx); /* ctx may be NULL */
int sl_get_stats(sl_ctx *ctx, sl_stats *out);
/* Page-locked host memory (cudaHostAlloc, portable) for the store's mass
 * columns: uploads and downloads from it run at copy-engine speed.  The
 * reference's arrays are plain numpy (store.py:123-151); the host side moves
 * the mass columns into such buffers on first push (engine.DeviceMirror). */
int sl_host_alloc(size_t bytes, void **out);
int sl_host_free(void *p);

/* ------------------------------------------------------------------ upload */
/* Whole mass SoA, slots [0, m_n) (store.py:123-132; mass-pass arguments of
 * kernels.py:250-253).  Vectors are double[m_n][3]; any of acc/fext/load may
 * be NULL (= zero). */
int sl_upload_masses(sl_ctx *ctx, int64_t m_n, const double *pos,
                     const double *vel, const double *acc, const double *fext,
                     const double *load, const double *mass,
                     const uint8_t *fixed, const uint8_t *alive,
                     const int64_t *gen);

/* Whole spring SoA, slots [0, s_n) (store.py:134-151; spring-pass
 * arguments of kernels.py:28-32).  mode: 0 none, 1 sine, 2 sine quiescent
 * before offset, 3 custom (store.py:36-40).  Triggers a device rebuild of the
 * incidence layout. */
int sl_upload_springs(sl_ctx *ctx, int64_t s_n, const int64_t *m1,
                      const int64_t *m2, const int64_t *m1gen,
                      const int64_t *m2gen, const double *rest,
                      const double *k, const double *diam,
                      const double *yield, const int8_t *mode,
                      const double *amp, const double *freq,
                      const double *off, const double *per,
                      const uint8_t *alive, const uint8_t *degen);

/* Environment flattened as engine.mass_pass does every call
 * (engine.py:223-245): gravity[3], drag, planes[n][7] =
 * (nx,ny,nz,offset,k,mu_s,mu_k), balls[n][5] = (cx,cy,cz,r,k), global
 * constraints kind (1 direction, 2 plane; kernels.py:24-25) + unit vector,
 * v_stick (engine.py:38). */
int sl_set_environment(sl_ctx *ctx, const double *gravity, double drag,
                       const double *planes, int64_t n_planes,
                       const double *balls, int64_t n_balls,
                       const int8_t *gc_kind, const double *gc_vec,
                       int64_t n_gc, double v_stick);

/* Per-mass local constraints as the CSR of engine._refresh_constraints
 * (engine.py:121-146): lc_off[m_n+1], lc_kind[n_lc], lc_vec[n_lc][3]. */
int sl_set_local_constraints(sl_ctx *ctx, int64_t m_n, const int64_t *lc_off,
                             const int8_t *lc_kind, const double *lc_vec,
                             int64_t n_lc);

/* Host-evaluated factors of callable waveforms (mode 3), the device copy of
 * engine._fill_custom_factors (engine.py:149-155). */
int sl_set_custom_factors(sl_ctx *ctx, int64_t n, const int64_t *slots,
                          const double *factors);

/* ------------------------------------------------------------ O(1) edits */
/* Overwrite individual mass slots (store setters at a pause point,
 * store.py:536-601, control.py:480-515).  Slots must be < current m_n. */
int sl_write_masses(sl_ctx *ctx, int64_t n, const int64_t *slots,
                    const double *pos, const double *vel, const double *acc,
                    const double *fext, const double *load,
                    const double *mass, const uint8_t *fixed,
                    const uint8_t *alive, const int64_t *gen);
/* Overwrite parameters of existing spring slots in place (set_spring_field,
 * store.py:563-588): rest, k, diam, yield and actuation, same arrays as
 * sl_upload_springs minus topology.  O(n), no layout rebuild. */
int sl_write_spring_params(sl_ctx *ctx, int64_t n, const int64_t *slots,
                           const double *rest, const double *k,
                           const double *diam, const double *yield,
                           const int8_t *mode, const double *amp,
                           const double *freq, const double *off,
                           const double *per);
/* Kill spring slots (delete_spring / reconcile, store.py:440-473). O(n). */
/* Whole spring records for the given slots (< the current spring count):
 * spring creations into reused slots at a pause (store.py:356-370).  Only
 * the touched slots cross the bus; the incidence layout is re-indexed on
 * the device at the next step. */
int sl_write_springs(sl_ctx *ctx, int64_t n, const int64_t *slots,
                     const int64_t *m1, const int64_t *m2,
                     const int64_t *m1gen, const int64_t *m2gen,
                     const double *rest, const double *k, const double *diam,
                     const double *yield, const int8_t *mode,
                     const double *amp, const double *freq, const double *off,
                     const double *per, const uint8_t *alive,
                     const uint8_t *degen);
int sl_kill_springs(sl_ctx *ctx, int64_t n, const int64_t *slots);

/* -------------------------------------------------------------------- step */
/* n_steps of engine.step (engine.py:258-264): spring pass + mass pass per
 * step, sim time of step i = sim_times[i] (engine.step's sim_t argument;
 * the controller passes t0 + step_count*dt, control.py:306-307).
 * Stops after the first step that produces non-finite state (that step's
 * writes are kept, as the reference's mass pass writes before raising):
 * returns SL_ENUMERIC, *err_slot = offending slot + 1 (highest, the serial
 * loop's last write, kernels.py:374-376), *steps_done includes that step.
 * counters[3] (+=) = (broken, invalid, degenerate_new), kernels.py:84-86.
 * write_acc: also store per-mass acceleration of the final step. */
int sl_step(sl_ctx *ctx, int64_t n_steps, const double *sim_times, double dt,
            int accumulation, int64_t *counters, int64_t *err_slot,
            int64_t *steps_done);

/* Asynchronous stepping (partitioned runs, partition.py): enqueue n_steps
 * on the context's stream and return at once; successive calls continue
 * the same run (step indices and status accumulate) until sl_step_finish
 * synchronises and reports exactly what sl_step would have for the
 * concatenated steps.  Between calls the caller may enqueue its own work
 * on the context stream (sl_get_stream), e.g. a halo exchange that
 * rewrites ghost positions in the buffer the next step reads
 * (sl_state_pointers). */
int sl_step_async(sl_ctx *ctx, int64_t n_steps, const double *sim_times,
                  double dt, int accumulation);
int sl_step_finish(sl_ctx *ctx, int64_t *counters, int64_t *err_slot,
                   int64_t *steps_done);

/* Single spring pass only (engine.spring_pass, engine.py:158-202): spring
 * forces are added into the device f_ext accumulator. */
int sl_spring_pass(sl_ctx *ctx, double sim_t, int accumulation,
                   int64_t *counters);
/* Single mass pass only (engine.mass_pass, engine.py:218-255). */
int sl_mass_pass(sl_ctx *ctx, double dt, int64_t *err_slot);

/* Host state of EVERY mass back into a context that holds the rest:
 * positions, velocities and/or accelerations (NULL keeps the device copy)
 * of m_n masses (== the uploaded count); flags, masses, loads and f_ext
 * stay.  The device mirror's partial push: after a pause only the columns
 * the host touched travel (engine.DeviceMirror.push). */
int sl_write_state(sl_ctx *ctx, int64_t m_n, const double *pos,
                   const double *vel, const double *acc);
/* The same, returning once the copies and the conversion are enqueued on
 * the context's stream: the host arrays (page-locked for a true overlap)
 * must stay unchanged until sl_sync(ctx) returns.  io.apply_snapshot's
 * write-through: the upload runs while the host copies the same columns
 * into the store. */
int sl_write_state_async(sl_ctx *ctx, int64_t m_n, const double *pos,
                         const double *vel, const double *acc);

/* Opt-in spring damping (north_star "Hooke plus damping"): damping[s] =
 * c >= 0 (N s / m) for every spring slot [0, s_n); the force on m1 gains
 * c ((v2 - v1) . d^) d^ (equal and opposite on m2).  No reference
 * counterpart (kernels.py:66 is Hooke only): c = 0 everywhere restores the
 * reference path bit for bit.  A full sl_upload_springs clears the
 * dampers; damped contexts step the force pass and the mass pass as two
 * kernels. */
int sl_set_spring_damping(sl_ctx *ctx, int64_t n, const double *damping);

/* ---------------------------------------------------------------- download */
/* Copy mass state back into host arrays double[m_n][3]; NULL skips. */
int sl_download_masses(sl_ctx *ctx, double *pos, double *vel, double *acc,
                       double *fext);
/* The pause-time pull of engine.DeviceMirror.pull (control.py pause):
 * like sl_download_state, plus optional EXTRA page-locked destinations
 * pos2 / vel2 (a snapshot's own buffers) copied first.  wait_head = 0
 * returns as soon as everything is enqueued: sl_download_wait_extra waits
 * for pos2 / vel2, sl_download_wait for all of it (the host store settles
 * on first access).  The destinations must stay allocated until then. */
int sl_download_state_ex(sl_ctx *ctx, double *pos, double *vel, double *acc,
                         double *fext, double *pos2, double *vel2,
                         int wait_head);
int sl_download_wait_extra(sl_ctx *ctx);
/* Stash the current mass state (positions, velocities, accelerations,
 * f_ext as fp64) in a device buffer, enqueued on the context stream -- the
 * next run's step kernels do not wait for anything.  sl_download_stash
 * copies (parts of) the stash into host arrays on the side stream and
 * waits for them: the host store's lock-time state, fetched only when a
 * reader needs it (ObjectStore.lock_for_run). */
int sl_stash_state(sl_ctx *ctx);
/* Speculative predicate checks (control.py condition breakpoints): keep a
 * device copy of the current state (positions, velocities, accelerations,
 * f_ext, the ping-pong index) and, when view_pos / view_vel are given
 * (page-locked double[m_n][3]), copy positions / velocities there on the
 * side stream -- the next run goes on while the host evaluates the
 * predicate; sl_checkpoint_view_wait waits for the view.  sl_restore puts
 * the checkpointed state back (the run after it is undone; the caller
 * guarantees no topology change happened in between). */
int sl_checkpoint(sl_ctx *ctx, double *view_pos, double *view_vel);
int sl_checkpoint_view_wait(sl_ctx *ctx);
int sl_restore(sl_ctx *ctx);
int sl_download_stash(sl_ctx *ctx, double *pos, double *vel, double *acc,
                      double *fext);
/* As sl_download_masses, but returns once pos / vel have landed: acc and
 * f_ext (which must be page-locked) keep arriving on the context stream;
 * sl_download_wait blocks until they have.  Work enqueued afterwards is
 * ordered after the copies. */
int sl_download_state(sl_ctx *ctx, double *pos, double *vel, double *acc,
                      double *fext);
int sl_download_wait(sl_ctx *ctx);
/* Spring liveness / zero-length flags back into bool[s_n]; NULL skips. */
int sl_download_springs(sl_ctx *ctx, uint8_t *alive, uint8_t *degen);

/* ------------------------------------------------------------ diagnostics */
/* engine.mechanical_energy (engine.py:366-389) from the device state:
 * out = {kinetic, spring potential (actuated rest length at sim_t),
 * gravitational potential (origin reference, gravity[3])}; fp64 partial
 * sums in a fixed order (deterministic). */
int sl_energy(sl_ctx *ctx, double sim_t, const double *gravity, double *out);
/* engine.spring_loads (engine.py:392-412): per spring slot [0, s_n) the
 * length and |k (|d| - f L0)| at sim_t; NaN for dead slots (the caller
 * compacts over alive slots and forms the stress from its diameters). */
int sl_spring_loads(sl_ctx *ctx, double sim_t, double *lengths,
                    double *force_magnitudes);

/* Asynchronous snapshot (north_star "pinned-memory async snapshots"):
 * enqueue a D2H copy of positions + velocities into library-owned pinned
 * buffers on a side stream, ordered after all work issued so far; returns
 * immediately.  sl_snapshot_wait blocks until it lands and copies it out. */
int sl_snapshot_begin(sl_ctx *ctx);
int sl_snapshot_ready(sl_ctx *ctx, int *ready);
int sl_snapshot_wait(sl_ctx *ctx, double *pos, double *vel);

/* ------------------------------------------------- partitioned runs */
/* Mark mass slots as ghosts (copies of masses owned by another rank):
 * they must also be fixed (never integrated); spring events whose m1
 * endpoint is a ghost are not counted here (the owner counts them).
 * Cleared when the mass count changes. */
int sl_mark_ghosts(sl_ctx *ctx, int64_t n, const int64_t *slots);
/* Device pointer of the position buffer the next step reads: rows records
 * of record_bytes (x, y, z, m as float or double).  Valid until the next
 * step call. */
int sl_state_pointers(sl_ctx *ctx, void **pos_read, int64_t *rows,
                      int32_t *record_bytes);
/* fp32 mode: device pointer of the position LOW parts (ly, lz) (float2 per
 * mass) of the buffer the next step reads; the record (sl_state_pointers)
 * is (x, y, z, lx) in this mode, a position is record + low part and the
 * masses live apart.  NULL in fp64 / mixed. */
int sl_state_lo(sl_ctx *ctx, void **lo_read);
/* In-library halo of a mass-range partition (config E; replaces the
 * per-step Python exchange of partition.py).  Each rank's context holds its
 * owned masses then its ghosts (fixed + sl_mark_ghosts).  dst[2 * i + q]
 * (q = 0, 1) names where owned mass i's position goes after every step:
 * (row << 3) | peer, row = the ghost's local index at that peer, or -1.
 * The step kernels store those rows straight into the peers' position
 * buffers (mapped with sl_halo_ipc_open across processes, or the pointers
 * of sl_halo_local within one process), and after every step a one-block
 * kernel publishes a per-peer step counter and waits for the peers' --
 * no host round trip, no collective.  Setup: sl_halo_init, then per peer
 * sl_halo_set_peer(peer, its 5 pointers, the counter slot it reserved for
 * this rank), then sl_halo_commit.  All ranks must step in lockstep (same
 * step counts per call) from the same buffer parity; damping is
 * unsupported (ghost velocities are not exchanged).
 * The 5 pointers: position records [2], fp32 low parts [2] (NULL in fp64 /
 * mixed), the counter words [8]. */
#define SL_IPC_HANDLE_BYTES 64
int sl_halo_init(sl_ctx *ctx, int n_peers, const int32_t *dst);
int sl_halo_local(sl_ctx *ctx, void **ptrs5);
int sl_halo_ipc_handles(sl_ctx *ctx, void *out5x64);
int sl_halo_ipc_open(sl_ctx *ctx, const void *handles5x64, void **ptrs5);
int sl_halo_set_peer(sl_ctx *ctx, int peer, void *const *ptrs5, int slot);
int sl_halo_commit(sl_ctx *ctx);
/* The context's CUDA stream (cudaStream_t) for ordering foreign work. */
int sl_get_stream(sl_ctx *ctx, void **stream);

/* ---------------------------------------------------------------- snapshots */
/* Snapshot CSV of io.py:19-32 (format_snapshot): header "id,x,y,z,vx,vy,vz"
 * then one row per mass, each double as Python's "{:.17g}" (bit-exact
 * round trip; "inf"/"-inf"/"nan" for non-finite values).  Host only, no
 * context.  `out` must hold 18 + n * SL_SNAPSHOT_ROW_MAX bytes; *len gets
 * the text length (no terminating NUL). */
#define SL_SNAPSHOT_ROW_MAX 176
int sl_format_snapshot(int64_t n, const int64_t *ids, const double *pos,
                       const double *vel, int threads, char *out, size_t cap,
                       size_t *len);

/* ------------------------------------------------------------ host builder */
/* Lattice generation of builder.py:112-186 (build_lattice + materialize):
 * n_masses = nx*ny*nz row-major nodes, springs grouped by the 13 cell
 * offsets; outputs are bit-identical to the numpy builder (rest, k = E A / L,
 * node mass = half-bar masses in np.add.at order; the caller applies the
 * minimum-mass rule to bare nodes).  Host only, `threads` workers. */
int sl_lattice_counts(int64_t nx, int64_t ny, int64_t nz, int64_t *n_masses,
                      int64_t *n_springs);
int sl_build_lattice(int64_t nx, int64_t ny, int64_t nz, const double *corner,
                     double spacing, double elastic_modulus, double density,
                     double diameter, int threads, double *pos,
                     double *node_mass, int64_t *a, int64_t *b, double *rest,
                     double *stiff);
/* Fill count elements of elem_bytes (<= 64) with *value on `threads`
 * workers (first touch of fresh store capacity in parallel). */
int sl_host_fill(void *dst, const void *value, size_t elem_bytes,
                 int64_t count, int threads);
/* *out = 1 iff ids[i] == i for every i < n (host, `threads` workers). */
int sl_host_is_iota(const int64_t *ids, int64_t n, int threads, int *out);
/* memcpy on `threads` workers (snapshot copies into fresh arrays). */
int sl_host_copy(void *dst, const void *src, size_t bytes, int threads);
/* min / max of v over mask != 0 (mask may be NULL), NaN-propagating like
 * numpy; empty selection gives +inf / -inf (check_stability's extrema). */
int sl_host_masked_extrema(const double *v, const uint8_t *mask, int64_t n,
                           int threads, double *out_min, double *out_max);

/* ---------------------------------------------------------- timing / sync */
/* CUDA events on the context's stream (bench.py measures with these). */
int sl_timer_start(sl_ctx *ctx);
int sl_timer_stop(sl_ctx *ctx, float *ms);
/* Device time of the step kernels of the last sl_step call: CUDA events
 * recorded on the context stream right before its first step kernel and
 * right after its last (the call's validation, status reset and status
 * read-back excluded). */
int sl_last_step_ms(sl_ctx *ctx, float *ms);
int sl_sync(sl_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* SOFTLAT_CUDA_H */
