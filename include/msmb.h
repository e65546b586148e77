/*
 * msmb.h -- C ABI of the B200-native MSM force / velocity-Verlet / parareal path.
 *
 * This is the drop-in boundary for the reference library `paramd`
 * (arXiv 1309.1889, /root/reference/proj).  Each entry point names the
 * reference interface it replaces (file:line, relative to /root/reference).
 * Plain pointers and sizes only; the library owns device memory, the caller
 * owns every host array.  Positions/velocities/forces are interleaved
 * double[3*n] -- the layout of std::vector<paramd::Vec3>
 * (include/paramd/vec3.hpp:6-7, a standard-layout {double x,y,z}), so
 * `system.positions.data()` can be passed directly.
 *
 * Error codes map 1:1 to the reference exception hierarchy
 * (include/paramd/errors.hpp:12-49, include/paramd/parareal.hpp:124-128); the
 * message text and the particle indices match the reference's
 * (src/msm_phases.cpp:25-26 and 238-239, include/paramd/msm_kernels.hpp:31,
 * src/msm_grid.cpp:11-22, include/paramd/units.hpp:23-26,
 * src/integrate.cpp:7-11, src/parareal.cpp:43-56 and 221-226) and are read
 * back with msmb_last_error().  There is no CPU fallback: every compute entry
 * point runs on the GPU and fails with MSMB_ERR_CUDA when none is usable.
 */
#ifndef MSMB_H
#define MSMB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MSMB_ABI_VERSION 2

/* Status codes == reference exception types. */
enum msmb_status {
    MSMB_OK = 0,
    MSMB_ERR_CONFIG = 1,         /* paramd::ConfigError              errors.hpp:12-14 */
    MSMB_ERR_DOMAIN = 2,         /* paramd::DomainError              errors.hpp:17-19 */
    MSMB_ERR_COVERAGE = 3,       /* paramd::CoverageError            errors.hpp:37-39 */
    MSMB_ERR_COINCIDENT = 4,     /* paramd::CoincidentParticlesError errors.hpp:32-34 */
    MSMB_ERR_HIERARCHY = 5,      /* paramd::HierarchyError           errors.hpp:42-44 */
    MSMB_ERR_RUNTIME = 6,        /* paramd::RuntimeFault             errors.hpp:47-49 */
    MSMB_ERR_NONCONVERGENCE = 7, /* paramd::NonConvergenceError      parareal.hpp:124-128 */
    MSMB_ERR_CUDA = 8,           /* no usable B200 / CUDA failure (no reference equivalent) */
    MSMB_ERR_INTERNAL = 9
};

/* paramd::MsmConfig, include/paramd/msm_grid.hpp:10-18 (same defaults: 8, 2, 2, 3, 2). */
typedef struct msmb_msm_config {
    double cutoff_a;
    double spacing_h;
    int levels_l;
    int interp_order_p;
    int smoothing_m;
} msmb_msm_config;

/* paramd::UnitsConfig, include/paramd/units.hpp:16-27 (physical: 332.0636, 4.184e-4). */
typedef struct msmb_units {
    double coulomb_constant;
    double energy_to_native;
} msmb_units;

/* One MSM force field bound to one GPU: the state of paramd::MsmField
 * (include/paramd/force_field.hpp:62-73).  Owns device workspaces and a
 * stream; calls on one handle are serialised internally, so a handle may be
 * shared by threads the way the reference's AsyncExecutor shares a ForceField
 * (src/parareal.cpp:27-33). */
typedef struct msmb_field msmb_field;

/* A device-resident ParticleSystem (include/paramd/system.hpp:10-18). */
typedef struct msmb_system msmb_system;

int msmb_abi_version(void);
/* Number of usable CUDA devices (0 on a machine without a GPU). */
int msmb_device_count(void);

/* MsmField::MsmField(MsmConfig, UnitsConfig)  force_field.hpp:64.  Validates
 * like MsmConfig::validate (src/msm_grid.cpp:11-22) and UnitsConfig::validate
 * (units.hpp:23-26) before touching the GPU. */
int msmb_create(const msmb_msm_config* cfg, const msmb_units* units, int device,
                msmb_field** out);
void msmb_destroy(msmb_field* f);

/* ---- pair-only fields ----------------------------------
 * paramd::SimpleCutoffField and paramd::WolfField (include/paramd/force_field.hpp:34-60;
 * simple_cutoff / wolf_summation, src/electrostatics.cpp:66-132): the paper's
 * coarse propagators and the CLI's default parareal coarse field
 * (tools/paramd_main.cpp:417).  A field handle of either kind works with every
 * entry point that takes a msmb_field (evaluate, propagate, systems, parareal as
 * fine or coarse propagator); the MSM-only entry points (spatial decomposition,
 * debug lattices/stages, lattice method) return MSMB_ERR_CONFIG for them.
 * The result is the reference's: per-particle potential, forces with k_C,
 * E = k_C sum 0.5 q_i phi_i in index order; phi_short receives phi and phi_long
 * zeros (the reference leaves PotentialResult::short_part/long_part empty).
 * Positions need not lie in the box: the box only sets the binning extent, atoms
 * outside it are clamped into the boundary cells (correct for any position, fast
 * when most atoms are inside).  A NaN coordinate makes every output NaN, as in the
 * reference (every pair with that particle is NaN); an infinite coordinate, for
 * which the reference mixes skipped and NaN pairs, is rejected with MSMB_ERR_DOMAIN. */
enum msmb_field_kind { MSMB_FIELD_MSM = 0, MSMB_FIELD_CUTOFF = 1, MSMB_FIELD_WOLF = 2, MSMB_FIELD_DIRECT = 3 };

/* paramd::CutoffParams (include/paramd/potential.hpp:26-31: cutoff 12 A, optional
 * wolf_alpha), plus the fields' cost-model constant flops_per_particle
 * (force_field.hpp:36,50; <= 0 selects the reference defaults 301 / 350). */
typedef struct msmb_cutoff_params {
    double cutoff;
    int has_wolf_alpha;
    double wolf_alpha;
    double flops_per_particle;
} msmb_cutoff_params;

/* SimpleCutoffField(params, units) / WolfField(params, units)  force_field.hpp:36,50.
 * Validates like CutoffParams::validate(need_alpha = kind == WOLF)
 * (src/electrostatics.cpp:38-42) and UnitsConfig::validate before touching the GPU. */
int msmb_create_cutoff(int kind, const msmb_cutoff_params* params, const msmb_units* units,
                       int device, msmb_field** out);
/* msmb_field_kind of a handle. */
int msmb_field_kind(const msmb_field* f);

/* ---- all-pairs fields ---------------------------------
 * DirectCoulombField(units) (force_field.hpp:23-32; direct_coulomb,
 * src/electrostatics.cpp:43-64): the exact O(N^2) Coulomb sum, the reference's
 * accuracy oracle (tools/paramd_main.cpp:148-212), on the GPU.  No box is needed.
 * Coincident particles raise MSMB_ERR_COINCIDENT with the reference's first pair. */
int msmb_create_direct(const msmb_units* units, int device, msmb_field** out);

/* PairRepulsionOverlay(base, epsilon, sigma)  force_field.hpp:75-97,
 * force_field.cpp:45-68: a NEW handle evaluating `base`'s field (same kind,
 * parameters and units; `base` itself is unchanged) plus the pair repulsion
 * U = sum_{i<j} eps (sigma/r)^12 over ALL pairs (O(N^2), as the reference):
 * forces and total energy include it, the per-particle potential stays
 * electrostatic.  name() = base name + "+rep"; cost = base cost + 30 n.  An
 * overlay of an overlay adds both terms (innermost first), as the reference's
 * nested decorators do. */
int msmb_create_overlay(const msmb_field* base, double epsilon, double sigma, msmb_field** out);

/* MsmField::evaluate / msm_potential(s, cfg, units)  force_field.cpp:37-39,
 * msm.cpp:52-90.  Host arrays; any output pointer may be NULL.
 * phi = per-particle potential per unit charge, phi_short/phi_long its two
 * halves (PotentialResult::short_part/long_part, potential.hpp:18-24). */
int msmb_evaluate(msmb_field* f, int64_t n, const double* pos_xyz, const double* q,
                  const double box[3], double* phi, double* phi_short, double* phi_long,
                  double* force_xyz, double* energy);

/* propagate(PropagatorSpec{field, dt, steps}, s, units)  integrate.cpp:13-36:
 * one initial evaluation, then `steps` velocity-Verlet steps.  pos/vel are
 * read and, on success, overwritten with the propagated state (on error they
 * are left untouched, as the reference throws before returning). */
int msmb_propagate(msmb_field* f, int64_t n, double* pos_xyz, double* vel_xyz, const double* q,
                   const double* mass, const double box[3], double dt, int steps);

/* propagate(spec, s, units) with an explicit UnitsConfig (the reference passes
 * `units` separately from the field, integrate.hpp:27-28; energy_to_native
 * converts the field's forces into accelerations).  units == NULL means the
 * field's own units. */
int msmb_propagate_ex(msmb_field* f, int64_t n, double* pos_xyz, double* vel_xyz, const double* q,
                      const double* mass, const double box[3], double dt, int steps,
                      const msmb_units* units);

/* energy_report(s, ff, units)  integrate.cpp:47-55: out = [kinetic, potential,
 * total]; the kinetic energy (system.cpp:51-55, divided by units->energy_to_native)
 * is summed on the device by a fixed-order tree, the potential is this field's
 * evaluation.  units == NULL means the field's own units. */
int msmb_energy_report(msmb_field* f, int64_t n, const double* pos_xyz, const double* vel_xyz, const double* q,
                       const double* mass, const double box[3], const msmb_units* units, double* out);

/* Page-locked host memory for fast transfers (cudaHostAlloc / cudaFreeHost). */
void* msmb_host_alloc(int64_t bytes);
void msmb_host_free(void* p);

/* MsmField::cost_flops_per_step = msm_flops_simplified(a, h, n)
 * force_field.cpp:41-43, cost_model.cpp:37-43; SimpleCutoffField / WolfField:
 * flops_per_particle * n (force_field.cpp:25-35); DirectCoulombField 20 n^2
 * (:17-19); an overlay adds 30 n (:70-72). */
double msmb_cost_flops_per_step(const msmb_field* f, int64_t n);

/* Details of the last failure on this handle: kind = msmb_status, i/j the
 * particle indices named by the message (-1 when none), step = the Verlet
 * step whose evaluation failed (0 = the initial evaluation, -1 = n/a). */
int msmb_last_error(const msmb_field* f, int* kind, int64_t* idx_i, int64_t* idx_j, int* step,
                    char* msg, int cap);

/* ---- device-resident systems (inputs stay in HBM across calls) ------------ */
int msmb_system_create(msmb_field* f, int64_t n, const double* pos_xyz, const double* vel_xyz,
                       const double* q, const double* mass, const double box[3],
                       msmb_system** out);
void msmb_system_destroy(msmb_system* s);
int msmb_system_upload(msmb_system* s, const double* pos_xyz, const double* vel_xyz);
int msmb_system_download(const msmb_system* s, double* pos_xyz, double* vel_xyz);
int msmb_system_copy(msmb_system* dst, const msmb_system* src);
/* In-place device-resident propagate (same semantics as msmb_propagate). */
int msmb_system_propagate(msmb_field* f, msmb_system* s, double dt, int steps);
/* ... with an explicit UnitsConfig (as msmb_propagate_ex; NULL = the field's). */
int msmb_system_propagate_ex(msmb_field* f, msmb_system* s, double dt, int steps,
                             const msmb_units* units);
/* Device-resident evaluate; outputs copied to the (optional) host arrays. */
int msmb_system_evaluate(msmb_field* f, msmb_system* s, double* phi, double* phi_short,
                         double* phi_long, double* force_xyz, double* energy);

/* ---- parareal (src/parareal.cpp:94-239; include/paramd/parareal.hpp:40-144) -- */
typedef struct msmb_propagator {
    msmb_field* field; /* PropagatorSpec::force_field */
    double dt;         /* PropagatorSpec::dt */
    int steps_per_slice;
} msmb_propagator;

typedef struct msmb_parareal_config {
    int window_points; /* T_W */
    int max_iter;      /* K */
    double tol;        /* RMS position tolerance */
    msmb_propagator fine;
    msmb_propagator coarse;
    msmb_units units;
    int has_skip_threshold; /* std::optional<double> skip_threshold */
    double skip_threshold;
    int short_circuit;
} msmb_parareal_config;

/* parareal_init(v, cfg) + k_iters x parareal_iterate(w, cfg): one window of
 * t_points slices.  Returns the final lambda row (t_points+1 states,
 * interleaved pos/vel per state, n = 0..t) and, optionally, the per-slice
 * delta rms of the last iteration (t_points+1 entries, [0] unused) and the
 * evaluation counts [g_evals, f_evals, f_skipped]. */
int msmb_parareal_window(const msmb_parareal_config* cfg, int64_t n, const double* pos_xyz,
                         const double* vel_xyz, const double* q, const double* mass,
                         const double box[3], int t_points, int k_iters, double* row_pos,
                         double* row_vel, double* delta_rms, int64_t* counts);

/* parareal_run(v, total_points, cfg, exec)  parareal.cpp:182-239: sliding
 * windows with RMS-position convergence.  traj_* receive total_points states
 * (T_1..T_total).  report = [g_evals, f_evals, f_skipped, windows, converged]. */
int msmb_parareal_run(const msmb_parareal_config* cfg, int64_t n, const double* pos_xyz,
                      const double* vel_xyz, const double* q, const double* mass,
                      const double box[3], int total_points, double* traj_pos,
                      double* traj_vel, int64_t* report);

/* One row of paramd::ConvergenceReport::rows (include/paramd/parareal.hpp:93-110,
 * filled at src/parareal.cpp:208): window (1-based), point n (1..t), iteration k
 * (0-based), the fine delta's RMS position change, and whether the point met tol. */
typedef struct msmb_parareal_row {
    int window;
    int point;
    int iteration;
    double delta_rms;
    int converged;
} msmb_parareal_row;

/* parareal_run(v, total_points, cfg, exec)  parareal.cpp:182-239, with the
 * Executor (parareal.hpp:15-31, used at parareal.cpp:151) over GPUs:
 * fine_replicas[0..n_replicas) are extra fine fields with cfg->fine.field's kind
 * and parameters, typically one per device (msmb_create(..., device = k, ...)).
 * The fine slices of every iteration are dealt to cfg->fine.field and the
 * replicas as they free up (AsyncExecutor::parallel_for, parareal.cpp:16-36);
 * every slice's end state is copied back to cfg->fine.field's device, where the
 * state algebra and the coarse sweep run.  Results do not depend on the
 * replicas (pure propagators): they are bitwise those of msmb_parareal_run.
 * A failing fine slice reports the error of the lowest failing slice index, as
 * the sequential executor would.  report has 6 entries: msmb_parareal_run's 5
 * plus [5] = output points so far (ConvergenceReport::point_iterations size).
 * Besides the report,
 * `rows` receives up to rows_cap ConvergenceReport rows (*rows_written = the
 * total, which may exceed rows_cap) and point_iterations[total_points] the
 * iterations each output point took (ConvergenceReport::point_iterations);
 * both are filled on success and on MSMB_ERR_NONCONVERGENCE.  Any of the
 * output pointers may be NULL. */
int msmb_parareal_run_ex(const msmb_parareal_config* cfg, msmb_field* const* fine_replicas, int n_replicas,
                         int64_t n, const double* pos_xyz, const double* vel_xyz, const double* q,
                         const double* mass, const double box[3], int total_points, double* traj_pos,
                         double* traj_vel, int64_t* report, msmb_parareal_row* rows, int64_t rows_cap,
                         int64_t* rows_written, int* point_iterations);

/* ---- raw device states, for multi-process (one process per GPU) drivers -----
 * A "state" is 6*n doubles in device memory of the field's GPU, SoA:
 * x[n] y[n] z[n] vx[n] vy[n] vz[n] (the first six arrays of a msmb_system).
 * A "delta" is the reference's StateDelta (include/paramd/parareal.hpp:53-59):
 * dpos as n interleaved Vec3, then dvel, 6*n doubles.  Each call runs on the
 * field's stream and returns after the stream is synchronised, so the buffers
 * may be handed to a communication library (e.g. NCCL) right away.  The
 * arithmetic and reduction order are those of msmb_parareal_run, so a
 * multi-process parareal built on these calls reproduces it bit for bit. */
/* state_sub(a, b)  src/parareal.cpp:58-73; *rms_pos = sqrt(sum |dpos|^2 / 3n). */
int msmb_state_sub_device(msmb_field* f, int64_t n, const double* a, const double* b,
                          double* delta, double* rms_pos);
/* state_add(base, d)  src/parareal.cpp:75-82. */
int msmb_state_add_device(msmb_field* f, int64_t n, const double* base, const double* delta,
                          double* out);
/* rms_pos_change(a, b)  src/parareal.cpp:86-90. */
int msmb_state_rms_change_device(msmb_field* f, int64_t n, const double* a, const double* b,
                                 double* rms);
/* Copy a device state into / out of a msmb_system (device to device). */
int msmb_system_set_state_device(msmb_system* s, const double* state);
int msmb_system_get_state_device(const msmb_system* s, double* state);

/* ---- spatial decomposition plans ----------------------------
 * Work plan of `part` of an nparts-way slab decomposition (msmb_slab_* below; no
 * GPU needed): out = [ncx, cx0, cx1, levels, (d0_k, plane0_k, plane1_k) per level],
 * the part's pair columns [cx0, cx1) and its x-planes on every level;
 * cap >= 4 + 3 * levels. */
int msmb_dd_plan(const msmb_msm_config* cfg, const msmb_units* units, const double box[3], int64_t n,
                 int nparts, int part, int* out, int cap);

/* ---- spatial slab decomposition over GPUs ----------------
 * propagate(spec, s, units) (src/integrate.cpp:13-36) over msm_potential
 * (src/msm.cpp:52-90) split into x-slabs of pair columns, one part per GPU
 * (csrc/msmb_slab.cu).  A part owns the atoms binned into its columns and the
 * x-planes of its slab on every grid level; it keeps halo copies of the atoms its
 * pair lists and anterpolation read, and fetches the lattice planes its stencils
 * read (R = ceil(2a/h) charge planes for the lattice cutoff, the restriction and
 * prolongation windows, the interpolation window; the top level whole).  Per
 * step only halo positions and those planes travel (ncclSend/Recv); at a pair-list
 * rebuild (the single-GPU rule, decided globally) atoms migrate to the part owning
 * their new column.  With the direct lattice method on the single-GPU run the
 * decomposed trajectory is bitwise the single-GPU one; the energy is the sum of
 * the parts' shares in part order.
 *
 * Two transports:
 *  - one process per GPU: nfields = 1, nparts = world size, rank = this process's
 *    rank, and either nccl_id (128 bytes from msmb_nccl_unique_id on rank 0,
 *    distributed by the caller) or nccl_comm (an existing ncclComm_t); also valid
 *    with nparts = 1 (a one-rank communicator);
 *  - local: nfields = nparts fields (distinct handles; typically one per device,
 *    several on one device for tests), all parts driven by this process, the
 *    exchanges as stream-ordered copies; nccl_id / nccl_comm unused.
 * Only MSM fields (no overlay).  With nparts > 1 the lattice cutoff runs as the
 * direct stencil on the owned planes (msmb_set_lattice_method(f, 1) is set). */
typedef struct msmb_slab msmb_slab;
int msmb_nccl_unique_id(void* id128);
int msmb_slab_create(msmb_field* const* fields, int nfields, int nparts, int rank, const void* nccl_id,
                     void* nccl_comm, msmb_slab** out);
void msmb_slab_destroy(msmb_slab* d);
/* Every process passes the caller's whole system (host AoS arrays, as
 * msmb_propagate); on success pos/vel hold the whole final state on every
 * process and *energy the last evaluation's energy.  step_ms (optional, steps + 2
 * entries): device times of the initial evaluation, each step and the closing
 * half-kick on this process's first part.  Errors: the reference's exception of
 * the earliest failing step, the same on every part (msmb_slab_last_error). */
int msmb_slab_propagate(msmb_slab* d, int64_t n, double* pos_xyz, double* vel_xyz, const double* q,
                        const double* mass, const double box[3], double dt, int steps, const msmb_units* units,
                        double* energy, double* step_ms);
/* [0] bytes received per step by one part (max over the call's steps and this
 * process's parts), [1] bytes received in the last rebuild's exchanges, [2] owned
 * atoms and [3] halo atoms of this process's first part, [4] rebuilds, [5] atoms
 * migrated away from this process's parts, [6] parts.  Returns the count written. */
int msmb_slab_stats(msmb_slab* d, int64_t* out, int cap);
int msmb_slab_last_error(const msmb_slab* d, int* kind, int64_t* idx_i, int64_t* idx_j, int* step, char* msg,
                         int cap);

/* ---- measurement ------------------------------------------------------------ */
/* When enabled, every evaluation records CUDA events around each stage on the
 * handle's stream (eager launches, no graph) and accumulates durations. */
int msmb_set_stage_timing(msmb_field* f, int enable);
/* Stage names/times (ms, summed since the last reset) and launch counts.
 * Returns the number of stages (<= cap). */
int msmb_stage_times(msmb_field* f, double* ms, int64_t* launches, const char** names, int cap);
void msmb_reset_stage_times(msmb_field* f);
/* Work counters of the most recent evaluation: [0] in-cutoff unordered pairs
 * P_u, [1] candidate pair tests (both counted by evaluations launched eagerly --
 * evaluate, stage-timing passes; the captured step graphs skip the counting), [2] clusters, [3] clipped lattice taps
 * (all levels except the top), [4] top-level taps, [5] kernel launches per
 * evaluation, [6] pair-list rebuilds since the workspace was created, [7] warps
 * per i-cluster in the pair kernel (1 = the large-system instance). */
int msmb_work_counters(msmb_field* f, int64_t* out, int cap);
/* Device-timed propagate for benchmarking: the same computation as
 * msmb_system_propagate, with CUDA events on the field's stream around the
 * initial evaluation, every step and the closing half-kick (step_ms[0..steps+1]),
 * and an optional >L2 buffer write between them (flush_l2, outside the events).
 * stage_names receives the 11 stage names; stage_ms is zero-filled (per-stage
 * times come from a msmb_set_stage_timing pass). */
int msmb_bench_propagate(msmb_field* f, msmb_system* s, double dt, int steps, int flush_l2,
                         double* step_ms, double* stage_ms, const char** stage_names,
                         int64_t* launches);
/* Sustained FP64 FMA throughput of `device` (TFLOP/s, FMA = 2 flops), measured
 * with an FMA-chain microbenchmark for about `seconds`. */
int msmb_measure_fp64_peak(int device, double seconds, double* tflops);
/* Lattice-cutoff method for levels 0..l-2: 0 (default) = zero-padded FFT
 * convolution, 1 = direct stencil sum as the reference (src/msm_phases.cpp:93-134).
 * Both agree to rounding; the direct sum is kept for comparison and tests. */
int msmb_set_lattice_method(msmb_field* f, int direct);
/* Pair-list skin (A, default 0.2): within one evaluate/propagate call the cluster
 * pair list is built at the first evaluation and rebuilt only once some atom moved
 * more than skin/2; the pair kernel always applies the exact cutoff, so results are
 * the reference's within rounding.  Every call starts from a fresh list, so results
 * are a pure, bitwise-repeatable function of the call's input.
 * skin = 0 rebuilds at every evaluation. */
int msmb_set_pair_skin(msmb_field* f, double skin);
/* reuse = 1: a call whose atoms are still within skin/2 of the last list build
 * keeps that list (saves one rebuild per call when a host loop calls evaluate /
 * propagate step by step); the last bits of the forces then depend on the call
 * history.  Default 0. */
int msmb_set_list_reuse(msmb_field* f, int reuse);
/* Kernel launches issued by this handle since creation. */
int64_t msmb_kernel_launches(const msmb_field* f);

/* Level geometry of the hierarchy built for `box` (src/msm_grid.cpp:24-54):
 * dims[3*l], spacing[l], origin[3*l]. */
int msmb_grid_geometry(const msmb_msm_config* cfg, const double box[3], int* dims,
                       double* spacing, double* origin);

/* Debug/parity hooks (tests only): per-level charge/potential lattices of the
 * last evaluation on `f` (concatenated level 0..l-1), and the level-0 cell
 * triple floor((x - origin) / h) of every particle (the reference's
 * stencil_at base + 1, src/msm_phases.cpp:23). */
int msmb_debug_levels(msmb_field* f, double* level_charge, double* level_potential);
int msmb_debug_cells(msmb_field* f, int64_t n, const double* pos_xyz, const double box[3],
                     int32_t* cells_xyz, int32_t* covered);
/* Runs one stage kernel on caller lattices, for bitwise stage parity:
 * stage 0 restrict (level k -> k+1), 1 lattice cutoff (level k),
 * 2 top level, 3 prolongate (k+1 -> k, `out` holds the fine potential in/out),
 * 4 interpolate (level-0 potential -> per-atom u, uses pos/n); these are the
 * bit-exact variants.  The production kernels an evaluation runs (tolerance
 * tests): 5 restriction chain (in = level-0 charges, out = all levels' charges),
 * 6 top level, 7 prolongation chain (in/out = all levels' potentials). */
int msmb_debug_stage(msmb_field* f, int stage, int k, const double box[3], const double* in,
                     double* out, int64_t n, const double* pos_xyz);
/* The production binning kernel's level-0 cell triples (decoded from its sort
 * keys) and coverage flags, for the bit-exact binning test of the kernel every
 * evaluation runs (msmb_debug_cells runs a stand-alone copy of the formula). */
int msmb_debug_bin_keys(msmb_field* f, int64_t n, const double* pos_xyz, const double box[3],
                        int32_t* cells_xyz, int32_t* covered);

#ifdef __cplusplus
}
#endif
#endif /* MSMB_H */
