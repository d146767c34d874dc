/*
 * citywind_b200 -- C ABI of the B200-native RANS step path.
 *
 * Drop-in boundary for the reference's Python step path
 * (/root/reference/pkg/src/citywind/, "ref" below).  The reference has no
 * native FFI of its own: its hot path is the Python call
 *     solver.step(state, params, psys, preconditioner, profile, advector, pcg_tol)
 * (ref solver.py:407-461) plus the per-design precompute of
 * CompiledScenario (ref scenario.py:364-445).  Each entry point below
 * replaces one of those Python-level interfaces; the Python mirror
 * (paper_2204_01117_b200/_native.py) binds them with ctypes.
 *
 * Conventions
 *  - plain C types only; device buffers are passed as raw device pointers
 *    (void*), streams as cudaStream_t cast to void*.
 *  - every field is x-fastest: a cell field has nx*ny*nz entries with x
 *    fastest; u has (nx+1)*ny*nz, v nx*(ny+1)*nz, w nx*ny*(nz+1).
 *  - "real" buffers are float or double according to the precision the
 *    context was created with (4 or 8).
 *  - functions return CW_OK or an error code; cw_last_error() gives a
 *    thread-local message.  Error codes map to the reference's exceptions
 *    (see the CW_ERR_* comments).
 */
#ifndef CITYWIND_B200_H
#define CITYWIND_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define CW_ABI_VERSION 2

#define CW_OK 0
#define CW_ERR_INVALID 1       /* ValueError: bad argument / shape */
#define CW_ERR_CUDA 2          /* CUDA runtime failure */
#define CW_ERR_SINGULAR 3      /* SingularSystemError, ref linalg.py:23,114-117 */
#define CW_ERR_PCG 4           /* ProjectionError, ref solver.py:113-116,275-276 */
#define CW_ERR_NONFINITE 5     /* FloatingPointError, ref turbulence.py:123-127 */
#define CW_ERR_TIMEOUT 6       /* device grid barrier timed out (never expected) */
#define CW_ERR_RHS 7           /* ValueError non-finite rhs, ref linalg.py:326-327 */
#define CW_ERR_GEOMETRY 8      /* ClassificationError, ref geometry.py:31,236-240 */
#define CW_ERR_HALO 9          /* ValueError: a z-slab window's halo is shallower than the step's
                                  reach 2 floor(max|w| dt/dz) + 4 (report: criterion = max|w| dt/dz,
                                  bad_cell = planes needed) -- the reference's backtrace is unbounded,
                                  ref advection.py:125-142 */

typedef struct cw_ctx cw_ctx;

/* GridSpec, ref grid.py:33-84 */
typedef struct {
  int nx, ny, nz;
  double dx, dy, dz;
  double origin[3];
} cw_grid;

/* SolverParams, ref solver.py:26-50 (inlet k/omega derived host-side) */
typedef struct {
  double dt, nu, cd_tree, cd_building, drag_a, drag_b, drag_eps;
  double c_mu, alpha, beta, sigma, sigma_star, c_lim;
  double k_in, omega_in;       /* SolverParams.inlet_k_omega(), ref solver.py:48-50 */
  int turbulence;
} cw_params;

/* InletProfile, ref solver.py:54-97: speed_at() sampled at cell-centre heights */
typedef struct {
  int kind;                    /* 0 uniform, 1 logarithmic */
  double speed, u_star, z0, kappa;
  double dir_x, dir_y;         /* already normalised (ref solver.py:69-75) */
} cw_inlet;

/* FlowState device buffers, ref grid.py:492-571 */
typedef struct {
  void *u, *v, *w, *p, *k, *omega, *nu_t;   /* real */
  const signed char *labels;                /* int8 CellLabel, ref grid.py:19-29 */
  const void *g;                            /* real per-cell drag coefficient C_d*G */
  int has_drag;                             /* any(g != 0), ref solver.py:157-158 */
  long long labels_version;                 /* != 0: changes whenever the labels content may have
                                               changed; lets the context reuse its boundary-write
                                               lists (0: no reuse, full-volume boundary kernels) */
} cw_fields;

/* StepReport + PcgReport, ref solver.py:101-110, linalg.py:27-31 */
typedef struct {
  int iterations, converged, status;        /* status: CW_OK or a CW_ERR_* code */
  int bad_field;                            /* 0 k, 1 omega when status == CW_ERR_NONFINITE */
  double criterion, cfl, div_before, div_after;
  long long bad_cell;                       /* ref C-order (i*ny+j)*nz+k of first non-finite */
  float ms_total;                           /* device time of the step, when timed */
} cw_report;

int cw_abi_version(void);
const char *cw_last_error(void);

/* Context = one grid on one device. Replaces CompiledScenario's per-grid
 * state (ref scenario.py:364-381). precision: 4 (fp32) or 8 (fp64). */
int cw_ctx_create(const cw_grid *grid, int precision, int device, cw_ctx **out);
void cw_ctx_destroy(cw_ctx *ctx);

/* z-slab decomposition (the reference is single-process, so these
 * have no reference counterpart: they split the grid of one
 * CompiledScenario, ref scenario.py:364-381, over devices).
 * A slab context covers global planes [k_lo - halo, k_hi + halo) clipped to
 * [0, nz) and owns [k_lo, k_hi).  Its fields are that window (x-fastest, the
 * same shapes as a grid of nz_local planes).  Every stage runs on the whole
 * window; reductions and reports cover the owned planes only.  The caller
 * refreshes the halo planes from the neighbours (state at the start of a
 * step, p after the projection).  halo >= 2. */
#define CW_MAX_SLABS 64
#define CW_MAX_CHUNKS 4096   /* PCG z-chunks over all slabs of one solve */
int cw_ctx_create_slab(const cw_grid *global_grid, int k_lo, int k_hi, int halo, int precision,
                       int device, cw_ctx **out);
int cw_slab_info(cw_ctx *ctx, int *kg0, int *nz_local, int *own0, int *own1);

/* Owned-plane sums behind default_projection_tol (ref solver.py:235-243) for
 * combining over slabs: sum of diag(W) (AI1), sum of 1/diag(A) (Jacobi),
 * unknown count, and whether the window has an outlet cell. */
int cw_operator_partials(cw_ctx *ctx, double *wdiag_sum, double *jacobi_sum, long long *n_unknown,
                         int *has_outlet);

/* Device buffers a neighbouring slab writes into (halo planes of the pitched
 * PCG vectors) and the root slab's barrier / value table.  o0, o1: the
 * owner's owned local planes. */
typedef struct {
  void *r0, *r1, *p0, *p1, *z, *Ap;
  void *xbar, *xval;
  int o0, o1;
} cw_slab_buffers;
int cw_slab_buffers_get(cw_ctx *ctx, cw_slab_buffers *out);

/* One device per slab: attach this context as slab `slab` of `nslab` with
 * the neighbours' buffers (NULL z pointer = no neighbour) and the root
 * slab's (slab 0) barrier, as pointers valid on this device (same process,
 * or opened with cw_ipc_open).  The projection then pushes its boundary
 * planes into the neighbours while it computes them and meets the other
 * slabs at the root's barrier (system-scope atomics over NVLink). */
int cw_slab_attach(cw_ctx *ctx, int slab, int nslab, const cw_slab_buffers *lower,
                   const cw_slab_buffers *upper, const cw_slab_buffers *root);

/* The PCG's work split: z-chunks of zc planes times 32 x 32 (x, y) tiles.
 * Dot products are summed per chunk in a fixed tree, then over chunks in
 * global order, so a whole grid and any z-slab split whose slab boundaries
 * fall on chunk boundaries give the same bits.
 * cw_pcg_chunk_of: the chunk size a whole-grid context picks for g;
 * cw_set_pcg_chunk: force a context's chunk size (slab contexts take the
 * whole grid's); cw_slab_chunks: this slab's first chunk in the whole
 * solve's chunk order and the total (cross-device solves; cw_slab_group_pcg
 * sets them itself); cw_pcg_chunks: the current split. */
int cw_pcg_chunk_of(const cw_grid *g, int precision, int device, int *zc);
int cw_set_pcg_chunk(cw_ctx *ctx, int zc);
int cw_slab_chunks(cw_ctx *ctx, int chunk0, int nchunk_g);
int cw_pcg_chunks(cw_ctx *ctx, int *zc, int *nchunk);

/* All slabs on one device: the projection of every slab in one cooperative
 * launch (the same kernel code as the attached multi-device solve, blocks
 * partitioned by slab).  ctxs in z order, fields per slab. */
int cw_slab_group_pcg(cw_ctx **ctxs, const cw_fields *fields, int n, const cw_params *prm,
                      double pcg_tol, void *stream);

/* CUDA IPC for cw_slab_buffers between processes (64-byte handles). */
int cw_ipc_get(void *d_ptr, unsigned char handle[64]);
int cw_ipc_open(const unsigned char handle[64], int device, void **d_ptr);
int cw_ipc_close(void *d_ptr);

/* build_pressure_matrix + build_ai_preconditioner(A, omega, 1, truncate=False)
 * (ref linalg.py:57-126, 201-232; called from scenario.py:377-379), matrix-free:
 * derives the per-cell operator code from labels (device int8).  Returns the
 * unknown count and default_projection_tol (ref solver.py:235-243). */
int cw_set_operator(cw_ctx *ctx, const signed char *d_labels, double ai_omega,
                    long long *n_unknown, double *tol_default, void *stream);

/* Select the preconditioner of the projection: 0 identity (plain CG),
 * 1 Jacobi (build_jacobi, ref linalg.py:194-198), 2 untruncated AI1 (default).
 * Returns the matching default_projection_tol. */
int cw_set_preconditioner(cw_ctx *ctx, int kind, double *tol_default);

/* Drag coefficient per cell, drag_factor_cells (ref solver.py:123-135), from
 * float64 phi/lad (device) into the context-precision buffer g. */
int cw_drag_coefficient(cw_ctx *ctx, const double *d_phi, const double *d_lad,
                        const signed char *d_labels, const cw_params *prm, void *d_g,
                        int *has_drag, void *stream);

/* apply_boundary_conditions (ref solver.py:330-400) on a state. */
int cw_apply_boundary(cw_ctx *ctx, const cw_fields *f, const cw_params *prm,
                      const cw_inlet *inl, void *stream);

/* Enqueue nsteps calls of step() (ref solver.py:407-461) without any host
 * synchronisation; pcg_tol < 0 selects default_projection_tol.  Reports are
 * collected on the device; read them with cw_read_reports. */
int cw_step(cw_ctx *ctx, const cw_fields *f, const cw_params *prm, const cw_inlet *inl,
            double pcg_tol, int nsteps, void *stream);

/* Let the NEXT step enqueued on this ctx start before nu_t and p are on the
 * device: the step waits for nu_t_ready (a cudaEvent_t) before its diffusion,
 * the first stage that reads nu_t, and for p_ready before its first boundary
 * pass, the first stage that touches p.  One-shot; NULL = no wait.  A caller
 * that copies the state in from host memory every step (solver.HostStepper)
 * uploads those two fields while the advection runs.  Same stage order as
 * step() (ref solver.py:407-461); no reference counterpart. */
int cw_step_defer(cw_ctx *ctx, void *nu_t_ready, void *p_ready);

/* With cw_step_defer: let the NEXT step also start before k and omega are on
 * the device.  Their only readers before the projection are the upwind step
 * (advection.py:154-173) and the first boundary pass; the step then saves
 * the old cell-centred velocity in the predictor, runs the projection on
 * u, v, w, p first and waits for k_omega_ready (a cudaEvent_t) only after
 * it, before the upwind step and the k / omega / nu_t writes of the first
 * boundary pass.  Results are bit-identical to the undeferred step.  Needs
 * turbulence-independent composed boundary lists (labels_version != 0);
 * otherwise the step waits for the event before its first stage.  One-shot;
 * NULL = no wait.  No reference counterpart. */
int cw_step_defer_kw(cw_ctx *ctx, void *k_omega_ready);

/* Run ONE stage function of the reference on a state, with dt = prm->dt:
 * advect (advect_velocity + upwind_scalar k/omega, advection.py:125-173),
 * diffuse (solver.py:193-208), apply_drag (:150-168), apply_boundary_conditions
 * (:330-400), project (:246-304, incl. div before/after), update_turbulence
 * (turbulence.py:100-132).  Uses one report slot like a step. */
#define CW_STAGE_ADVECT 1
#define CW_STAGE_DIFFUSE 2
#define CW_STAGE_DRAG 3
#define CW_STAGE_BOUNDARY 4
#define CW_STAGE_PROJECT 5
#define CW_STAGE_TURBULENCE 6
/* a step split around the projection (z-slab steps exchange halos between):
 * PRE = advect, diffuse, drag, boundary; SOLVE = the PCG alone (p on the
 * owned planes); POST = pressure gradient, div after, turbulence, boundary,
 * CFL.  PRE, SOLVE, POST in order equal one step. */
#define CW_STAGE_PRE 7
#define CW_STAGE_POST 8
#define CW_STAGE_SOLVE 9
int cw_run_stage(cw_ctx *ctx, const cw_fields *f, const cw_params *prm, const cw_inlet *inl,
                 int stage, double pcg_tol, void *stream);

/* Synchronise `stream`, copy up to n pending step reports (oldest first) into
 * out, clear them and the error latch.  *n_out = number written.  Returns
 * the status of the first failed step (CW_OK if none). */
int cw_read_reports(cw_ctx *ctx, cw_report *out, int n, int *n_out, void *stream);

/* Layout conversion for a reference-layout caller (refbind.py): the
 * reference's FlowState holds float64 C-order arrays (ex, ey, ez), x slowest
 * (ref grid.py:492-571); device fields are x-fastest (ez, ey, ex) in the
 * context precision.  direction 0: reference float64 (device copy) -> device
 * field; 1: device field -> reference float64.  field 0 u, 1 v, 2 w, 3 a cell
 * field (p, k, omega, nu_t).  Device pointers; no synchronisation. */
int cw_ref_layout(cw_ctx *ctx, int direction, int field, const void *src, void *dst, void *stream);

/* Iteration cap of the projection's PCG (ref project(max_iter=10_000),
 * solver.py:246-249 -> pcg_solve(max_iter), linalg.py:310-368): a solve that
 * has not met the stopping rule after max_iter iterations reports
 * CW_ERR_PCG with iterations == max_iter.  Default 10000. */
int cw_set_max_iter(cw_ctx *ctx, int max_iter);

/* After a step reported CW_ERR_NONFINITE: put the state back as the
 * reference leaves it when update_turbulence raises (ref turbulence.py:121-131,
 * before any assignment) -- k and omega as advected this step, nu_t as before
 * the step.  Synchronises `stream`. */
int cw_turb_rollback(cw_ctx *ctx, const cw_fields *f, void *stream);

/* After a step reported CW_ERR_PCG or CW_ERR_RHS: the state as the reference
 * leaves it when project() raises (ref solver.py:272-276, linalg.py:326-327)
 * -- u, v, w, nu_t, p after the first boundary pass (p is not replaced by a
 * solve that fails), and with turbulence on, k and omega as advected this step
 * with their boundary values (copied from the step's upwind buffers).
 * Synchronises `stream`. */
int cw_proj_rollback(cw_ctx *ctx, const cw_fields *f, int turbulence, void *stream);

/* Per-stage device timings of the next cw_step call (ms per stage, keys of
 * StepReport.timings, ref solver.py:418-454): enable before, read after. */
int cw_set_stage_timing(cw_ctx *ctx, int enabled);
int cw_read_stage_timings(cw_ctx *ctx, float out_ms[7]);

/* Evidence hooks for the benchmark: device time of each PCG launch
 * (CUDA events on the launching stream, first max_launches launches after
 * the call), and the number of kernels this context has enqueued. */
int cw_pcg_timing(cw_ctx *ctx, int max_launches);
int cw_read_pcg_timing(cw_ctx *ctx, float *ms, int n, int *n_out);
/* device time of the MacCormack predictor and corrector launches of the steps
   timed since cw_pcg_timing (bench.py advection roofline); no reference
   counterpart (instrumentation) */
int cw_read_adv_timing(cw_ctx *ctx, float *predict_ms, float *correct_ms, int n, int *n_out);
long long cw_launch_count(cw_ctx *ctx, int reset);

/* region_average_speed (ref solver.py:535-549) for n boxes in one pass:
 * mean cell-centred speed over AIR cells whose centres lie in [lo, hi];
 * count_out[b] = 0 means "region contains no air cells". Deterministic. */
int cw_region_speed(cw_ctx *ctx, const cw_fields *f, int n, const double *lo3n,
                    const double *hi3n, double *mean_out, long long *count_out, void *stream);

/* The trailing window of evaluate_objective (ref optimize.py:93-99,
 * `sums[ri] += region_average_speed(state, r.lo, r.hi)` after every step):
 * while n > 0, every following cw_step adds the n region means of the
 * stepped state to the device array d_sums (float64, in step order) and
 * writes the air-cell counts to d_counts -- no host synchronisation per step.
 * n = 0 turns it off.  Boxes as for cw_region_speed. */
int cw_step_regions(cw_ctx *ctx, int n, const double *lo3n, const double *hi3n, double *d_sums,
                    long long *d_counts);

/* Velocity at physical points, float64 trilinear samples of the staggered
 * grids (the probes of run_simulation, ref scenario.py:473-478, via
 * Advector.velocity_at, ref advection.py:107-111).  Device arrays: pts 3n,
 * out 3n = (u, v, w) per point.  No host synchronisation. */
int cw_probe(cw_ctx *ctx, const cw_fields *f, int n, const double *d_points, double *d_out, void *stream);

/* trace_streamlines (ref solver.py:488-532): one device thread per seed, RK2
 * midpoint steps of step_len along the normalised velocity, ending on domain
 * exit, after max_steps, or below min_speed.  Device outputs: paths
 * [nseeds][max_steps + 1][3], len[nseeds] points per polyline (0 for a seed
 * outside the domain). */
int cw_streamlines(cw_ctx *ctx, const cw_fields *f, int nseeds, const double *d_seeds, double step_len,
                   int max_steps, double min_speed, double *d_paths, int *d_len, void *stream);

/* Voxelizer, ref grid.py:233-325 + scenario.py:327-360 (bit-exact float64).
 * Objects in order; kind 1 building / 2 tree; shape 0 box (lo, hi), shape 1
 * closed triangle mesh given by (verts, tris) slices of the packed arrays.
 * Outputs device buffers: labels (int8, merged with boundary labels), phi, lad
 * (float64).  Returns CW_ERR_GEOMETRY if a point cannot be classified. */
typedef struct {
  int kind, shape;
  double phi, lad;
  double lo[3], hi[3];
  int vert_offset, n_verts, tri_offset, n_tris;
} cw_object;

/* Painted-porosity base layer for the following cw_voxelize calls
 * (decode_painted_porosity, ref grid.py:337-377, combined with the objects by
 * combine_porosity, ref scenario.py:351-360, as in voxelize_design,
 * ref scenario.py:402-412): an 8-bit (ny, nx) raster on the device (row 0 =
 * min-y row), phi = pixel / 255 on planes [0, kmax); an optional tree mask of
 * the same shape (non-zero = TREE with LAD tree_lad).  d_image NULL: open air. */
int cw_set_paint(cw_ctx *ctx, const unsigned char *d_image, const unsigned char *d_tree_mask, int kmax,
                 double tree_lad);

int cw_voxelize(cw_ctx *ctx, const cw_object *objs, int n_obj, const double *verts,
                const int *tris, int subdiv, const signed char *d_boundary_labels,
                signed char *d_labels, double *d_phi, double *d_lad, int *n_overlap_warnings,
                void *stream);

#ifdef __cplusplus
}
#endif
#endif
