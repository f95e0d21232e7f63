/*
 * wbflow_b200.h -- C ABI of the B200-native time-stepping hot path.
 *
 * Drop-in boundary: the reference (pkg/src/wbflow, Python + Numba) has no
 * native FFI of its own; its hot-path boundary is the Python driver API in
 * timestepper.py and the Numba kernel entry points in kernels.py.  Each entry
 * point below names the reference interface it replaces.  Conventions:
 * plain C types only, int return status (WB_OK = 0), one opaque handle per
 * simulation (or per x-slab for multi-GPU), all device work stream-ordered on
 * the handle's stream, not thread-safe per handle.  State arrays crossing the
 * boundary use the reference layout (i, j, m) with m fastest and 5
 * components (a*rho, a*rho*u, a*rho*v, alpha, y).
 */
#ifndef WBFLOW_B200_H
#define WBFLOW_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WB_OK 0
#define WB_E_ARG -1       /* invalid argument / configuration */
#define WB_E_CUDA -2      /* CUDA runtime failure */
#define WB_E_HEIGHT -3    /* q[...,4] != y_centers for a fluid cell */
#define WB_E_STATE -4     /* no state uploaded */

/* numerical error codes reported in wb_error.code (timestepper.py:154-158,
 * 181-182, 205-207) */
#define WB_ERR_NONE 0
#define WB_ERR_CELL_STATE 1   /* "non-admissible cell state" */
#define WB_ERR_WAVE_SPEED 2   /* "non-finite wave speed (max rate ...)" */
#define WB_ERR_FACE 3         /* "non-admissible reconstructed face state" */
#define WB_ERR_MASS 4         /* "negative mass or volume fraction after update" */

typedef struct wb_handle wb_handle;

typedef struct {
  int32_t nx, ny;            /* global grid (grid.py:21-38) */
  int32_t i_begin, i_end;    /* owned global columns [i_begin, i_end) (x-slab) */
  double dx, dy;
  double k0, rho0, gamma, g, epsilon; /* params.py:6-21 */
  double cfl;                /* timestepper.py:51 */
  int32_t bc_kind[4];        /* left,right,bottom,top: 1 reflective 2 transmissive 3 inflow */
  double inflow_seg[4][2];   /* grid.py:110-123 segment per side */
  double inflow_q[4][4];     /* conserved inflow state (timestepper.py:33-37) */
  int32_t device;            /* CUDA device ordinal */
  int32_t rows_per_block;    /* 0 = auto */
} wb_config;

typedef struct {
  int32_t code;              /* WB_ERR_* */
  int64_t step;              /* committed steps when the error happened */
  int32_t i, j;              /* first failing cell in i-major order, -1 if none */
  double rmax;               /* the offending rate for WB_ERR_WAVE_SPEED */
} wb_error;

typedef struct {
  double t, dt, rmax;
  int64_t step;
  int32_t stop;              /* 0 running, >0 error code, -1 target reached */
  int32_t cur;
  uint64_t n_second_order, x_faces_solved, y_faces_solved; /* last step */
  uint64_t replays;          /* exact IEEE unit replays since wb_create (cumulative) */
  uint64_t replays_by_kind[6]; /* reconstruction, flux_y(S), x-face, flux_x pair, y-face,
                                  update */
} wb_status;

/* Simulation.__init__ (timestepper.py:51-103): grid, params, boundary and
 * per-face BC classification.  mask is the global (nx, ny) uint8 array
 * (grid.py:35); xcent/ycent/yfaces are grid.x_centers/y_centers/y_faces
 * (grid.py:40-54), passed so the device uses the reference's exact doubles.
 * rho0, k0, c = sqrt(gamma k0 / rho0), c^2, dx and dy must lie in
 * [2^-100, 2^100] (the exact-division scheme's constant range; every
 * physical configuration does): WB_E_ARG otherwise. */
int wb_create(const wb_config* cfg, const uint8_t* mask, const double* xcent,
              const double* ycent, const double* yfaces, wb_handle** out);
int wb_destroy(wb_handle* h);
/* run all work on this CUDA stream (e.g. torch.cuda.current_stream()) */
int wb_set_stream(wb_handle* h, void* cuda_stream);

/* Simulation.q assignment (timestepper.py:64-69): q holds n_cols columns
 * starting at global column i_first, (n_cols, ny, 5); it must cover the owned
 * columns plus the 2-column halo that exists in the domain.  is_device != 0
 * means q is a device pointer.  On WB_E_HEIGHT, *bad_i / *bad_j name the cell. */
int wb_set_state(wb_handle* h, const double* q, int32_t i_first, int32_t n_cols,
                 int32_t is_device, int32_t* bad_i, int32_t* bad_j);
/* Device-side initial condition of the detection-consistent column-equilibrium
 * family (the dambreak / weir / wall-impact / lake configurations; scenario
 * builders after SPEC.md:554-659, host twin: scenarios.py
 * column_equilibrium_state): alpha = alpha_liq in the union of n_boxes
 * (<= 8) closed rectangles {x0, x1, y0, y1} of cell centres, alpha_gas
 * elsewhere; each column's (y0, aeq) detected from alpha as the solver
 * detects (kernels.py:506-520); alpha*rho = aeq * eq_rho(y_c, y0)
 * (kernels.py:53-55), or alpha * gas_rho where alpha <= 10 eps if gas_rho is
 * not NaN; zero momenta.  Replaces wb_set_state (no host build or upload);
 * bit-identical to the host builder. */
int wb_init_column_equilibrium(wb_handle* h, int32_t n_boxes, const double* boxes,
                               double alpha_liq, double alpha_gas, double gas_rho);
/* Simulation.q read (owned columns, (i_end-i_begin, ny, 5)); solid cells come
 * back with the values uploaded for them and q[...,4] = y_centers. */
int wb_get_state(wb_handle* h, double* q, int32_t is_device);
/* which = 0: current state (Simulation.q), 1: the other buffer (Simulation.q_next) */
int wb_get_state_buf(wb_handle* h, double* q, int32_t which, int32_t is_device);
/* one cell of the current state (error messages) */
int wb_get_cell(wb_handle* h, int32_t i, int32_t j, double* q5);

/* Simulation.max_rate / compute_dt (timestepper.py:143-159, 232-237):
 * detection + admissibility + CFL rate max of the current state */
int wb_max_rate(wb_handle* h, double* rmax, wb_error* err);
/* Simulation.detect (timestepper.py:132-135): per-column (y0, aeq), owned */
int wb_get_columns(wb_handle* h, double* y0s, double* aeqs);

/* Simulation.advance (timestepper.py:163-218): one step; max_dt = NaN for
 * none.  On a numerical error the step is not committed (t, step and the
 * state stay at step n) and err->code != 0. */
int wb_advance(wb_handle* h, double max_dt, double* dt_out, wb_error* err);
/* Simulation.run_until (timestepper.py:220-229) without callback, as a
 * device-side loop: t_end = NaN for "no time limit", max_steps < 0 for none,
 * chunk = steps enqueued between host checks (captured in a CUDA graph). */
int wb_run(wb_handle* h, double t_end, int64_t max_steps, int32_t chunk, wb_error* err);
int wb_get_status(wb_handle* h, wb_status* s);
/* Device diagnostics of the current state (deterministic reduction):
 * out9 = {total mass (sum alpha*rho * dx*dy, cf. Simulation.total_mass,
 * timestepper.py:127-130), max|u|, max|v|, min alpha, max alpha,
 * E_rho, E_u, E_v, E_P} where the E_* are max-norm errors against the exact
 * water-at-rest profile of surface level y0_eq (NaN skips) */
int wb_diagnostics(wb_handle* h, double y0_eq, double* out9);
/* depth-averaged velocity u_bar(x) = sum(u alpha dy) / sum(alpha dy) per
 * owned column, fluid cells in j order (the reference has no
 * such function) */
int wb_depth_averaged_velocity(wb_handle* h, double* out_nx);
/* the error that stopped the device-side run (code 0 if none) */
int wb_get_error(wb_handle* h, wb_error* err);
int wb_set_time(wb_handle* h, double t, int64_t step);
/* per-step dt log written by the device (first `cap` steps) */
int wb_get_dt_log(wb_handle* h, double* out, int64_t n);

/* Stage arrays of one step (the reference's fW,fE,fS,fN,vol,psi,quiet,
 * DW,DE,DS,DN, rhoE_c, rhoE_fy work arrays, timestepper.py:82-95): runs the
 * same fused kernel with debug stores enabled; arrays are host pointers in
 * the reference layout for the owned columns (any may be NULL). */
typedef struct {
  double *fW, *fE, *fS, *fN, *vol, *psi, *DW, *DE, *DS, *DN, *rhoE_c, *rhoE_fy;
  uint8_t* quiet;
} wb_stage_arrays;
int wb_advance_debug(wb_handle* h, double max_dt, double* dt_out, wb_error* err,
                     const wb_stage_arrays* out);

/* ---- x-slab multi-GPU building blocks (driven by the host over NCCL) ---- */
/* device address of the 2 x int64 reduction vector [enc(errkey), rate bits],
 * enc(k) = 2^62 - k (0 = no error): a signed-int64 MAX allreduce across
 * ranks between wb_step_local and wb_finalize yields the globally first
 * failing cell (stage precedence included) and the global CFL rate */
int wb_reduce_ptr(wb_handle* h, void** dev_ptr);
int wb_prepare_ptrs(wb_handle* h, void** rmax_bits, void** key_prep);
int wb_prepare_local(wb_handle* h);         /* enqueue detect + prepare (no sync) */
int wb_prepare_pack(wb_handle* h);          /* [enc(key_prep), rmax] -> reduction vector */
int wb_prepare_unpack(wb_handle* h);        /* reduced vector -> key_prep, rmax */
int wb_get_stream(wb_handle* h, void** cuda_stream);
int wb_check_prepare(wb_handle* h, double* rmax, wb_error* err); /* sync + read */
int wb_step_local(wb_handle* h, double max_dt, double t_end, int32_t mode);
int wb_finalize(wb_handle* h);
/* halo buffers: 2 contiguous side blocks of (4 x 2 x ny state doubles
 * (component, column, j) + 2 x (y0, aeq) of those columns) */
int wb_halo_count(wb_handle* h, int64_t* n_doubles);
int wb_pack_halo(wb_handle* h, void* send_dev);
int wb_unpack_halo(wb_handle* h, const void* recv_dev, int32_t have_left, int32_t have_right);
int wb_sync(wb_handle* h);

/* Overlapped step (SURVEY.md 8(e) "Overlap"; replaces the same
 * Simulation.advance, timestepper.py:163-218): the two slab-edge column
 * strips run on the edge stream and their new boundary columns are packed
 * into send_dev while the interior strips run on the handle's stream.
 *   wb_step_begin -> [exchange send/recv on the edge stream]
 *   -> wb_unpack_halo_next -> wb_step_end -> all-reduce -> wb_finalize
 * The halo lands in the step's output buffer, so it is committed (or
 * discarded) together with the step. */
int wb_set_edge_stream(wb_handle* h, void* cuda_stream);
int wb_step_begin(wb_handle* h, double max_dt, double t_end, int32_t mode, void* send_dev);
int wb_unpack_halo_next(wb_handle* h, const void* recv_dev, int32_t have_left,
                        int32_t have_right);
int wb_step_end(wb_handle* h);

/* Halo over peer memory (replaces the pack -> NCCL
 * send/recv -> unpack of the exchange above): the slab's new boundary columns
 * are stored by one kernel straight into the x-neighbours' halo columns of
 * their step output buffer -- NVLink/NVSwitch stores to another GPU's HBM, or
 * plain stores for another slab on the same GPU.  A wb_peer describes a
 * slab's buffers as pointers valid on the calling handle's device. */
typedef struct {
  void* q[2][4];      /* state planes [buffer][component], index j*pitch + c */
  void* y0s[2];       /* per stored column, detection of buffer b */
  void* aeqs[2];
  int32_t pitch, nxl, ny, pad;
} wb_peer;
/* this handle's own buffers (for a peer in the same process) */
int wb_peer_desc(wb_handle* h, wb_peer* out);
/* export this handle's buffers for another process (cudaIpcGetMemHandle):
 * writes WB_PEER_IPC_BYTES bytes to blob */
#define WB_PEER_IPC_BYTES 256
int wb_peer_ipc_export(wb_handle* h, void* blob);
/* open another process's exported buffers on this handle's device (closed by
 * wb_destroy) */
int wb_peer_ipc_open(wb_handle* h, const void* blob, wb_peer* out);
/* the left / right x-neighbour (NULL: none; peer access is enabled when a
 * peer lives on another device) */
int wb_set_peers(wb_handle* h, const wb_peer* left, const wb_peer* right);
/* wb_step_begin with the halo stored into the peers instead of packed: then
 * wb_step_end -> all-reduce -> wb_finalize.  The all-reduce orders the peer
 * stores before any rank's next step, and no rank stores into a buffer a
 * neighbour still reads (the halo goes to the step's output buffer). */
int wb_step_begin_peer(wb_handle* h, double max_dt, double t_end, int32_t mode);
/* the plain step's counterpart: wb_step_local -> wb_push_halo_next ->
 * all-reduce -> wb_finalize */
int wb_push_halo_next(wb_handle* h);

/* ---- measurement ---- */
/* n steps launched one by one with CUDA events on the handle's stream:
 * average device time of the detection kernel, the fused step kernel and the
 * whole step pipeline (ms) */
int wb_profile_steps(wb_handle* h, int32_t n, double* ms_detect, double* ms_step,
                     double* ms_total);
/* self-test of the inlined IEEE division against a/b on n pseudo-random
 * operand pairs (bit patterns, zeros, all binades, subnormals) */
int wb_selftest_div(int32_t device, int64_t n, uint64_t seed, uint64_t* mismatches);
/* the device exp() used by eq_rho (glibc 2.39 restatement) on n host values */
int wb_eval_exp(int32_t device, const double* x, double* y, int64_t n);
/* face solvers on host arrays of state pairs (components 0..3 of each state;
 * both at the same height, as in the time loop), with the handle's physics:
 * kind 0 = osher_x_edge (kernels.py:215-271), kind 1 = or_y_edge
 * (kernels.py:308-425) with aux = (y, y0, aeq) per pair.  dm/dp get D-/D+
 * components 0..3 (component 4 is exactly 0).  For randomized parity tests. */
int wb_eval_faces(wb_handle* h, int32_t kind, int64_t n, const double* qm, const double* qp,
                  const double* aux, double* dm, double* dp);
/* measured FP64 FMA throughput of the device (TFLOP/s, 2 flop per DFMA) */
int wb_fp64_peak(int32_t device, double* tflops);

const char* wb_last_error(void);
int wb_version(void);

#ifdef __cplusplus
}
#endif
#endif
