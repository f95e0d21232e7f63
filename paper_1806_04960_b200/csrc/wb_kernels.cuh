// wb_kernels.cuh -- device-side data layout, status block and kernel params.
#pragma once
#include <stdint.h>
#include "wb_device.cuh"

namespace wb {

constexpr unsigned long long KEY_NONE = ~0ull;
constexpr int HALO = 2;  // x-halo columns per side (update(i) needs q(i +- 2))

// Device-resident run status.  Every step reads dt inputs from here and the
// finalize kernel commits / stops here, so many steps can be enqueued (or
// captured in a CUDA graph) without a host round trip.
struct Status {
  unsigned long long rmax_bits;       // CFL rate max of the current state
  unsigned long long rmax_next_bits;  // accumulated by the step kernel for q^{n+1}
  unsigned long long key_recon;       // min (i*ny+j) of bad reconstructed faces (code 3)
  unsigned long long key_update;      // min (i*ny+j) of bad updated cells (code 4)
  unsigned long long key_prep;        // min (i*ny+j) of non-admissible states (code 1)
  unsigned long long red[2];          // [~errkey, rmax_next_bits] (MAX-allreduced for N>1)
  unsigned long long n2nd, nxs, nys, nfluid;  // work counters of the last step
  double t, dt, t_end, max_dt, tiny;
  long long step, max_steps;
  int cur;        // index of the buffer holding the current state
  int stop;       // 0 running, >0 error code, -1 target reached
  int mode;       // 0 = free (optional max_dt), 1 = run_until(t_end)
  int has_max_dt;
  int err_code;
  int pad;
  long long err_key, err_step;
  double err_rmax;
  unsigned long long rmax_used_bits;  // rate the last committed step used for dt
  unsigned long long launch_id;       // incremented before every step launch
  unsigned int ticket[2];  // dynamic CTA index of the step kernel, per concurrent launch
  unsigned long long n_replay;  // exact IEEE replays of units (cumulative, never reset)
  unsigned long long n_replay_kind[6];  // the same per unit kind (see WB_REPLAY)
};

struct Geo {
  int nx, ny;          // global grid
  int i_begin;         // global index of the first owned column
  int nxl;             // owned columns
  int ncol;            // stored columns = nxl + 2*HALO
  int pitch;           // doubles per stored row (>= ncol)
  int bcw, bce, bcs, bcn;                 // reconstruction ghost codes
  int kind[4];                            // edge kinds: left right bottom top
  double seg[4][2];
  double inflow[4][4];
  double cfl;
};

struct Bufs {
  double* q[2][4];        // [buffer][component] planes, index j*pitch + c
  const uint8_t* mask;    // j*pitch + c (0 outside the domain)
  double* y0s[2];         // per stored column, detection of buffer b's state
  double* aeqs[2];
  // fused-detection chain: running (sum, aeq, first fluid row) per row
  // segment and column, and a publish flag per (segment, column strip)
  double* ch_sum;
  double* ch_aeq;
  int* ch_jlo;
  unsigned long long* ch_flag;
  int nbx_max;
  int fuse_detect;  // 1: detection of q^{n+1} is chained inside k_step; 0: k_detect per step
  const double* ycent;    // ny
  const double* yfaces;   // ny + 1
  const double* xcent;    // per stored column (x centre, for bottom/top inflow)
  Status* st;
  double* dtlog;          // optional per-step dt log (may be null)
  long long dtlog_cap;
};

// An x-neighbour slab's buffers as seen from this device (k_push_halo);
// q[0][0] == nullptr: no neighbour on that side
struct PeerBufs {
  double* q[2][4];
  double* y0s[2];
  double* aeqs[2];
  int pitch, nxl;
};

// Debug outputs in the reference layout (owned columns, (nxl, ny, 5))
// Column-strip partition of one step launch: launch-local strip k is global
// strip bx0 + k*bxs; tslot picks the ticket counter (two launches of one step
// -- slab-edge strips and interior strips -- run concurrently)
struct Part {
  int bx0, bxs, tslot;
  int nofuse;  // 1: this launch leaves the detection of q^{n+1} to k_detect_cols
};
struct Dbg {
  double *fW, *fE, *fS, *fN, *vol, *psi, *DW, *DE, *DS, *DN;
  uint8_t* quiet;
};

}  // namespace wb
