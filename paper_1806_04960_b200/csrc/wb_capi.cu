// wb_capi.cu -- extern "C" boundary of the B200 hot path (include/wbflow_b200.h).
//
// Host-side runtime: owns the device buffers of one simulation slab, launches
// the step pipeline (detect -> fused step -> finalize) on its own stream,
// captures multi-step chunks in a CUDA graph for device-side run loops, and
// translates device status into the reference's error contract.  No torch
// types cross this boundary.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <algorithm>
#include <string>
#include "../../include/wbflow_b200.h"
#include "wb_kernels.cuh"
#include "wb_step.cu"  // single translation unit: kernels + g_exp_tab


using namespace wb;

static thread_local std::string g_err;

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) {                                                      \
      g_err = std::string(#x) + ": " + cudaGetErrorString(e_);                    \
      return WB_E_CUDA;                                                           \
    }                                                                             \
  } while (0)

namespace {
constexpr int NT = 64;
constexpr long long DTLOG_CAP = 1 << 20;
constexpr size_t PLANE_SHIFT = 2;  // doubles; see wb_create

// small kernel that sets the run parameters in the device status
__global__ void k_set_run(Status* st, int mode, int has_max_dt, double max_dt, double t_end,
                          double tiny, long long max_steps, int reset_stop) {
  st->mode = mode;
  st->has_max_dt = has_max_dt;
  st->max_dt = max_dt;
  st->t_end = t_end;
  st->tiny = tiny;
  st->max_steps = max_steps;
  // a reached target (stop = -1, set by k_finalize at t_end / max_steps) never
  // carries over into the next step; error stops (> 0) stay sticky unless the
  // caller resets them
  if (reset_stop || st->stop < 0) st->stop = 0;
}
__global__ void k_reset_state(Status* st, double t, long long step) {
  st->rmax_bits = 0ull;
  st->rmax_next_bits = 0ull;
  st->key_recon = KEY_NONE;
  st->key_update = KEY_NONE;
  st->key_prep = KEY_NONE;
  st->cur = 0;
  st->stop = 0;
  st->t = t;
  st->step = step;
  st->dt = 0.0;
  st->max_steps = -1;
  st->mode = 0;
  st->has_max_dt = 0;
  st->err_code = 0;
  st->rmax_used_bits = 0ull;
}
__global__ void k_begin_prepare(Status* st) {
  st->rmax_bits = 0ull;
  st->key_prep = KEY_NONE;
  st->stop = 0;
}
__global__ void k_set_time(Status* st, double t, long long step) {
  st->t = t;
  st->step = step;
}
}  // namespace

struct wb_handle {
  Geo G;
  Phys P;
  Bufs B;
  int dev = 0;
  bool g1 = true;
  int L = 64;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t edge = nullptr;  // slab-edge strips + halo exchange (wb_set_edge_stream)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // host transfers: copies on their own stream, double-buffered staging, so
  // the copy of one column chunk overlaps the layout transpose of the other
  cudaStream_t xfer = nullptr;
  cudaEvent_t ev_x0 = nullptr, ev_copy[2] = {nullptr, nullptr}, ev_used[2] = {nullptr, nullptr};
  double* planes = nullptr;
  uint8_t* mask = nullptr;
  // TMA descriptors of the plane stack and the mask, one pair per CTA width
  // (box {NT, 1, 4} / {NT, 1}); index NT / 32 - 1
  CUtensorMap tq[4], tm[4];
  double *y0s = nullptr, *aeqs = nullptr, *ycent = nullptr, *yfaces = nullptr,
         *xcent = nullptr;
  double *ch_sum = nullptr, *ch_aeq = nullptr;
  int* ch_jlo = nullptr;
  unsigned long long* ch_flag = nullptr;
  Status* st = nullptr;
  Status* h_st = nullptr;
  double* dtlog = nullptr;
  unsigned long long* scratch = nullptr;  // [0] bad-height key
  double* tmp = nullptr;                  // AoS staging
  size_t tmp_bytes = 0;
  bool have_state = false;
  bool need_prepare = true;
  // Simulation.y0s / aeqs (timestepper.py:76-77) hold the detection the last
  // advance() used, i.e. of the state *before* that step: after a committed
  // step that is the other buffer's detection, after max_rate() the current.
  bool cols_prev = false;
  double t = 0.0;
  long long step = 0;
  cudaGraphExec_t graph = nullptr;
  int graph_chunk = 0;
  int variant = 0;  // k_step launch configuration (auto, or WB_KSTEP_VARIANT)
  // halo over peer memory: the x-neighbours' buffers, and the allocations of
  // other processes opened here (closed by wb_destroy)
  PeerBufs peer[2] = {};
  void* ipc_open[6] = {};
  int n_ipc_open = 0;
};

// columns per host-transfer chunk: ~128 MB of AoS, a multiple of the
// transpose tile
static int chunk_cols(int ny) {
  long long c = (128LL << 20) / ((long long)ny * 5 * sizeof(double));
  c = std::max(32LL, c / TT * TT);
  return (int)c;
}

// two staging buffers of `bytes` each (h->tmp, h->tmp + bytes) and the
// transfer stream / events
static int ensure_tmp(wb_handle* h, size_t bytes) {
  if (!h->xfer) {
    CK(cudaStreamCreateWithFlags(&h->xfer, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&h->ev_x0, cudaEventDisableTiming));
    for (int b = 0; b < 2; b++) {
      CK(cudaEventCreateWithFlags(&h->ev_copy[b], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&h->ev_used[b], cudaEventDisableTiming));
    }
  }
  if (h->tmp_bytes >= 2 * bytes) return WB_OK;
  if (h->tmp) cudaFree(h->tmp);
  h->tmp = nullptr;
  h->tmp_bytes = 0;
  CK(cudaMalloc(&h->tmp, 2 * bytes));
  h->tmp_bytes = 2 * bytes;
  return WB_OK;
}

static int read_status(wb_handle* h) {
  CK(cudaMemcpyAsync(h->h_st, h->st, sizeof(Status), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  h->t = h->h_st->t;
  h->step = h->h_st->step;
  return WB_OK;
}

static void fill_error(wb_handle* h, wb_error* err) {
  if (!err) return;
  const Status& s = *h->h_st;
  err->code = s.stop > 0 ? s.err_code : WB_ERR_NONE;
  err->step = s.err_step;
  err->i = -1;
  err->j = -1;
  err->rmax = s.err_rmax;
  if (s.stop > 0 && s.err_key >= 0) {
    err->i = (int32_t)(s.err_key / h->G.ny);
    err->j = (int32_t)(s.err_key % h->G.ny);
  }
}

static dim3 step_grid(const wb_handle* h, int nt) {
  return dim3((h->G.nxl + nt - 2 * HALO - 1) / (nt - 2 * HALO), (h->G.ny + h->L - 1) / h->L);
}

// TMA descriptors (cuTensorMapEncodeTiled through the runtime's driver entry
// point, so the library needs no -lcuda).  q: 3-D {pitch, ny, 8 planes}
// FP64 with box {nt, 1, 4} (plane coordinate cur*4 selects the buffer);
// mask: 2-D {pitch, ny} u8 with box {nt + 16, 1}.  Out-of-range rows / columns
// are zero-filled.
static int make_tensor_maps(wb_handle* h) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult qr;
    void* fn = nullptr;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr));
    if (qr != cudaDriverEntryPointSuccess || !fn) {
      g_err = "cuTensorMapEncodeTiled not available";
      return WB_E_CUDA;
    }
    encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  const Geo& G = h->G;
  const size_t plane = (size_t)G.pitch * G.ny;
  for (int k = 0; k < 4; k++) {
    const cuuint32_t nt = 32u * (k + 1);
    cuuint64_t qdim[3] = {(cuuint64_t)G.pitch, (cuuint64_t)G.ny, 8};
    cuuint64_t qstr[2] = {(cuuint64_t)G.pitch * sizeof(double), plane * sizeof(double)};
    cuuint32_t qbox[3] = {nt, 1, 4};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = encode(&h->tq[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, h->B.q[0][0], qdim, qstr,
                        qbox, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      g_err = "cuTensorMapEncodeTiled (state planes) failed";
      return WB_E_CUDA;
    }
    cuuint64_t mdim[2] = {(cuuint64_t)G.pitch, (cuuint64_t)G.ny};
    cuuint64_t mstr[1] = {(cuuint64_t)G.pitch};
    cuuint32_t mbox[2] = {nt + 16, 1};  // starts at a 16-column boundary (see k_step)
    r = encode(&h->tm[k], CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, h->mask, mdim, mstr, mbox, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      g_err = "cuTensorMapEncodeTiled (mask) failed";
      return WB_E_CUDA;
    }
  }
  return WB_OK;
}

// dynamic shared memory of every built k_step instantiation (> 48 KB needs
// the opt-in attribute)
template <int NTV, int MB, bool G1, bool DBG>
static cudaError_t step_attr() {
  cudaError_t e = cudaFuncSetAttribute(k_step<NTV, MB, G1, DBG>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       step_smem_bytes<NTV>());
  if (e != cudaSuccess) return e;
  // the shared-memory rings are the point: prefer the largest carveout
  return cudaFuncSetAttribute(k_step<NTV, MB, G1, DBG>,
                              cudaFuncAttributePreferredSharedMemoryCarveout,
                              (int)cudaSharedmemCarveoutMaxShared);
}
template <int NTV, int MB, bool G1>
static cudaError_t push_attr() {
  cudaError_t e = cudaFuncSetAttribute(k_step_push<NTV, MB, G1>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       step_smem_bytes<NTV>());
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_step_push<NTV, MB, G1>,
                              cudaFuncAttributePreferredSharedMemoryCarveout,
                              (int)cudaSharedmemCarveoutMaxShared);
}
static int init_step_kernels() {
  CK((push_attr<128, 3, true>()));
  CK((push_attr<64, 1, true>()));
  CK((push_attr<64, 1, false>()));
  CK((step_attr<64, 1, true, false>()));
  CK((step_attr<64, 1, true, true>()));
  CK((step_attr<64, 1, false, false>()));
  CK((step_attr<64, 1, false, true>()));
  CK((step_attr<128, 2, true, false>()));
  CK((step_attr<128, 3, true, false>()));
  CK((step_attr<96, 4, true, false>()));
  CK((step_attr<32, 12, true, false>()));
#ifdef WB_EXPERIMENTS
  CK((step_attr<64, 6, true, false>()));
  CK((step_attr<64, 8, true, false>()));
  CK((step_attr<128, 4, true, false>()));
  CK((step_attr<32, 8, true, false>()));
  CK(cudaFuncSetAttribute(k_step_r<64, 200, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          step_smem_bytes<64>()));
  CK(cudaFuncSetAttribute(k_step_r<64, 224, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          step_smem_bytes<64>()));
#endif
  return WB_OK;
}

// CTA width of each launch variant (WB_KSTEP_VARIANT)
static const int kVariantNT[11] = {64, 64, 64, 128, 128, 32, 128, 96, 64, 64, 32};
// variants compiled into this build (the others need -DWB_EXPERIMENTS)
static bool variant_built(int v) {
#ifdef WB_EXPERIMENTS
  return v >= 0 && v < 11;
#else
  return v == 0 || v == 3 || v == 5 || v == 6 || v == 7;
#endif
}
static int step_nt(const wb_handle* h, bool debug) {
  if (!h->g1 || debug) return 64;
  return (h->variant >= 0 && h->variant < 11) ? kVariantNT[h->variant] : 64;
}

// Which column strips of the step grid a launch covers: all of them, only the
// two slab-edge strips (they produce the columns the x-neighbours need), or
// the interior strips (run concurrently with the edge strips' halo exchange).
enum { PART_ALL = 0, PART_EDGE = 1, PART_INTERIOR = 2 };

// whether the edge launch can store the halo into the peers itself
// (k_step_push is built for the default variants; tiny slabs, whose two
// halo-source column pairs overlap, use k_push_halo)
static bool edge_push_built(const wb_handle* h) {
  return (h->peer[0].q[0][0] || h->peer[1].q[0][0]) && h->G.nxl >= 2 * HALO &&
         (!h->g1 || h->variant == 0 || h->variant == 3);
}

template <bool DEBUG>
static void launch_step(wb_handle* h, const Dbg& D, cudaStream_t s = nullptr,
                        int which = PART_ALL, bool push = false) {
  if (!s) s = h->stream;
  const Geo& G = h->G;
  const int nt = step_nt(h, DEBUG);
  dim3 g = step_grid(h, nt);
  Part part{0, 1, 0, 0};
  // the edge launch must produce both halo-source column pairs: split only if
  // there is an interior strip and the last strip owns at least HALO columns
  const bool split = g.x >= 3 && h->G.nxl - ((int)g.x - 1) * (nt - 2 * HALO) >= HALO;
  if (which == PART_EDGE) {
    // split: the edge strips detect their columns with k_detect_cols (a
    // 256-link fused chain over two strips would be the edge stream's
    // critical path); unsplit, this launch is the whole step and fuses it
    part = split ? Part{0, (int)g.x - 1, 1, 1} : Part{0, 1, 1, 0};
    if (split) g.x = 2;
  } else if (which == PART_INTERIOR) {
    if (!split) return;
    part = Part{1, 1, 0, 0};
    g.x -= 2;
  }
#define WB_LAUNCH(K, NTV)                                                          \
  K<<<g, NTV, step_smem_bytes<NTV>(), s>>>(G, h->B, h->P, h->L, D, part, h->tq[NTV / 32 - 1], \
                                          h->tm[NTV / 32 - 1])
#define WB_LAUNCH_PUSH(K, NTV)                                                             \
  K<<<g, NTV, step_smem_bytes<NTV>(), s>>>(G, h->B, h->P, h->L, D, part, h->tq[NTV / 32 - 1], \
                                          h->tm[NTV / 32 - 1], h->peer[0], h->peer[1])
  if (!DEBUG && push) {  // the slab-edge launch, storing the halo into the peers
    if (!h->g1) WB_LAUNCH_PUSH((k_step_push<64, 1, false>), 64);
    else if (h->variant == 3) WB_LAUNCH_PUSH((k_step_push<128, 3, true>), 128);
    else WB_LAUNCH_PUSH((k_step_push<64, 1, true>), 64);
    return;
  }
#undef WB_LAUNCH_PUSH
  if (!h->g1) {
    WB_LAUNCH((k_step<64, 1, false, DEBUG>), 64);
    return;
  }
  if (DEBUG) {
    WB_LAUNCH((k_step<64, 1, true, true>), 64);
    return;
  }
  switch (h->variant) {
    case 3: WB_LAUNCH((k_step<128, 3, true, false>), 128); break;
    case 5: WB_LAUNCH((k_step<32, 12, true, false>), 32); break;
    case 6: WB_LAUNCH((k_step<128, 2, true, false>), 128); break;
    case 7: WB_LAUNCH((k_step<96, 4, true, false>), 96); break;
#ifdef WB_EXPERIMENTS
    case 1: WB_LAUNCH((k_step<64, 6, true, false>), 64); break;
    case 2: WB_LAUNCH((k_step<64, 8, true, false>), 64); break;
    case 4: WB_LAUNCH((k_step<128, 4, true, false>), 128); break;
    case 8: WB_LAUNCH((k_step_r<64, 200, true>), 64); break;
    case 9: WB_LAUNCH((k_step_r<64, 224, true>), 64); break;
    case 10: WB_LAUNCH((k_step<32, 8, true, false>), 32); break;
#endif
    default: WB_LAUNCH((k_step<64, 1, true, false>), 64);
  }
#undef WB_LAUNCH
}

static void launch_detect(wb_handle* h) {
  // the pitch is a multiple of 32 and the mask is zero outside the domain,
  // so whole 32-column groups can be streamed
  k_detect_coop<<<h->G.pitch / 32, 256, DET_SMEM, h->stream>>>(h->G, h->B, h->P.dy);
}

// One step: detection of the current state comes from the previous step's
// fused chain (or from the prepare after an upload).
static void enqueue_step(wb_handle* h) {
  if (!h->B.fuse_detect) launch_detect(h);
  k_reset_counters<<<1, 1, 0, h->stream>>>(h->st);
  launch_step<false>(h, Dbg{});
  k_prefinalize<<<1, 1, 0, h->stream>>>(h->st);
  k_finalize<<<1, 1, 0, h->stream>>>(h->st, h->G.cfl, h->dtlog, DTLOG_CAP);
}

// detect + admissibility/rate of the current state; sets code 1 / 2 errors
static int do_prepare(wb_handle* h, double* rmax, wb_error* err) {
  h->cols_prev = false;
  k_begin_prepare<<<1, 1, 0, h->stream>>>(h->st);
  launch_detect(h);
  if (h->g1)
    k_prepare<true><<<148 * 4, 256, 0, h->stream>>>(h->G, h->B, h->P);
  else
    k_prepare<false><<<148 * 4, 256, 0, h->stream>>>(h->G, h->B, h->P);
  CK(cudaGetLastError());
  int rc = read_status(h);
  if (rc) return rc;
  Status& s = *h->h_st;
  double r = 0.0;
  unsigned long long b = s.rmax_bits;
  memcpy(&r, &b, 8);
  if (rmax) *rmax = r;
  if (err) {
    err->code = WB_ERR_NONE;
    err->i = err->j = -1;
    err->step = s.step;
    err->rmax = r;
    if (s.key_prep != KEY_NONE) {
      err->code = WB_ERR_CELL_STATE;
      err->i = (int32_t)(s.key_prep / h->G.ny);
      err->j = (int32_t)(s.key_prep % h->G.ny);
    } else if (!(isfinite(r) && r > 0.0)) {
      err->code = WB_ERR_WAVE_SPEED;
    }
  }
  return WB_OK;
}

extern "C" {

const char* wb_last_error(void) { return g_err.c_str(); }
int wb_version(void) { return 1; }

static int create_body(wb_handle* h, const wb_config* cfg, const uint8_t* mask,
                       const double* xcent, const double* ycent, const double* yfaces);

int wb_create(const wb_config* cfg, const uint8_t* mask, const double* xcent,
              const double* ycent, const double* yfaces, wb_handle** out) {
  if (!cfg || !mask || !xcent || !ycent || !yfaces || !out) return WB_E_ARG;
  if (cfg->nx < 2 || cfg->ny < 2 || cfg->i_begin < 0 || cfg->i_end > cfg->nx ||
      cfg->i_end <= cfg->i_begin || !(cfg->cfl > 0.0 && cfg->cfl < 1.0)) {
    g_err = "invalid wb_config";
    return WB_E_ARG;
  }
  wb_handle* h = new wb_handle();
  h->dev = cfg->device;
  const int rc = create_body(h, cfg, mask, xcent, ycent, yfaces);
  if (rc != WB_OK) {  // e.g. out of device memory: release what was allocated
    const std::string msg = g_err;
    wb_destroy(h);
    g_err = msg;
    return rc;
  }
  *out = h;
  return WB_OK;
}

static int create_body(wb_handle* h, const wb_config* cfg, const uint8_t* mask,
                       const double* xcent, const double* ycent, const double* yfaces) {
  CK(cudaSetDevice(h->dev));
  static bool tab_done[64] = {false};
  if (h->dev < 64 && !tab_done[h->dev]) {
    CK(cudaMemcpyToSymbol(g_exp_tab, WB_EXP_TAB, sizeof(WB_EXP_TAB)));
    tab_done[h->dev] = true;
  }
  CK(cudaFuncSetAttribute(k_detect_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, DET_SMEM));
  CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  h->own_stream = true;

  Geo& G = h->G;
  memset(&G, 0, sizeof(G));
  G.nx = cfg->nx;
  G.ny = cfg->ny;
  G.i_begin = cfg->i_begin;
  G.nxl = cfg->i_end - cfg->i_begin;
  G.ncol = G.nxl + 2 * HALO;
  G.pitch = (G.ncol + 31) / 32 * 32;
  for (int s = 0; s < 4; s++) {
    G.kind[s] = cfg->bc_kind[s];
    G.seg[s][0] = cfg->inflow_seg[s][0];
    G.seg[s][1] = cfg->inflow_seg[s][1];
    for (int m = 0; m < 4; m++) G.inflow[s][m] = cfg->inflow_q[s][m];
  }
  // reconstruction ghost codes: reflective -> 1, everything else -> 2
  // (timestepper.py:98-101)
  G.bcw = cfg->bc_kind[0] == BC_REFL ? BC_REFL : BC_TRANS;
  G.bce = cfg->bc_kind[1] == BC_REFL ? BC_REFL : BC_TRANS;
  G.bcs = cfg->bc_kind[2] == BC_REFL ? BC_REFL : BC_TRANS;
  G.bcn = cfg->bc_kind[3] == BC_REFL ? BC_REFL : BC_TRANS;
  G.cfl = cfg->cfl;

  Phys& P = h->P;
  P.k0 = cfg->k0;
  P.rho0 = cfg->rho0;
  P.gamma = cfg->gamma;
  P.g = cfg->g;
  P.eps = cfg->epsilon;
  P.c2ref = cfg->k0 / cfg->rho0;
  P.cref = sqrt(P.c2ref);
  P.grk = cfg->g * cfg->rho0 / cfg->k0;
  P.neg_grk = -P.grk;
  P.athr = 10.0 * cfg->epsilon;
  P.dx = cfg->dx;
  P.dy = cfg->dy;
  P.hx = 0.5 * cfg->dx;
  P.hy = 0.5 * cfg->dy;
  P.rdx2 = 1.0 / (2.0 * cfg->dx);
  P.rdy2 = 1.0 / (2.0 * cfg->dy);
  P.area = cfg->dx * cfg->dy;
  P.rho_lo = 0.5 * cfg->rho0;
  P.rho_hi = 2.0 * cfg->rho0;
  // vmax = 2 sqrt(sound_c2(rho0)) (kernels.py:1237); sound_c2(rho0) for any
  // gamma is gamma*k0/rho0*(1)^(gamma-1)
  double c2r = cfg->gamma == 1.0 ? cfg->k0 / cfg->rho0
                                 : cfg->gamma * cfg->k0 / cfg->rho0 * pow(1.0, cfg->gamma - 1.0);
  P.vmax = 2.0 * sqrt(c2r);
  P.c2c = P.cref * P.cref;
  P.halfc = 0.5 / P.cref;
  h->g1 = cfg->gamma == 1.0;
  {
    double* d;
    double hv[5];
    CK(cudaMalloc(&d, 5 * sizeof(double)));
    k_init_rcp<<<1, 1, 0, h->stream>>>(d, P.rho0, P.cref, P.c2c, P.dx, P.dy);
    CK(cudaMemcpyAsync(hv, d, sizeof(hv), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    cudaFree(d);
    P.yrho0 = hv[0]; P.ycref = hv[1]; P.yc2c = hv[2]; P.ydx = hv[3]; P.ydy = hv[4];
  }
  {
    // FastDiv::divc assumes positive constant divisors in [2^-100, 2^100];
    // the range arguments of divc_q also use k0 and c^2 = gamma k0 / rho0 there
    const double lo = ldexp(1.0, -100), hi = ldexp(1.0, 100);
    const double cs[7] = {P.rho0, P.cref, P.c2c, P.dx, P.dy, P.k0, P.c2ref};
    for (double v : cs)
      if (!(v >= lo && v <= hi)) {
        g_err = "rho0, k0, c, c^2, dx, dy must lie in [2^-100, 2^100]";
        return WB_E_ARG;
      }
  }

  const size_t plane = (size_t)G.pitch * G.ny;
  // PLANE_SHIFT doubles in front of the stack: stored column HALO (the first
  // owned one) then starts a 32-B sector, so every CTA strip's owned columns
  // (a multiple of 4 doubles wide) write whole sectors
  CK(cudaMalloc(&h->planes, (8 * plane + 2 * PLANE_SHIFT) * sizeof(double)));
  CK(cudaMemsetAsync(h->planes, 0, (8 * plane + 2 * PLANE_SHIFT) * sizeof(double), h->stream));
  for (int b = 0; b < 2; b++)
    for (int m = 0; m < 4; m++) h->B.q[b][m] = h->planes + PLANE_SHIFT + (b * 4 + m) * plane;
  // mask in device layout (j, stored column), zero outside the domain
  {
    uint8_t* hm = (uint8_t*)calloc(plane, 1);
    for (int c = 0; c < G.ncol; c++) {
      int gi = G.i_begin + c - HALO;
      if (gi < 0 || gi >= G.nx) continue;
      for (int j = 0; j < G.ny; j++) hm[(size_t)j * G.pitch + c] = mask[(size_t)gi * G.ny + j];
    }
    CK(cudaMalloc(&h->mask, plane));
    cudaError_t e = cudaMemcpy(h->mask, hm, plane, cudaMemcpyHostToDevice);
    free(hm);
    CK(e);
  }
  CK(cudaMalloc(&h->y0s, 2 * G.pitch * sizeof(double)));
  CK(cudaMalloc(&h->aeqs, 2 * G.pitch * sizeof(double)));
  CK(cudaMemset(h->y0s, 0, 2 * G.pitch * sizeof(double)));
  CK(cudaMemset(h->aeqs, 0, 2 * G.pitch * sizeof(double)));
  CK(cudaMalloc(&h->ycent, G.ny * sizeof(double)));
  CK(cudaMalloc(&h->yfaces, (G.ny + 1) * sizeof(double)));
  CK(cudaMemcpy(h->ycent, ycent, G.ny * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(h->yfaces, yfaces, (G.ny + 1) * sizeof(double), cudaMemcpyHostToDevice));
  {
    double* hx = (double*)calloc(G.pitch, sizeof(double));
    for (int c = 0; c < G.ncol; c++) {
      int gi = G.i_begin + c - HALO;
      if (gi >= 0 && gi < G.nx) hx[c] = xcent[gi];
    }
    CK(cudaMalloc(&h->xcent, G.pitch * sizeof(double)));
    cudaError_t e = cudaMemcpy(h->xcent, hx, G.pitch * sizeof(double), cudaMemcpyHostToDevice);
    free(hx);
    CK(e);
  }
  CK(cudaMalloc(&h->st, sizeof(Status)));
  CK(cudaMemsetAsync(h->st, 0, sizeof(Status), h->stream));  // counters, tickets, launch id
  CK(cudaHostAlloc(&h->h_st, sizeof(Status), cudaHostAllocDefault));
  CK(cudaMalloc(&h->dtlog, DTLOG_CAP * sizeof(double)));
  CK(cudaMalloc(&h->scratch, 4 * sizeof(unsigned long long)));
  k_reset_state<<<1, 1, 0, h->stream>>>(h->st, 0.0, 0);
  CK(cudaGetLastError());

  Bufs& B = h->B;
  B.mask = h->mask;
  {
    int rc = make_tensor_maps(h);
    if (rc) return rc;
    rc = init_step_kernels();
    if (rc) return rc;
  }
  B.y0s[0] = h->y0s;
  B.y0s[1] = h->y0s + G.pitch;
  B.aeqs[0] = h->aeqs;
  B.aeqs[1] = h->aeqs + G.pitch;
  B.ycent = h->ycent;
  B.yfaces = h->yfaces;
  B.xcent = h->xcent;
  B.st = h->st;
  B.dtlog = h->dtlog;
  B.dtlog_cap = DTLOG_CAP;

  int L = cfg->rows_per_block > 0 ? cfg->rows_per_block : 64;
  if (const char* v = getenv("WB_KSTEP_VARIANT")) {
    h->variant = atoi(v);
    if (!variant_built(h->variant)) {
      g_err = "WB_KSTEP_VARIANT names a launch variant that is not built";
      return WB_E_ARG;
    }
  } else {
    // 128-thread CTAs (124 owned columns) halve the redundant halo columns of
    // the 64-thread ones once the grid is large enough to keep several such
    // CTAs per SM busy at 64 rows per CTA; with the row state in shared
    // memory (162 registers) three of them fit per SM (12 warps)
    const long long ctas128 = (long long)((G.nxl + 123) / 124) * ((G.ny + 63) / 64);
    h->variant = ctas128 >= 148 * 4 ? 3 : 0;
  }
  const int nt = (h->variant >= 0 && h->variant < 11) ? kVariantNT[h->variant] : 64;
  // keep at least ~4 CTAs per SM on small grids: a CTA marches its rows
  // sequentially, so on a small grid the step time is the row latency times
  // the rows per CTA (C1 200x100: 0.093 ms/step at 8 rows, 0.055 at 2)
  int bx = (G.nxl + nt - 2 * HALO - 1) / (nt - 2 * HALO);
  if (const char* v = getenv("WB_ROWS")) L = atoi(v);
  else if (cfg->rows_per_block <= 0)
    while (L > 2 && (long long)bx * ((G.ny + L - 1) / L) < 148 * 4) L /= 2;
  if (L > 64) L = 64;  // the fused detection keeps one fluid bit per row
  h->L = L;
  {
    const int nby = (G.ny + L - 1) / L;
    const int nbx_max = (G.nxl + 32 - 2 * HALO - 1) / (32 - 2 * HALO) + 1;  // smallest CTA width
    CK(cudaMalloc(&h->ch_sum, (size_t)nby * G.pitch * sizeof(double)));
    CK(cudaMalloc(&h->ch_aeq, (size_t)nby * G.pitch * sizeof(double)));
    CK(cudaMalloc(&h->ch_jlo, (size_t)nby * G.pitch * sizeof(int)));
    CK(cudaMalloc(&h->ch_flag, (size_t)nby * nbx_max * sizeof(unsigned long long)));
    CK(cudaMemset(h->ch_flag, 0, (size_t)nby * nbx_max * sizeof(unsigned long long)));
    h->B.ch_sum = h->ch_sum;
    h->B.ch_aeq = h->ch_aeq;
    h->B.ch_jlo = h->ch_jlo;
    h->B.ch_flag = h->ch_flag;
    h->B.nbx_max = nbx_max;
    // Fused (chained) detection pays ~1-3 us per row segment on the critical
    // path; the separate column-sequential detect pays ~1.7 us per 32 rows.
    // Chain when the columns are long relative to the segment count.
    h->B.fuse_detect = G.ny >= 2048 ? 1 : 0;
    if (const char* v = getenv("WB_FUSE_DETECT")) h->B.fuse_detect = atoi(v) ? 1 : 0;
  }
  CK(cudaStreamSynchronize(h->stream));
  return WB_OK;
}

int wb_destroy(wb_handle* h) {
  if (!h) return WB_OK;
  cudaSetDevice(h->dev);
  if (h->stream) cudaStreamSynchronize(h->stream);
  if (h->graph) cudaGraphExecDestroy(h->graph);
  cudaFree(h->planes);
  cudaFree(h->mask);
  cudaFree(h->y0s);
  cudaFree(h->aeqs);
  cudaFree(h->ch_sum);
  cudaFree(h->ch_aeq);
  cudaFree(h->ch_jlo);
  cudaFree(h->ch_flag);
  cudaFree(h->ycent);
  cudaFree(h->yfaces);
  cudaFree(h->xcent);
  cudaFree(h->st);
  cudaFreeHost(h->h_st);
  cudaFree(h->dtlog);
  cudaFree(h->scratch);
  if (h->tmp) cudaFree(h->tmp);
  if (h->xfer) {
    cudaStreamDestroy(h->xfer);
    cudaEventDestroy(h->ev_x0);
    for (int b = 0; b < 2; b++) {
      cudaEventDestroy(h->ev_copy[b]);
      cudaEventDestroy(h->ev_used[b]);
    }
  }
  for (int k = 0; k < h->n_ipc_open; k++) cudaIpcCloseMemHandle(h->ipc_open[k]);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  delete h;
  return WB_OK;
}

int wb_set_stream(wb_handle* h, void* s) {
  if (!h) return WB_E_ARG;
  CK(cudaStreamSynchronize(h->stream));
  if (h->own_stream) cudaStreamDestroy(h->stream);
  h->stream = (cudaStream_t)s;
  h->own_stream = false;
  if (h->graph) {
    cudaGraphExecDestroy(h->graph);
    h->graph = nullptr;
  }
  return WB_OK;
}

int wb_set_state(wb_handle* h, const double* q, int32_t i_first, int32_t n_cols,
                 int32_t is_device, int32_t* bad_i, int32_t* bad_j) {
  if (!h || !q || n_cols <= 0) return WB_E_ARG;
  const Geo& G = h->G;
  int need_lo = std::max(0, G.i_begin - HALO);
  int need_hi = std::min(G.nx, G.i_begin + G.nxl + HALO);
  if (i_first > need_lo || i_first + n_cols < need_hi) {
    g_err = "wb_set_state: q does not cover the owned columns plus halo";
    return WB_E_ARG;
  }
  CK(cudaSetDevice(h->dev));
  CK(cudaMemsetAsync(h->scratch, 0xff, sizeof(unsigned long long), h->stream));
  if (is_device) {
    k_aos_to_planes<<<dim3((n_cols + TT - 1) / TT, (G.ny + TT - 1) / TT), 256, 0,
                      h->stream>>>(h->G, h->B, q, i_first, n_cols, h->scratch);
  } else {
    // host source: column chunks through two ~128 MB device staging buffers
    // (instead of a full 40 B/cell AoS copy on the device); chunk i is copied
    // on the transfer stream into buffer i % 2 once the transpose of chunk
    // i - 2 has released it, and transposed on the handle's stream once copied
    const int ch = chunk_cols(G.ny);
    const size_t cb = (size_t)ch * G.ny * 5;
    int rc = ensure_tmp(h, cb * sizeof(double));
    if (rc) return rc;
    CK(cudaEventRecord(h->ev_x0, h->stream));
    CK(cudaStreamWaitEvent(h->xfer, h->ev_x0, 0));
    for (int k = 0, i = 0; k < n_cols; k += ch, i++) {
      const int nk = std::min(ch, n_cols - k), b = i & 1;
      double* buf = h->tmp + b * cb;
      if (i >= 2) CK(cudaStreamWaitEvent(h->xfer, h->ev_used[b], 0));
      CK(cudaMemcpyAsync(buf, q + (size_t)k * G.ny * 5, (size_t)nk * G.ny * 5 * sizeof(double),
                         cudaMemcpyHostToDevice, h->xfer));
      CK(cudaEventRecord(h->ev_copy[b], h->xfer));
      CK(cudaStreamWaitEvent(h->stream, h->ev_copy[b], 0));
      k_aos_to_planes<<<dim3((nk + TT - 1) / TT, (G.ny + TT - 1) / TT), 256, 0, h->stream>>>(
          h->G, h->B, buf, i_first + k, nk, h->scratch);
      CK(cudaEventRecord(h->ev_used[b], h->stream));
    }
  }
  CK(cudaGetLastError());
  unsigned long long bad = 0;
  CK(cudaMemcpyAsync(&bad, h->scratch, 8, cudaMemcpyDeviceToHost, h->stream));
  k_reset_state<<<1, 1, 0, h->stream>>>(h->st, h->t, h->step);
  CK(cudaStreamSynchronize(h->stream));
  h->need_prepare = true;
  if (bad != KEY_NONE) {
    if (bad_i) *bad_i = (int32_t)(bad / G.ny);
    if (bad_j) *bad_j = (int32_t)(bad % G.ny);
    h->have_state = false;
    g_err = "q[..., 4] must equal grid.y_centers for fluid cells";
    return WB_E_HEIGHT;
  }
  h->have_state = true;
  return WB_OK;
}

int wb_init_column_equilibrium(wb_handle* h, int32_t n_boxes, const double* boxes,
                               double alpha_liq, double alpha_gas, double gas_rho) {
  if (!h || n_boxes < 0 || n_boxes > IC_MAX_BOXES || (n_boxes && !boxes)) {
    g_err = "wb_init_column_equilibrium: at most 8 boxes";
    return WB_E_ARG;
  }
  CK(cudaSetDevice(h->dev));
  IcBoxes ib{};
  ib.n = n_boxes;
  for (int k = 0; k < n_boxes; k++)
    for (int m = 0; m < 4; m++) ib.b[k][m] = boxes[4 * k + m];
  ib.alpha_liq = alpha_liq;
  ib.alpha_gas = alpha_gas;
  k_reset_state<<<1, 1, 0, h->stream>>>(h->st, h->t, h->step);  // buffer 0 current
  k_ic_alpha<<<148 * 8, 256, 0, h->stream>>>(h->G, h->B, ib);
  launch_detect(h);  // (y0, aeq) of every stored column, like the solver's detection
  k_ic_rho<<<148 * 8, 256, 0, h->stream>>>(h->G, h->B, h->P, gas_rho);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(h->stream));
  h->need_prepare = true;
  h->have_state = true;
  return WB_OK;
}

int wb_get_state(wb_handle* h, double* q, int32_t is_device) {
  return wb_get_state_buf(h, q, 0, is_device);
}

int wb_get_state_buf(wb_handle* h, double* q, int32_t which, int32_t is_device) {
  if (!h || !q) return WB_E_ARG;
  if (!h->have_state) return WB_E_STATE;
  CK(cudaSetDevice(h->dev));
  const Geo& G = h->G;
  if (is_device) {
    k_planes_to_aos<<<dim3((G.nxl + TT - 1) / TT, (G.ny + TT - 1) / TT), 256, 0, h->stream>>>(
        G, h->B, q, which ? 1 : -1, 0, G.nxl);
  } else {
    // column chunks: transposed on the handle's stream into staging buffer
    // i % 2 (once the copy of chunk i - 2 has released it), copied out on the
    // transfer stream
    const int ch = chunk_cols(G.ny);
    const size_t cb = (size_t)ch * G.ny * 5;
    int rc = ensure_tmp(h, cb * sizeof(double));
    if (rc) return rc;
    for (int k = 0, i = 0; k < G.nxl; k += ch, i++) {
      const int nk = std::min(ch, G.nxl - k), b = i & 1;
      double* buf = h->tmp + b * cb;
      if (i >= 2) CK(cudaStreamWaitEvent(h->stream, h->ev_copy[b], 0));
      k_planes_to_aos<<<dim3((nk + TT - 1) / TT, (G.ny + TT - 1) / TT), 256, 0, h->stream>>>(
          G, h->B, buf, which ? 1 : -1, k, nk);
      CK(cudaEventRecord(h->ev_used[b], h->stream));
      CK(cudaStreamWaitEvent(h->xfer, h->ev_used[b], 0));
      CK(cudaMemcpyAsync(q + (size_t)k * G.ny * 5, buf, (size_t)nk * G.ny * 5 * sizeof(double),
                         cudaMemcpyDeviceToHost, h->xfer));
      CK(cudaEventRecord(h->ev_copy[b], h->xfer));
    }
    CK(cudaStreamSynchronize(h->xfer));
  }
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(h->stream));
  return WB_OK;
}

int wb_get_cell(wb_handle* h, int32_t i, int32_t j, double* q5) {
  if (!h || !q5) return WB_E_ARG;
  int c = i - h->G.i_begin + HALO;
  if (c < 0 || c >= h->G.ncol || j < 0 || j >= h->G.ny) return WB_E_ARG;
  CK(cudaSetDevice(h->dev));
  int rc = read_status(h);
  if (rc) return rc;
  int cur = h->h_st->cur;
  size_t o = (size_t)j * h->G.pitch + c;
  for (int m = 0; m < 4; m++)
    CK(cudaMemcpy(q5 + m, h->B.q[cur][m] + o, sizeof(double), cudaMemcpyDeviceToHost));
  double y;
  CK(cudaMemcpy(&y, h->ycent + j, sizeof(double), cudaMemcpyDeviceToHost));
  q5[4] = y;
  return WB_OK;
}

int wb_max_rate(wb_handle* h, double* rmax, wb_error* err) {
  if (!h) return WB_E_ARG;
  if (!h->have_state) return WB_E_STATE;
  CK(cudaSetDevice(h->dev));
  int rc = do_prepare(h, rmax, err);
  if (rc) return rc;
  h->need_prepare = err ? err->code != WB_ERR_NONE : false;
  return WB_OK;
}

int wb_get_columns(wb_handle* h, double* y0s, double* aeqs) {
  if (!h) return WB_E_ARG;
  CK(cudaSetDevice(h->dev));
  int rc = read_status(h);
  if (rc) return rc;
  const int b = h->h_st->cur ^ (h->cols_prev && h->h_st->step > 0 ? 1 : 0);
  const size_t off = (size_t)b * h->G.pitch + HALO;
  if (y0s)
    CK(cudaMemcpy(y0s, h->y0s + off, h->G.nxl * sizeof(double), cudaMemcpyDeviceToHost));
  if (aeqs)
    CK(cudaMemcpy(aeqs, h->aeqs + off, h->G.nxl * sizeof(double), cudaMemcpyDeviceToHost));
  return WB_OK;
}

static int advance_impl(wb_handle* h, double max_dt, double* dt_out, wb_error* err,
                        const Dbg* dbg) {
  if (!h) return WB_E_ARG;
  if (!h->have_state) return WB_E_STATE;
  CK(cudaSetDevice(h->dev));
  if (err) err->code = WB_ERR_NONE;
  bool prepared_now = false;
  if (h->need_prepare) {
    wb_error e{};
    int rc = do_prepare(h, nullptr, &e);
    if (rc) return rc;
    if (e.code != WB_ERR_NONE) {
      if (err) *err = e;
      return WB_OK;
    }
    h->need_prepare = false;
    prepared_now = true;
  }
  int has = !isnan(max_dt);
  k_set_run<<<1, 1, 0, h->stream>>>(h->st, 0, has, has ? max_dt : 0.0, 0.0, 0.0,
                                     h->step + 1, 1);
  if (!h->B.fuse_detect && !prepared_now) launch_detect(h);
  k_reset_counters<<<1, 1, 0, h->stream>>>(h->st);
  if (dbg)
    launch_step<true>(h, *dbg);
  else
    launch_step<false>(h, Dbg{});
  k_prefinalize<<<1, 1, 0, h->stream>>>(h->st);
  k_finalize<<<1, 1, 0, h->stream>>>(h->st, h->G.cfl, h->dtlog, DTLOG_CAP);
  CK(cudaGetLastError());
  int rc = read_status(h);
  if (rc) return rc;
  fill_error(h, err);
  if (h->h_st->stop > 0) h->need_prepare = true;  // a failed step leaves q^n current
  else h->cols_prev = true;
  if (dt_out) *dt_out = h->h_st->dt;
  return WB_OK;
}

int wb_advance(wb_handle* h, double max_dt, double* dt_out, wb_error* err) {
  return advance_impl(h, max_dt, dt_out, err, nullptr);
}

int wb_advance_debug(wb_handle* h, double max_dt, double* dt_out, wb_error* err,
                     const wb_stage_arrays* out) {
  if (!h || !out) return WB_E_ARG;
  CK(cudaSetDevice(h->dev));
  const size_t n = (size_t)h->G.nxl * h->G.ny;
  const size_t b5 = n * 5 * sizeof(double);
  double* base = nullptr;
  uint8_t* qd = nullptr;
  CK(cudaMalloc(&base, 10 * b5));
  CK(cudaMemset(base, 0, 10 * b5));
  CK(cudaMalloc(&qd, n));
  CK(cudaMemset(qd, 0, n));
  Dbg D;
  double** slots[10] = {&D.fW, &D.fE, &D.fS, &D.fN, &D.vol, &D.psi, &D.DW, &D.DE, &D.DS, &D.DN};
  for (int k = 0; k < 10; k++) *slots[k] = base + k * n * 5;
  D.quiet = qd;
  int rc = advance_impl(h, max_dt, dt_out, err, &D);
  if (rc == WB_OK) {
    double* outs[10] = {out->fW, out->fE, out->fS, out->fN, out->vol,
                        out->psi, out->DW, out->DE, out->DS, out->DN};
    for (int k = 0; k < 10; k++)
      if (outs[k]) CK(cudaMemcpy(outs[k], *slots[k], b5, cudaMemcpyDeviceToHost));
    if (out->quiet) CK(cudaMemcpy(out->quiet, qd, n, cudaMemcpyDeviceToHost));
    if (out->rhoE_c || out->rhoE_fy) {
      double *rc_d = nullptr, *rf_d = nullptr;
      CK(cudaMalloc(&rc_d, n * sizeof(double)));
      CK(cudaMalloc(&rf_d, (size_t)h->G.nxl * (h->G.ny + 1) * sizeof(double)));
      k_profiles<<<148 * 4, 256, 0, h->stream>>>(h->G, h->B, h->P, rc_d, rf_d,
                                                  h->cols_prev ? 1 : 0);
      CK(cudaStreamSynchronize(h->stream));
      if (out->rhoE_c) CK(cudaMemcpy(out->rhoE_c, rc_d, n * sizeof(double), cudaMemcpyDeviceToHost));
      if (out->rhoE_fy)
        CK(cudaMemcpy(out->rhoE_fy, rf_d, (size_t)h->G.nxl * (h->G.ny + 1) * sizeof(double),
                      cudaMemcpyDeviceToHost));
      cudaFree(rc_d);
      cudaFree(rf_d);
    }
  }
  cudaFree(base);
  cudaFree(qd);
  return rc;
}

int wb_run(wb_handle* h, double t_end, int64_t max_steps, int32_t chunk, wb_error* err) {
  if (!h) return WB_E_ARG;
  if (!h->have_state) return WB_E_STATE;
  CK(cudaSetDevice(h->dev));
  if (err) err->code = WB_ERR_NONE;
  int mode = isnan(t_end) ? 0 : 1;
  double tiny = mode ? 1.0e-12 * std::max(1.0, fabs(t_end)) : 0.0;
  if (mode && !(h->t < t_end - tiny)) return WB_OK;  // run_until's loop does not execute
  if (mode == 0 && max_steps < 0) {
    g_err = "wb_run needs t_end or max_steps";
    return WB_E_ARG;
  }
  if (mode == 0 && max_steps <= h->step) return WB_OK;  // nothing left to take
  if (h->need_prepare) {
    wb_error e{};
    int rc = do_prepare(h, nullptr, &e);
    if (rc) return rc;
    if (e.code != WB_ERR_NONE) {
      if (err) *err = e;
      return WB_OK;
    }
    h->need_prepare = false;
  }
  k_set_run<<<1, 1, 0, h->stream>>>(h->st, mode, 0, 0.0, mode ? t_end : 0.0, tiny,
                                     max_steps, 1);
  CK(cudaGetLastError());
  if (chunk <= 0) chunk = 16;
  if (!h->graph || h->graph_chunk != chunk) {
    if (h->graph) cudaGraphExecDestroy(h->graph);
    h->graph = nullptr;
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
    for (int k = 0; k < chunk; k++) enqueue_step(h);
    CK(cudaStreamEndCapture(h->stream, &g));
    CK(cudaGraphInstantiate(&h->graph, g, 0));
    cudaGraphDestroy(g);
    h->graph_chunk = chunk;
  }
  for (;;) {
    CK(cudaGraphLaunch(h->graph, h->stream));
    int rc = read_status(h);
    if (rc) return rc;
    if (h->h_st->stop != 0) break;
  }
  fill_error(h, err);
  if (h->h_st->stop > 0) h->need_prepare = true;
  else h->cols_prev = true;
  return WB_OK;
}

int wb_diagnostics(wb_handle* h, double y0_eq, double* out9) {
  if (!h || !out9) return WB_E_ARG;
  if (!h->have_state) return WB_E_STATE;
  CK(cudaSetDevice(h->dev));
  const int nblk = 148 * 2;
  double* d;
  CK(cudaMalloc(&d, (size_t)(nblk + 1) * DIAG_N * sizeof(double)));
  k_diag1<<<nblk, DIAG_T, 0, h->stream>>>(h->G, h->B, h->P, y0_eq, d);
  k_diag2<<<1, 1, 0, h->stream>>>(d, nblk, h->P.area, d + (size_t)nblk * DIAG_N);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out9, d + (size_t)nblk * DIAG_N, DIAG_N * sizeof(double),
                     cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  cudaFree(d);
  return WB_OK;
}

int wb_depth_averaged_velocity(wb_handle* h, double* out_host) {
  if (!h || !out_host) return WB_E_ARG;
  if (!h->have_state) return WB_E_STATE;
  CK(cudaSetDevice(h->dev));
  double* d;
  CK(cudaMalloc(&d, (size_t)h->G.nxl * sizeof(double)));
  k_depth_avg<<<(h->G.nxl + 127) / 128, 128, 0, h->stream>>>(h->G, h->B, h->P.dy, d);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out_host, d, (size_t)h->G.nxl * sizeof(double), cudaMemcpyDeviceToHost,
                     h->stream));
  CK(cudaStreamSynchronize(h->stream));
  cudaFree(d);
  return WB_OK;
}

int wb_get_error(wb_handle* h, wb_error* err) {
  if (!h || !err) return WB_E_ARG;
  CK(cudaSetDevice(h->dev));
  int rc = read_status(h);
  if (rc) return rc;
  fill_error(h, err);
  return WB_OK;
}

int wb_get_status(wb_handle* h, wb_status* s) {
  if (!h || !s) return WB_E_ARG;
  CK(cudaSetDevice(h->dev));
  int rc = read_status(h);
  if (rc) return rc;
  const Status& d = *h->h_st;
  s->t = d.t;
  s->dt = d.dt;
  unsigned long long b = d.rmax_used_bits;
  memcpy(&s->rmax, &b, 8);
  s->step = d.step;
  s->stop = d.stop;
  s->cur = d.cur;
  s->n_second_order = d.n2nd;
  s->x_faces_solved = d.nxs;
  s->y_faces_solved = d.nys;
  s->replays = d.n_replay;
  for (int k = 0; k < 6; k++) s->replays_by_kind[k] = d.n_replay_kind[k];
  return WB_OK;
}

int wb_set_time(wb_handle* h, double t, int64_t step) {
  if (!h) return WB_E_ARG;
  CK(cudaSetDevice(h->dev));
  k_set_time<<<1, 1, 0, h->stream>>>(h->st, t, step);
  CK(cudaStreamSynchronize(h->stream));
  h->t = t;
  h->step = step;
  return WB_OK;
}

int wb_get_dt_log(wb_handle* h, double* out, int64_t n) {
  if (!h || !out || n < 0 || n > DTLOG_CAP) return WB_E_ARG;
  CK(cudaSetDevice(h->dev));
  CK(cudaStreamSynchronize(h->stream));
  CK(cudaMemcpy(out, h->dtlog, n * sizeof(double), cudaMemcpyDeviceToHost));
  return WB_OK;
}

// ---- multi-GPU building blocks ----
int wb_reduce_ptr(wb_handle* h, void** p) {
  if (!h || !p) return WB_E_ARG;
  *p = (void*)&h->st->red[0];
  return WB_OK;
}
int wb_prepare_ptrs(wb_handle* h, void** rmax_bits, void** key_prep) {
  if (!h) return WB_E_ARG;
  if (rmax_bits) *rmax_bits = (void*)&h->st->rmax_bits;
  if (key_prep) *key_prep = (void*)&h->st->key_prep;
  return WB_OK;
}
int wb_prepare_pack(wb_handle* h) {
  if (!h) return WB_E_ARG;
  CK(cudaSetDevice(h->dev));
  k_prepare_pack<<<1, 1, 0, h->stream>>>(h->st);
  CK(cudaGetLastError());
  return WB_OK;
}
int wb_prepare_unpack(wb_handle* h) {
  if (!h) return WB_E_ARG;
  CK(cudaSetDevice(h->dev));
  k_prepare_unpack<<<1, 1, 0, h->stream>>>(h->st);
  CK(cudaGetLastError());
  return WB_OK;
}
int wb_get_stream(wb_handle* h, void** s) {
  if (!h || !s) return WB_E_ARG;
  *s = (void*)h->stream;
  return WB_OK;
}
int wb_prepare_local(wb_handle* h) {
  if (!h || !h->have_state) return WB_E_STATE;
  CK(cudaSetDevice(h->dev));
  k_begin_prepare<<<1, 1, 0, h->stream>>>(h->st);
  launch_detect(h);
  if (h->g1)
    k_prepare<true><<<148 * 4, 256, 0, h->stream>>>(h->G, h->B, h->P);
  else
    k_prepare<false><<<148 * 4, 256, 0, h->stream>>>(h->G, h->B, h->P);
  CK(cudaGetLastError());
  return WB_OK;
}
int wb_check_prepare(wb_handle* h, double* rmax, wb_error* err) {
  if (!h) return WB_E_ARG;
  int rc = read_status(h);
  if (rc) return rc;
  Status& s = *h->h_st;
  double r;
  unsigned long long b = s.rmax_bits;
  memcpy(&r, &b, 8);
  if (rmax) *rmax = r;
  if (err) {
    err->code = WB_ERR_NONE;
    err->i = err->j = -1;
    err->step = s.step;
    err->rmax = r;
    if (s.key_prep != KEY_NONE) {
      err->code = WB_ERR_CELL_STATE;
      err->i = (int32_t)(s.key_prep / h->G.ny);
      err->j = (int32_t)(s.key_prep % h->G.ny);
    } else if (!(isfinite(r) && r > 0.0)) {
      err->code = WB_ERR_WAVE_SPEED;
    }
  }
  h->need_prepare = err && err->code != WB_ERR_NONE;
  return WB_OK;
}
int wb_step_local(wb_handle* h, double max_dt, double t_end, int32_t mode) {
  if (!h || !h->have_state) return WB_E_STATE;
  CK(cudaSetDevice(h->dev));
  int has = !isnan(max_dt);
  double tiny = mode ? 1.0e-12 * std::max(1.0, fabs(t_end)) : 0.0;
  k_set_run<<<1, 1, 0, h->stream>>>(h->st, mode, has, has ? max_dt : 0.0, t_end, tiny, -1, 0);
  if (!h->B.fuse_detect) launch_detect(h);
  k_reset_counters<<<1, 1, 0, h->stream>>>(h->st);
  launch_step<false>(h, Dbg{});
  k_prefinalize<<<1, 1, 0, h->stream>>>(h->st);
  CK(cudaGetLastError());
  return WB_OK;
}
int wb_finalize(wb_handle* h) {
  if (!h) return WB_E_ARG;
  CK(cudaSetDevice(h->dev));
  k_finalize<<<1, 1, 0, h->stream>>>(h->st, h->G.cfl, h->dtlog, DTLOG_CAP);
  CK(cudaGetLastError());
  return WB_OK;
}
int wb_halo_count(wb_handle* h, int64_t* n) {
  if (!h || !n) return WB_E_ARG;
  *n = 2LL * 4 * HALO * h->G.ny + 4 * HALO;  // state columns + their (y0, aeq)
  return WB_OK;
}
int wb_pack_halo(wb_handle* h, void* send) {
  if (!h || !send) return WB_E_ARG;
  CK(cudaSetDevice(h->dev));
  k_pack_halo<<<148, 256, 0, h->stream>>>(h->G, h->B, (double*)send, 0);
  CK(cudaGetLastError());
  return WB_OK;
}
int wb_unpack_halo(wb_handle* h, const void* recv, int32_t hl, int32_t hr) {
  if (!h || !recv) return WB_E_ARG;
  CK(cudaSetDevice(h->dev));
  k_unpack_halo<<<148, 256, 0, h->stream>>>(h->G, h->B, (const double*)recv, hl, hr, 0);
  CK(cudaGetLastError());
  return WB_OK;
}

// ---- overlapped multi-GPU step (SURVEY.md 8(e) "Overlap") ----
int wb_set_edge_stream(wb_handle* h, void* s) {
  if (!h) return WB_E_ARG;
  CK(cudaSetDevice(h->dev));
  CK(cudaStreamSynchronize(h->stream));
  if (h->edge) CK(cudaStreamSynchronize(h->edge));
  h->edge = (cudaStream_t)s;
  if (!h->ev_fork) CK(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
  if (!h->ev_join) CK(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
  return WB_OK;
}
// Stream s: set_run, [detect], reset_counters, then the interior strips.
// Edge stream: after the reset, the two slab-edge strips, then the pack of
// their new halo-source columns (from the step's output buffer) into `send`.
// The caller exchanges `send`/`recv` on the edge stream, calls
// wb_unpack_halo_next there, then wb_step_end.
static int step_begin(wb_handle* h, double max_dt, double t_end, int32_t mode, void* send);
int wb_step_begin(wb_handle* h, double max_dt, double t_end, int32_t mode, void* send) {
  if (!h || !send) return WB_E_ARG;
  return step_begin(h, max_dt, t_end, mode, send);
}
int wb_step_begin_peer(wb_handle* h, double max_dt, double t_end, int32_t mode) {
  if (!h) return WB_E_ARG;
  return step_begin(h, max_dt, t_end, mode, nullptr);
}
// send == nullptr: store the halo into the peers (k_push_halo), else pack it
static int step_begin(wb_handle* h, double max_dt, double t_end, int32_t mode, void* send) {
  if (!h->have_state) return WB_E_STATE;
  if (!h->edge) return WB_E_STATE;
  CK(cudaSetDevice(h->dev));
  int has = !isnan(max_dt);
  double tiny = mode ? 1.0e-12 * std::max(1.0, fabs(t_end)) : 0.0;
  k_set_run<<<1, 1, 0, h->stream>>>(h->st, mode, has, has ? max_dt : 0.0, t_end, tiny, -1, 0);
  if (!h->B.fuse_detect) launch_detect(h);
  k_reset_counters<<<1, 1, 0, h->stream>>>(h->st);
  CK(cudaEventRecord(h->ev_fork, h->stream));
  CK(cudaStreamWaitEvent(h->edge, h->ev_fork, 0));
  // halo over peer memory with the default variants: the edge launch stores
  // its halo-source columns into the peers as it produces them
  const bool fused = !send && edge_push_built(h);
  launch_step<false>(h, Dbg{}, h->edge, PART_EDGE, fused);
  {
    // a split edge launch leaves the detection of its strips' owned columns
    // to k_detect_cols (see launch_step); the pack needs it for the halo
    const int nt = step_nt(h, false), w = nt - 2 * HALO;
    const dim3 g = step_grid(h, nt);
    const bool split = g.x >= 3 && h->G.nxl - ((int)g.x - 1) * w >= HALO;
    if (split && h->B.fuse_detect) {
      const int c0 = HALO, c1 = std::min(HALO + w, h->G.nxl + HALO);
      const int c2 = ((int)g.x - 1) * w + HALO, c3 = std::min(c2 + w, h->G.nxl + HALO);
      const int ncols = (c1 - c0) + (c3 - c2);
      // (fused: it also stores the detection of the halo-source columns
      // into the peers)
      const PeerBufs none{};
      k_detect_cols<<<(ncols + 7) / 8, 256, 0, h->edge>>>(
          h->G, h->B, h->P.dy, c0, c1, c2, c3, fused ? h->peer[0] : none,
          fused ? h->peer[1] : none);
    }
  }
  if (send)
    k_pack_halo<<<148, 256, 0, h->edge>>>(h->G, h->B, (double*)send, 1);
  else if (!fused && (h->peer[0].q[0][0] || h->peer[1].q[0][0]))
    k_push_halo<<<148, 256, 0, h->edge>>>(h->G, h->B, h->peer[0], h->peer[1], 1);
  launch_step<false>(h, Dbg{}, h->stream, PART_INTERIOR);
  CK(cudaGetLastError());
  return WB_OK;
}
int wb_unpack_halo_next(wb_handle* h, const void* recv, int32_t hl, int32_t hr) {
  if (!h || !recv || !h->edge) return WB_E_ARG;
  CK(cudaSetDevice(h->dev));
  k_unpack_halo<<<148, 256, 0, h->edge>>>(h->G, h->B, (const double*)recv, hl, hr, 1);
  CK(cudaGetLastError());
  return WB_OK;
}
// Join the edge stream into s and prepare the reduction vector (then the
// caller all-reduces it on s and calls wb_finalize).
int wb_step_end(wb_handle* h) {
  if (!h || !h->edge) return WB_E_ARG;
  CK(cudaSetDevice(h->dev));
  CK(cudaEventRecord(h->ev_join, h->edge));
  CK(cudaStreamWaitEvent(h->stream, h->ev_join, 0));
  k_prefinalize<<<1, 1, 0, h->stream>>>(h->st);
  CK(cudaGetLastError());
  return WB_OK;
}
// ---- halo over peer memory ----
namespace {
struct PeerIpc {  // WB_PEER_IPC_BYTES bytes
  cudaIpcMemHandle_t planes, y0s, aeqs;  // 3 x 64 bytes
  long long plane, shift;                // doubles per plane, PLANE_SHIFT
  int pitch, nxl, ny, magic;
  char pad[WB_PEER_IPC_BYTES - 3 * sizeof(cudaIpcMemHandle_t) - 2 * sizeof(long long) -
           4 * sizeof(int)];
};
static_assert(sizeof(PeerIpc) == WB_PEER_IPC_BYTES, "peer IPC blob size");
constexpr int PEER_MAGIC = 0x57425032;  // "WBP2"
void fill_peer(wb_peer* out, double* planes, double* y0s, double* aeqs, long long plane,
               long long shift, int pitch, int nxl, int ny) {
  memset(out, 0, sizeof(*out));
  for (int b = 0; b < 2; b++) {
    for (int m = 0; m < 4; m++) out->q[b][m] = planes + shift + (b * 4 + m) * plane;
    out->y0s[b] = y0s + b * pitch;
    out->aeqs[b] = aeqs + b * pitch;
  }
  out->pitch = pitch;
  out->nxl = nxl;
  out->ny = ny;
}
}  // namespace

int wb_peer_desc(wb_handle* h, wb_peer* out) {
  if (!h || !out) return WB_E_ARG;
  fill_peer(out, h->planes, h->y0s, h->aeqs, (long long)h->G.pitch * h->G.ny, PLANE_SHIFT,
            h->G.pitch, h->G.nxl, h->G.ny);
  return WB_OK;
}
int wb_peer_ipc_export(wb_handle* h, void* blob) {
  if (!h || !blob) return WB_E_ARG;
  CK(cudaSetDevice(h->dev));
  PeerIpc p;
  memset(&p, 0, sizeof(p));
  CK(cudaIpcGetMemHandle(&p.planes, h->planes));
  CK(cudaIpcGetMemHandle(&p.y0s, h->y0s));
  CK(cudaIpcGetMemHandle(&p.aeqs, h->aeqs));
  p.plane = (long long)h->G.pitch * h->G.ny;
  p.shift = PLANE_SHIFT;
  p.pitch = h->G.pitch;
  p.nxl = h->G.nxl;
  p.ny = h->G.ny;
  p.magic = PEER_MAGIC;
  memcpy(blob, &p, sizeof(p));
  return WB_OK;
}
int wb_peer_ipc_open(wb_handle* h, const void* blob, wb_peer* out) {
  if (!h || !blob || !out) return WB_E_ARG;
  PeerIpc p;
  memcpy(&p, blob, sizeof(p));
  if (p.magic != PEER_MAGIC || h->n_ipc_open + 3 > 6) {
    g_err = "wb_peer_ipc_open: not a wb_peer_ipc_export blob, or more than two peers";
    return WB_E_ARG;
  }
  CK(cudaSetDevice(h->dev));
  void *pl = nullptr, *y0 = nullptr, *ae = nullptr;
  CK(cudaIpcOpenMemHandle(&pl, p.planes, cudaIpcMemLazyEnablePeerAccess));
  h->ipc_open[h->n_ipc_open++] = pl;
  CK(cudaIpcOpenMemHandle(&y0, p.y0s, cudaIpcMemLazyEnablePeerAccess));
  h->ipc_open[h->n_ipc_open++] = y0;
  CK(cudaIpcOpenMemHandle(&ae, p.aeqs, cudaIpcMemLazyEnablePeerAccess));
  h->ipc_open[h->n_ipc_open++] = ae;
  fill_peer(out, (double*)pl, (double*)y0, (double*)ae, p.plane, p.shift, p.pitch, p.nxl, p.ny);
  return WB_OK;
}
// plain step: after wb_step_local, the halo of the step's output buffer into
// the peers (on the handle's stream; then all-reduce -> wb_finalize)
int wb_push_halo_next(wb_handle* h) {
  if (!h) return WB_E_ARG;
  CK(cudaSetDevice(h->dev));
  if (h->peer[0].q[0][0] || h->peer[1].q[0][0])
    k_push_halo<<<148, 256, 0, h->stream>>>(h->G, h->B, h->peer[0], h->peer[1], 1);
  CK(cudaGetLastError());
  return WB_OK;
}
int wb_set_peers(wb_handle* h, const wb_peer* left, const wb_peer* right) {
  if (!h) return WB_E_ARG;
  CK(cudaSetDevice(h->dev));
  CK(cudaStreamSynchronize(h->stream));
  if (h->edge) CK(cudaStreamSynchronize(h->edge));
  const wb_peer* src[2] = {left, right};
  for (int s = 0; s < 2; s++) {
    PeerBufs& d = h->peer[s];
    memset(&d, 0, sizeof(d));
    if (!src[s]) continue;
    if (src[s]->ny != h->G.ny) {
      g_err = "wb_set_peers: the neighbour slab has another number of rows";
      return WB_E_ARG;
    }
    // a peer on another device: enable access to it (a no-op for IPC
    // allocations, opened with cudaIpcMemLazyEnablePeerAccess)
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, src[s]->q[0][0]) == cudaSuccess && a.device != h->dev &&
        a.device >= 0) {
      cudaError_t e = cudaDeviceEnablePeerAccess(a.device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
        g_err = "wb_set_peers: no peer access to the neighbour's device";
        return WB_E_CUDA;
      }
      cudaGetLastError();
    }
    for (int b = 0; b < 2; b++) {
      for (int m = 0; m < 4; m++) d.q[b][m] = (double*)src[s]->q[b][m];
      d.y0s[b] = (double*)src[s]->y0s[b];
      d.aeqs[b] = (double*)src[s]->aeqs[b];
    }
    d.pitch = src[s]->pitch;
    d.nxl = src[s]->nxl;
  }
  return WB_OK;
}

// Kernel-level timing with CUDA events on the handle's stream: n steps
// launched individually, average duration of the detect and step kernels.
int wb_profile_steps(wb_handle* h, int32_t n, double* ms_detect, double* ms_step,
                     double* ms_total) {
  if (!h || n <= 0 || !h->have_state) return WB_E_ARG;
  CK(cudaSetDevice(h->dev));
  if (h->need_prepare) {
    wb_error e{};
    int rc = do_prepare(h, nullptr, &e);
    if (rc) return rc;
    if (e.code) return WB_E_STATE;
    h->need_prepare = false;
  }
  cudaEvent_t ev[4];
  for (int k = 0; k < 4; k++) CK(cudaEventCreate(&ev[k]));
  k_set_run<<<1, 1, 0, h->stream>>>(h->st, 0, 0, 0.0, 0.0, 0.0, -1, 1);
  double sd = 0, ss = 0;
  float a, b;
  CK(cudaEventRecord(ev[3], h->stream));
  cudaEvent_t t0;
  CK(cudaEventCreate(&t0));
  CK(cudaEventRecord(t0, h->stream));
  for (int k = 0; k < n; k++) {
    CK(cudaEventRecord(ev[0], h->stream));
    if (!h->B.fuse_detect) launch_detect(h);
    CK(cudaEventRecord(ev[1], h->stream));
    k_reset_counters<<<1, 1, 0, h->stream>>>(h->st);
    CK(cudaEventRecord(ev[2], h->stream));
    launch_step<false>(h, Dbg{});
    CK(cudaEventRecord(ev[3], h->stream));
    k_prefinalize<<<1, 1, 0, h->stream>>>(h->st);
    k_finalize<<<1, 1, 0, h->stream>>>(h->st, h->G.cfl, h->dtlog, DTLOG_CAP);
    CK(cudaEventSynchronize(ev[3]));
    CK(cudaEventElapsedTime(&a, ev[0], ev[1]));
    CK(cudaEventElapsedTime(&b, ev[2], ev[3]));
    sd += a;
    ss += b;
  }
  cudaEvent_t t1;
  CK(cudaEventCreate(&t1));
  CK(cudaEventRecord(t1, h->stream));
  CK(cudaEventSynchronize(t1));
  float tot;
  CK(cudaEventElapsedTime(&tot, t0, t1));
  for (int k = 0; k < 4; k++) cudaEventDestroy(ev[k]);
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  if (ms_detect) *ms_detect = sd / n;
  if (ms_step) *ms_step = ss / n;
  if (ms_total) *ms_total = tot / n;
  return read_status(h);
}

int wb_fp64_peak(int32_t device, double* tflops) {
  CK(cudaSetDevice(device));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  double* out;
  CK(cudaMalloc(&out, 8));
  const int iters = 4096, threads = 256, blocks = sms * 8;
  k_dfma_peak<<<blocks, threads>>>(out, 64, 1.0000001, 1e-7);  // warm-up
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float best = 1e30f;
  for (int r = 0; r < 5; r++) {
    CK(cudaEventRecord(e0));
    k_dfma_peak<<<blocks, threads>>>(out, iters, 1.0000001, 1e-7);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    best = std::min(best, ms);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  double flops = 2.0 * 64.0 * iters * (double)threads * blocks;
  if (tflops) *tflops = flops / (best * 1e-3) / 1e12;
  return WB_OK;
}

int wb_selftest_div(int32_t device, int64_t n, uint64_t seed, uint64_t* mismatches) {
  CK(cudaSetDevice(device));
  unsigned long long* d;
  CK(cudaMalloc(&d, 8));
  CK(cudaMemset(d, 0, 8));
  k_selftest_div<<<148 * 8, 256>>>(n, seed, d);
  CK(cudaGetLastError());
  unsigned long long hv = 0;
  CK(cudaMemcpy(&hv, d, 8, cudaMemcpyDeviceToHost));
  cudaFree(d);
  if (mismatches) *mismatches = hv;
  return WB_OK;
}

int wb_eval_exp(int32_t device, const double* x, double* y, int64_t n) {
  if (!x || !y || n <= 0) return WB_E_ARG;
  CK(cudaSetDevice(device));
  static bool tab_ok = false;
  if (!tab_ok) {
    CK(cudaMemcpyToSymbol(g_exp_tab, WB_EXP_TAB, sizeof(WB_EXP_TAB)));
    tab_ok = true;
  }
  double *dx, *dy;
  CK(cudaMalloc(&dx, n * sizeof(double)));
  CK(cudaMalloc(&dy, n * sizeof(double)));
  CK(cudaMemcpy(dx, x, n * sizeof(double), cudaMemcpyHostToDevice));
  k_eval_exp<<<148 * 4, 256>>>(dx, dy, n);
  CK(cudaGetLastError());
  CK(cudaMemcpy(y, dy, n * sizeof(double), cudaMemcpyDeviceToHost));
  cudaFree(dx);
  cudaFree(dy);
  return WB_OK;
}

int wb_eval_faces(wb_handle* h, int32_t kind, int64_t n, const double* qm, const double* qp,
                  const double* aux, double* dm, double* dp) {
  if (!h || n <= 0 || !qm || !qp || !dm || !dp || (kind != 0 && kind != 1) ||
      (kind == 1 && !aux))
    return WB_E_ARG;
  CK(cudaSetDevice(h->dev));
  CK(cudaStreamSynchronize(h->stream));
  double* d;
  const size_t na = kind == 1 ? 3 * (size_t)n : 1;
  CK(cudaMalloc(&d, (16 * (size_t)n + na) * sizeof(double)));
  double *dqm = d, *dqp = d + 4 * n, *ddm = d + 8 * n, *ddp = d + 12 * n, *dax = d + 16 * n;
  CK(cudaMemcpy(dqm, qm, 4 * n * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dqp, qp, 4 * n * sizeof(double), cudaMemcpyHostToDevice));
  if (kind == 1) CK(cudaMemcpy(dax, aux, 3 * n * sizeof(double), cudaMemcpyHostToDevice));
  if (h->g1)
    k_eval_faces<true><<<148 * 4, 128, 0, h->stream>>>(h->P, kind, n, dqm, dqp, dax, ddm, ddp);
  else
    k_eval_faces<false><<<148 * 4, 128, 0, h->stream>>>(h->P, kind, n, dqm, dqp, dax, ddm, ddp);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(h->stream));
  CK(cudaMemcpy(dm, ddm, 4 * n * sizeof(double), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(dp, ddp, 4 * n * sizeof(double), cudaMemcpyDeviceToHost));
  cudaFree(d);
  return WB_OK;
}

int wb_sync(wb_handle* h) {
  if (!h) return WB_E_ARG;
  int rc = read_status(h);
  return rc;
}

}  // extern "C"
