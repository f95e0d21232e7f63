// Occupancy probe (profiles/r01_summary.md): the y-face solver + cell update of
// k_step, stand-alone over synthetic face records, at three register budgets.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 \
//        -I paper_1806_04960_b200/csrc tools/yface_probe.cu -o /tmp/yface_probe
#include "wb_step.cu"
namespace wb {
// K_B-like probe: per column, rows ascending: y-face between R-1 and R, update R-1
template <bool G1, int MB>
__global__ void __launch_bounds__(64, MB) k_probe(const double* __restrict__ rec, double* out, int ny,
                                                  int pitch, Phys P, double rdx, double rdy,
                                                  double rvol) {
  int c = blockIdx.x * 64 + threadIdx.x;
  double fNp[4] = {0, 0, 0, 0}, qp[4] = {0, 0, 0, 0}, Xp[4] = {0, 0, 0, 0}, DSp[4] = {0, 0, 0, 0};
  double gys[3] = {0, 0, 0}, v2 = 0, v3 = 0, rmax = 0;
  for (int R = 0; R < ny; R++) {
    const double* r = rec + (size_t)R * pitch * 18 + c;
    double fS[4], fN[4], q[4], X[4];
    for (int m = 0; m < 4; m++) {
      fS[m] = r[m * pitch]; fN[m] = r[(4 + m) * pitch]; q[m] = r[(8 + m) * pitch];
      X[m] = r[(12 + m) * pitch];
    }
    double vv2 = r[16 * pitch], vv3 = r[17 * pitch];
    double dm[4], dp[4];
    FastDiv fd;
    osher_romberg_y<G1>(fNp, fS, 1000.0, 0.0, 1.0, P, fd, dm, dp);
    double qn[4];
    double rr = update_cell<G1>(qp, Xp, DSp, dm, fNp, gys, v2, v3, rdx, rdy, rvol, P, fd, qn);
    if (!fd.ok) rr = -2;
    for (int m = 0; m < 4; m++) out[(size_t)R * pitch * 4 + m * pitch + c] = qn[m];
    rmax = fmax(rmax, rr);
    for (int m = 0; m < 4; m++) { fNp[m] = fN[m]; qp[m] = q[m]; Xp[m] = X[m]; DSp[m] = dp[m]; }
    flux_y(fS, fd, gys);
    v2 = vv2; v3 = vv3;
  }
  out[c] = rmax;
}
}


#include <cstdio>
#include <vector>
#include <cmath>
using namespace wb;
int main() {
  const int nx = 75776, ny = 256, pitch = nx;
  std::vector<double> h((size_t)18 * nx * ny);
  for (int R = 0; R < ny; R++)
    for (int c = 0; c < nx; c++) {
      double* r = h.data() + (size_t)R * pitch * 18 + c;
      double a = 0.999 - 1e-7 * c, y = 1.0 - R * 1e-4;
      double rho = 1000.0 * exp(9.81 / 2.62e5 * 1000.0 * y * 1e-3);
      double vals[18] = {a * rho, 0.1 * sin(c * 0.01), 0.2 * cos(R * 0.01), a,
                         a * rho * (1 + 1e-6), 0.1 * sin(c * 0.01 + 1e-3), 0.2 * cos(R * 0.01 + 1e-3), a,
                         a * rho, 0.1, 0.2, a, 1e-3, 2e-3, 3e-3, 0.0, 1e-4, 1e-5};
      for (int k = 0; k < 18; k++) r[(size_t)k * pitch] = vals[k];
    }
  double *d_rec, *d_out;
  cudaMalloc(&d_rec, h.size() * 8);
  cudaMalloc(&d_out, (size_t)4 * nx * ny * 8);
  cudaMemcpy(d_rec, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  Phys P{};
  P.rho0 = 1000.0; P.k0 = 2.62e5; P.gamma = 1.0; P.g = 9.81; P.cref = sqrt(2.62e5 / 1000.0);
  P.c2c = P.cref * P.cref; P.c2ref = 262.0; P.halfc = 0.5 / P.cref; P.dx = 1e-3; P.dy = 1e-3;
  P.yrho0 = 1e-3; P.ycref = 1.0 / P.cref; P.yc2c = 1.0 / P.c2c;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](auto kern, const char* name) {
    for (int it = 0; it < 2; it++) kern<<<nx / 64, 64>>>(d_rec, d_out, ny, pitch, P, 1e-3, 1e-3, 1e-6);
    cudaEventRecord(e0);
    for (int it = 0; it < 5; it++) kern<<<nx / 64, 64>>>(d_rec, d_out, ny, pitch, P, 1e-3, 1e-3, 1e-6);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%s: %.3f ms/launch (%s)\n", name, ms / 5, cudaGetErrorString(cudaGetLastError()));
  };
  run(k_probe<true, 1>, "minb1 (244 regs, 8 warps)");
  run(k_probe<true, 6>, "minb6 (168 regs, 12 warps)");
  run(k_probe<true, 8>, "minb8 (128 regs, 16 warps)");
  return 0;
}
