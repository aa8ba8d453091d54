// C-only bring-up harness for BSSN variant 4 (no Python): create a small BSSN grid over a
// cudaMalloc workspace, RHS with variant 3 and 4, compare.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../include/chemora.h"
int main() {
  chemora_grid_desc d = {};
  d.system = CHEMORA_SYS_BSSN; d.ghost = 3; d.n_gf = 25; d.device = 0;
  d.extent[0] = 16; d.extent[1] = 8; d.extent[2] = 12;
  for (int a = 0; a < 3; ++a) d.spacing[a] = 1.0 / d.extent[a];
  d.rank = 0; d.nranks = 1;
  size_t bytes = 0;
  if (chemora_grid_required_bytes(&d, &bytes)) { printf("req: %s\n", chemora_last_error()); return 2; }
  void* ws; cudaMalloc(&ws, bytes);
  chemora_grid_t g;
  if (chemora_grid_create(&d, ws, bytes, &g)) { printf("create: %s\n", chemora_last_error()); return 2; }
  const size_t ni = 16 * 8 * 12 * 25;
  double *k3, *k4; cudaMalloc(&k3, ni * 8); cudaMalloc(&k4, ni * 8);
  double eps = 1e-2;
  if (chemora_set_initial(g, CHEMORA_INIT_MINK_PERT, nullptr, &eps, 1410, nullptr)) { printf("init: %s\n", chemora_last_error()); return 2; }
  fprintf(stderr, "init ok\n");
  chemora_set_kernel_variant(g, 3);
  int rc = chemora_rhs(g, k3, nullptr);
  fprintf(stderr, "rhs3 rc %d %s\n", rc, rc ? chemora_last_error() : "");
  chemora_set_kernel_variant(g, 4);
  rc = chemora_rhs(g, k4, nullptr);
  fprintf(stderr, "rhs4 rc %d %s\n", rc, rc ? chemora_last_error() : "");
  cudaError_t e = cudaDeviceSynchronize();
  fprintf(stderr, "sync %s\n", cudaGetErrorString(e));
  std::vector<double> a(ni), b(ni);
  cudaMemcpy(a.data(), k3, ni * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(b.data(), k4, ni * 8, cudaMemcpyDeviceToHost);
  double md = 0, ma = 0;
  for (size_t i = 0; i < ni; ++i) { md = fmax(md, fabs(a[i] - b[i])); ma = fmax(ma, fabs(a[i])); }
  printf("max |k3| %g  max |k3-k4| %g\n", ma, md);
  return 0;
}
