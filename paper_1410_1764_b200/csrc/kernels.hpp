// kernels.hpp -- host-side launch interface between the runtime (capi.cpp) and the
// CUDA kernels.  Internal; not part of the C ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "grid.hpp"

namespace chemora {

// Set pointers (interior-origin pointer of GF 0 of a set; GF v = base + v * L.gfs).
struct SetPtrs {
  double* y;
  double* q;
  double* b;
  double* c;
};

// z-face image destinations for the output of one stage: where the images of the first
// g planes (lo) and of the last g planes (hi) go.  For a whole-z grid both are the output
// set itself; for a slab they are the neighbours' copies of the same set.
struct FaceDst {
  double* lo;
  double* hi;
};

struct StageLaunch {
  Layout L;
  SetPtrs s;             // this slab's sets
  FaceDst img[4];        // per stage s=1..4 (index s-1): neighbour/own base of that stage's output set
  double h[3];
  double dt;
  int fd_order;          // wave: 2/4/6/8
  const double* params;  // device copy of BSSN gauge params (10)
  double hparams[10];    // host copy (folded into kernel arguments)
  unsigned long long* nan_flag;
  // dynamic work scheduler of the persistent wave pair kernels: [0] next item, [1] CTAs done;
  // zero between launches (the last CTA of a launch resets both)
  unsigned long long* sched;
  uint64_t step;         // global step index (for the non-finite report)
  int k_begin, k_end;    // local z-plane range [k_begin, k_end)
  int variant;           // kernel variant (0 = default fast, 1 = simple reference kernel)
  int band;              // wave simple-kernel CTA band order (-1 auto, 0 plain 3-D order)
  double* mon_partials;  // NEXT-3 fused energy monitor: per-CTA partials of stage 4 (or null)
  double* dtab;          // BSSN variant 3: HBM derivative table [136][interior point]
};

// Wave (Eq. 1) -------------------------------------------------------------------------
cudaError_t wave_stage(const StageLaunch& a, int stage, cudaStream_t st);
cudaError_t wave_rhs(const StageLaunch& a, double* dst, cudaStream_t st);
// variant 8 (wave_fused3.cu): temporally blocked stage pairs, pair 0 = stages 1+2, pair 1 =
// stages 3+4 (new state into the scratch set s.b), own-column z stencils from register
// queues; fd_order 4, storage ghost >= 4
cudaError_t wave_fused3_pair(const StageLaunch& a, int pair, cudaStream_t st);
// persistent TMA z-march (wave_tma.cu), fd_order 2/4/6/8, stages 1..4
cudaError_t wave_tma_stage(const StageLaunch& a, int stage, cudaStream_t st);

// BSSN (App. A) ------------------------------------------------------------------------
cudaError_t bssn_stage(const StageLaunch& a, int stage, cudaStream_t st);
cudaError_t bssn_rhs(const StageLaunch& a, double* dst, cudaStream_t st);
// variant 4 (bssn_fused.cu): one fused kernel per stage, derivatives on chip (SMEM plane tiles
// + TMEM z-windows); stage 0 = RHS only into dst
cudaError_t bssn_fused_stage(const StageLaunch& a, int stage, double* dst, cudaStream_t st);
// CTAs of a bssn_fused launch over nk planes (stage 1 with a.mon_partials set leaves 14
// partials [sum c_q^2, max|c_q|] per CTA: the fused constraint monitor)
int bssn_fused_grid(const Layout& L, int nk);
// fixed-order combination of nblocks x 14 constraint partials into out14 (device)
cudaError_t bssn_constraints_reduce(const double* part, int nblocks, double* out14, cudaStream_t st);
// BSSN constraints H, M^i, G^i of a.s.y (R16): optional interior fields
// [7][z][y][x] (nullable) and, on the device, out_dev[2q] = sum c_q^2, out_dev[2q+1] =
// max |c_q| (scratch: kNormBlocks x 14 doubles).
cudaError_t bssn_constraints(const StageLaunch& a, double* fields, double* scratch, double* out_dev,
                             cudaStream_t st);

// Ghost fill of one set (all GFs): x and y locally, then z images stored to face bases.
cudaError_t ghost_fill(const Layout& L, double* set, FaceDst z, cudaStream_t st);

// z ghost planes only: this slab's first/last g planes (x/y ghosts included) into the lo/hi
// faces (the neighbours' copies of the same set, or our own for a whole-z grid).
cudaError_t push_z_planes(const Layout& L, const double* set, FaceDst z, cudaStream_t st);

// Device initial data into the interior of set y (global coordinates).
struct InitArgs {
  int kind;
  int system;
  uint64_t seed;
  int64_t gext[3];   // global interior extents
  int64_t z0;        // global z of local plane 0
  double origin[3], h[3];
  double kp[4];      // kind params
};
cudaError_t init_interior(const Layout& L, double* set, const InitArgs& a, cudaStream_t st);

// Fused energy monitor: sum n partials in fixed order, write vol * sum to *out.
cudaError_t monitor_reduce(const double* partials, int64_t n, double vol, double* out, cudaStream_t st);

// Norm partials of set y: out_dev[len] (deterministic), len = 3 n_gf (+1 wave).
cudaError_t norms_partial(const Layout& L, const double* set, int system, double* scratch,
                          double* out_dev, cudaStream_t st);

}  // namespace chemora
