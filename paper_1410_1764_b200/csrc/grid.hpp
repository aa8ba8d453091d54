// grid.hpp -- internal (not installed) description of the device data layout.
//
// HBM layout (DESIGN.md §"Data layout in HBM"): one caller-owned workspace holding
//   4 state sets (Y, Q, B, C) x n_gf grid-function arrays, then reduction scratch, flags.
// Each GF array is a padded box [Pz][Py][Px] of doubles, x fastest:
//   Pz = nz + 2g, Py = ny + 2g, Px = round_up(XOFF + nx + g, 16), XOFF = 16,
// so that interior x = 0 of every row starts on a 128-byte boundary (full coalesced
// sectors for the interior; the 3 left ghosts sit at x = -3..-1 in the lead pad).
// Arrays start on 256-byte boundaries.  All pointers handed to kernels point at the
// interior origin (i, j, k) = (0, 0, 0) so that index(i, j, k) = k*plane + j*px + i
// also addresses ghosts with negative or >= n coordinates.
#pragma once
#include <cstdint>

namespace chemora {

constexpr int kXOff = 16;          // lead pad of every x row (doubles)
constexpr int kNumSets = 4;        // y, Q, B, C  (DESIGN.md §RK4 one-pass scheme)
enum SetId { SET_Y = 0, SET_Q = 1, SET_B = 2, SET_C = 3 };
constexpr int kNormBlocks = 592;   // 4 x 148 SMs; fixed => deterministic reduction order
constexpr int kNormThreads = 256;

struct Layout {
  int64_t nx, ny, nz;   // local interior extents
  int g;                // ghost width
  int n_gf;
  int64_t px, py, pz;   // padded pitches
  int64_t plane;        // px * py
  int64_t gfs;          // elements per GF array (256-byte multiple)
  int64_t c0;           // element offset of interior (0,0,0) inside a GF array
  __host__ __device__ int64_t idx(int64_t i, int64_t j, int64_t k) const {
    return k * plane + j * px + i;
  }
};

inline Layout make_layout(int64_t nx, int64_t ny, int64_t nz, int g, int n_gf) {
  Layout L;
  L.nx = nx; L.ny = ny; L.nz = nz; L.g = g; L.n_gf = n_gf;
  L.px = ((kXOff + nx + g) + 15) / 16 * 16;
  L.py = ny + 2 * g;
  L.pz = nz + 2 * g;
  L.plane = L.px * L.py;
  L.gfs = (L.plane * L.pz + 31) / 32 * 32;
  L.c0 = (int64_t(g) * L.py + g) * L.px + kXOff;
  return L;
}

}  // namespace chemora
