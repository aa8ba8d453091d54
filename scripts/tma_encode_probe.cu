// Which TMA box shapes does cuTensorMapEncodeTiled accept for a 4-D fp64 set map?
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
int main() {
  double* d;
  const size_t px = 48, py = 14, pz = 18, ng = 25;
  size_t gfs = (px * py * pz + 31) / 32 * 32;
  cudaMalloc(&d, gfs * ng * 8);
  const unsigned boxes[][4] = {{22, 14, 1, 1}, {22, 14, 1, 5}, {22, 14, 1, 8}, {22, 14, 1, 16}, {22, 14, 1, 25},
                               {24, 14, 1, 25}, {16, 8, 1, 25}, {22, 14, 2, 12}, {22, 12, 1, 25}, {22, 13, 1, 25}};
  for (auto& b : boxes) {
    CUtensorMap m;
    const cuuint64_t dims[4] = {px, py, pz, ng};
    const cuuint64_t strides[3] = {px * 8, px * py * 8, gfs * 8};
    const cuuint32_t box[4] = {b[0], b[1], b[2], b[3]};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    fprintf(stderr, "box %u %u %u %u ... ", b[0], b[1], b[2], b[3]);
    CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, d, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    fprintf(stderr, "%d\n", (int)r);
  }
  return 0;
}
