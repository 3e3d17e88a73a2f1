// scan_l1.cu -- instantiations of the FP32 pass (scan_kernels.cuh) for the L1 distance.
#include "scan_kernels.cuh"

namespace vpet {
cudaError_t launch_scan_l1(const ScanParams& p, uint32_t LP, int count_work, int tree, cudaStream_t st) {
  return scan::launch_dist<ABC_DIST_L1>(p, LP, count_work, tree, st);
}
}  // namespace vpet
