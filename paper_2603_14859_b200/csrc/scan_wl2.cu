// scan_wl2.cu -- instantiations of the FP32 pass (scan_kernels.cuh) for the weighted-L2 distance.
#include "scan_kernels.cuh"

namespace vpet {
cudaError_t launch_scan_wl2(const ScanParams& p, uint32_t LP, int count_work, int tree, cudaStream_t st) {
  return scan::launch_dist<ABC_DIST_WL2>(p, LP, count_work, tree, st);
}
}  // namespace vpet
