// patlak.cu -- Patlak K_i map (the clinical reference of P:282, Patlak 1983; SURVEY.md §8f-4;
// DESIGN.md R18): per voxel the least-squares line z = K_i x + V0 through the late frames, with
// x_f = int_0^{t_f} Cp / Cp_f and z_f = y_f / Cp_f.  The frame coefficients are draw- and
// voxel-independent and come from the host (api.cu):
//     K_i = sum_f a_f y_f,  a_f = (x_f - xbar) / (Sxx Cp_f);   V0 = sum_f b_f y_f - K_i xbar,  b_f = 1/(m Cp_f)
// (a_f = b_f = 0 for frames before t*), i.e. the centred OLS formulas written as two dot products.
// One thread per voxel, FP64 accumulation, TACs read once (HBM-bound).
#include "common.cuh"

namespace vpet {
namespace {

__global__ void __launch_bounds__(256) patlak_kernel(const PatlakParams p) {
  for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < p.J; j += uint64_t(gridDim.x) * blockDim.x) {
    const float* y = p.tacs + j * p.L;
    double s = 0.0, z = 0.0;
    for (uint32_t f = p.f0; f < p.L; ++f) {
      const double v = double(__ldg(y + f));
      s = fma(p.a[f], v, s);
      z = fma(p.b[f], v, z);
    }
    const float NANF = __int_as_float(0x7fc00000);
    p.ki[j] = p.valid ? float(s) : NANF;
    if (p.intercept) p.intercept[j] = p.valid ? float(z - s * p.xbar) : NANF;
  }
}

}  // namespace

void launch_patlak(const PatlakParams& p, cudaStream_t st) {
  uint64_t blocks = (p.J + 255) / 256;
  if (blocks > 148ull * 16) blocks = 148ull * 16;
  if (blocks == 0) blocks = 1;
  patlak_kernel<<<unsigned(blocks), 256, 0, st>>>(p);
}

}  // namespace vpet
