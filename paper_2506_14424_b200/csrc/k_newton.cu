// k_newton.cu — Newton-linearised viscous apply (K2).  Placeholder until the kernel lands.
#include "tu_tables.cuh"
#include "launch.h"

namespace dgvv {
cudaError_t upload_tables_newton(const Tab1D* tabs) { return tu_upload_tables(tabs); }
cudaError_t launch_newton(int, int, const ApplyArgs&, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace dgvv
