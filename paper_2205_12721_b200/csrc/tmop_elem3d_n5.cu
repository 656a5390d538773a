// Element-kernel instantiations: 3D hexes, p = 4 (n1 = 5), n_q = 2..9.
#include "tmop_launch.cuh"

namespace tmop {
int launch_elem_3d_n5(int nq, int kind, ElemArgs &a, const Tab &t, cudaStream_t s) {
  return launch_q<3, 5>(nq, kind, a, t, s);
}
}  // namespace tmop
