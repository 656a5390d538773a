// Element-kernel instantiations: 3D hexes, p = 1 (n1 = 2), n_q = 2..9.
#include "tmop_launch.cuh"

namespace tmop {
int launch_elem_3d_n2(int nq, int kind, ElemArgs &a, const Tab &t, cudaStream_t s) {
  return launch_q<3, 2>(nq, kind, a, t, s);
}
}  // namespace tmop
