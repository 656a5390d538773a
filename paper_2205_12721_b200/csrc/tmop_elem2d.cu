// Element-kernel instantiations: 2D quads, p = 1..4, n_q = 2..9.
#include "tmop_launch.cuh"

namespace tmop {
int launch_elem_2d(int n1, int nq, int kind, ElemArgs &a, const Tab &t, cudaStream_t s) {
  switch (n1) {
    case 2: return launch_q<2, 2>(nq, kind, a, t, s);
    case 3: return launch_q<2, 3>(nq, kind, a, t, s);
    case 4: return launch_q<2, 4>(nq, kind, a, t, s);
    case 5: return launch_q<2, 5>(nq, kind, a, t, s);
    default: return -1;
  }
}
}  // namespace tmop
