// tmop_internal.h -- host-side declarations shared by the C-ABI layer and
// the per-(dim, p) kernel instantiation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "tmop_device.cuh"

namespace tmop {

struct ElemArgs;

// Launch the element kernel `kind` for (dim, n1 = p+1, nq).  Returns the
// grid size used (>= 0) or -1 if (dim, n1, nq) is not instantiated.
int launch_elem(int dim, int n1, int nq, int kind, ElemArgs &a, const Tab &t, cudaStream_t s);
int launch_elem_2d(int n1, int nq, int kind, ElemArgs &a, const Tab &t, cudaStream_t s);
int launch_elem_3d_n2(int nq, int kind, ElemArgs &a, const Tab &t, cudaStream_t s);
int launch_elem_3d_n3(int nq, int kind, ElemArgs &a, const Tab &t, cudaStream_t s);
int launch_elem_3d_n4(int nq, int kind, ElemArgs &a, const Tab &t, cudaStream_t s);
int launch_elem_3d_n5(int nq, int kind, ElemArgs &a, const Tab &t, cudaStream_t s);
bool elem_supported(int dim, int n1, int nq);

}  // namespace tmop
