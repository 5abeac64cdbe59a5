// Kernel instantiations for conforming triangle + quad meshes (advection
// and Euler; register kernels only: N_eq * (p+1)^2 <= 64).
#include "dg_ops.h"

namespace mcdg {

Ops* ops_hyb(int phys, int p) {
  switch (phys * 16 + p) {
    case ADV * 16 + 1: return Instance<HYB, ADV, 1>::ops();
    case EULER * 16 + 1: return Instance<HYB, EULER, 1>::ops();
    case ADV * 16 + 2: return Instance<HYB, ADV, 2>::ops();
    case EULER * 16 + 2: return Instance<HYB, EULER, 2>::ops();
    case ADV * 16 + 3: return Instance<HYB, ADV, 3>::ops();
    case EULER * 16 + 3: return Instance<HYB, EULER, 3>::ops();
    default: return nullptr;
  }
}

}  // namespace mcdg
