// Kernel instantiations for quad elements (advection and Euler).
#include "dg_ops.h"

namespace mcdg {

Ops* ops_quad(int phys, int p) {
  switch (phys * 16 + p) {
    case ADV * 16 + 1: return Instance<QUAD, ADV, 1>::ops();
    case EULER * 16 + 1: return Instance<QUAD, EULER, 1>::ops();
    case ADV * 16 + 2: return Instance<QUAD, ADV, 2>::ops();
    case EULER * 16 + 2: return Instance<QUAD, EULER, 2>::ops();
    case ADV * 16 + 3: return Instance<QUAD, ADV, 3>::ops();
    case EULER * 16 + 3: return Instance<QUAD, EULER, 3>::ops();
    default: return nullptr;
  }
}

}  // namespace mcdg
