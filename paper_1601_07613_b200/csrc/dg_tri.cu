// Kernel instantiations for tri elements (advection and Euler).
#include "dg_ops.h"

namespace mcdg {

Ops* ops_tri(int phys, int p) {
  switch (phys * 16 + p) {
    case ADV * 16 + 1: return Instance<TRI, ADV, 1>::ops();
    case EULER * 16 + 1: return Instance<TRI, EULER, 1>::ops();
    case ADV * 16 + 2: return Instance<TRI, ADV, 2>::ops();
    case EULER * 16 + 2: return Instance<TRI, EULER, 2>::ops();
    case ADV * 16 + 3: return Instance<TRI, ADV, 3>::ops();
    case EULER * 16 + 3: return Instance<TRI, EULER, 3>::ops();
    case ADV * 16 + 4: return Instance<TRI, ADV, 4>::ops();
    case EULER * 16 + 4: return Instance<TRI, EULER, 4>::ops();
    default: return nullptr;
  }
}

}  // namespace mcdg
