"""h-convergence table of the DG path on periodic boxes (GPU): relative L2 errors
and observed rates for a wave carried by advection / the Euler free stream."""
import sys, numpy as np
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / 'tests'))
import paper_1601_07613_b200 as P
from test_convergence_gpu import wave_error
for name, gen in (("quad", lambda n: P.gen_quad_rect(n, n, (True, True))), ("tri", lambda n: P.gen_tri_rect(n, n, (True, True)))):
    for phys in ("euler", "advection"):
        for p in (1, 2, 3):
            ns = (8, 16, 32, 64)
            e = [wave_error(gen, n, p, phys) / n for n in ns]
            print(name, phys, p, ["%.3e" % x for x in e], ["%.2f" % np.log2(e[i] / e[i + 1]) for i in range(3)], flush=True)
