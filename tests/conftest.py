"""Shared fixtures: golden loader, GPU marker, product/oracle imports."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def load_golden(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def manifest() -> dict:
    return json.loads((GOLDEN / "manifest.json").read_text())


MESH_CASES = [n for n in manifest()["cases"] if not n.startswith("amr_")]
AMR_CASES = [n for n in manifest()["cases"] if n.startswith("amr_")]


def golden_mesh(g: dict, prefix: str = "mesh_"):
    """Rebuild a product Mesh from golden arrays (no re-assembly)."""
    from paper_1601_07613_b200.mesh import Mesh
    return Mesh(*(np.array(g[prefix + n]) for n in (
        "vertices", "elem_kind", "elem_verts", "elem_surfs", "surf_verts",
        "surf_elems")))


def build_case(name: str):
    """Rebuild a golden case with the PRODUCT generators."""
    import paper_1601_07613_b200 as P
    table = {
        "tri_6x5": lambda: P.gen_tri_rect(6, 5),
        "tri_8x8": lambda: P.gen_tri_rect(8, 8),
        "tri_8x8_per": lambda: P.gen_tri_rect(8, 8, (True, True)),
        "tri_6x6_per": lambda: P.gen_tri_rect(6, 6, (True, True)),
        "tri_64x64": lambda: P.gen_tri_rect(64, 64),
        "shuf_tri_64": lambda: P.shuffle_elements(P.gen_tri_rect(64, 64), 0),
        "shuf_tri_16": lambda: P.shuffle_elements(P.gen_tri_rect(16, 16), 0),
        "quad_5x5": lambda: P.gen_quad_rect(5, 5),
        "quad_16x16": lambda: P.gen_quad_rect(16, 16),
        "quad_4x4_per": lambda: P.gen_quad_rect(4, 4, (True, True)),
        "tet_2x2x2": lambda: P.gen_tet_prism(2, 2, 2),
        "tet_4x4x4": lambda: P.gen_tet_prism(4, 4, 4),
        "shuf_tet_3": lambda: P.shuffle_elements(P.gen_tet_prism(3, 3, 3), 5),
        "hybrid_4x4": lambda: hybrid_patch(4, 4),
    }
    return table[name]()


def hybrid_patch(nx, ny):
    """Conforming tri/quad mix (the reference tests' conftest.hybrid_patch)."""
    import paper_1601_07613_b200 as P
    verts = [(i, j) for j in range(ny + 1) for i in range(nx + 1)]
    vid = lambda i, j: j * (nx + 1) + i
    elems = []
    for j in range(ny):
        for i in range(nx):
            a, b, c, d = vid(i, j), vid(i + 1, j), vid(i + 1, j + 1), vid(i, j + 1)
            if (i + j) % 2 == 0:
                elems += [("tri", (a, b, c)), ("tri", (a, c, d))]
            else:
                elems.append(("quad", (a, b, c, d)))
    return P.build_surfaces(np.asarray(verts, dtype=float), elems)


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture
def cuda():
    if not has_gpu():
        pytest.skip("no CUDA device")
    import torch
    return torch.device("cuda")
