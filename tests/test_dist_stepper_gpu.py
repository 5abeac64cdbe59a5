"""The distributed stepper end to end through torch.distributed: torchrun
with 2 and 3 ranks (gloo, host-staged exchange, ranks sharing the one GPU of
this pool — a functional check, no timing) runs ``ssprk3_distributed``
(overlapped stage, kernel-packed send rows, receives into ghost rows) and
must reproduce the single-domain SSP-RK3 result bit for bit."""

import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,kind", [(2, "tet"), (3, "tet"), (2, "tri")])
def test_distributed_stepper_matches_single_domain(cuda, tmp_path, world, kind):
    out = tmp_path / "check.txt"
    env = dict(os.environ, MC_DIST_BACKEND="gloo", DIST_CHECK_OUT=str(out),
               DIST_CHECK_KIND=kind)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={world}", "--master-addr", "127.0.0.1",
                        "--master-port", str(_port()), str(ROOT / "tools" / "dist_check.py")],
                       env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
    assert out.read_text() == "ok"
