"""Multi-GPU path on real GPUs: torchrun with one rank per GPU, NCCL
communicator through the C ABI, parity with the oracle (tests/mgpu_parity.py):
with a single rank (nranks = 1: the NCCL allgathers, the grouped broadcasts,
the collective digest and the deferred cyclic join all run on one GPU) and
with every visible GPU when there are 2 or more."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("ranks", ["one", "all"])
def test_multi_gpu_sweep_matches_oracle(ranks):
    import torch
    n = torch.cuda.device_count()
    if n < 1:
        pytest.skip("no GPU")
    if ranks == "all" and n < 2:
        pytest.skip("needs >= 2 GPUs")
    n = 1 if ranks == "one" else min(n, 8)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={29561 + n}", str(ROOT / "tests" / "mgpu_parity.py")]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900,
                         env=dict(os.environ, PYTHONPATH=str(ROOT)))
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "MGPU_PARITY OK" in out.stdout
