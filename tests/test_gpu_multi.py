"""Multi-GPU (real NCCL over NVLink) parity of distributed-index-batching: world = 2, 4, 8 as
many GPUs as the box has (tests/dist_step_check.py, one rank per GPU under torchrun)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("precision", [0, 1])
def test_nccl_gradient_equals_union_batch(precision, world):
    if _ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", "--master-port",
           str(29500 + 11 + precision + 2 * world),
           os.path.join(ROOT, "tests", "dist_step_check.py"), str(precision)]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    print(p.stdout[-3000:], p.stderr[-2000:])
    assert p.returncode == 0, p.stderr[-3000:]
