"""The NCCL row-sharded path end to end on the GPU box: torchrun with one
rank per visible GPU (1 here) runs distributed.run_accumulate_sharded --
walks into device tensors, all-gathers the rows over NCCL -- and must equal
the single-process run_accumulate exactly."""

import os
import subprocess
import sys
import textwrap
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

WORKER = textwrap.dedent("""
    import sys
    import numpy as np
    import torch, torch.distributed as dist
    sys.path.insert(0, sys.argv[1])
    from paper_2409_03686_b200 import backend, configs
    from paper_2409_03686_b200.distributed import run_accumulate_sharded
    local = int(__import__("os").environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    for prec in ("fp32", "ref64"):
        cfg = configs.get(3).subset(24, 2000)
        s0 = backend.pack_side(cfg.fam0, 2, cfg.eps); s1 = backend.pack_side(cfg.fam1, 2, cfg.eps)
        r = run_accumulate_sharded(cfg.dom, cfg.kt.k_sqrt, cfg.poles, cfg.seed, cfg.eps, 10**6,
                                   cfg.n_rep, s0, s1, precision=prec)
        if dist.get_rank() == 0:
            ref = backend.run_accumulate(cfg.dom, cfg.kt.k_sqrt, cfg.poles, cfg.seed, cfg.eps,
                                         10**6, cfg.n_rep, s0, s1, precision=prec)
            assert np.array_equal(r.counts, ref.counts), prec
            assert np.array_equal(r.steps_sum, ref.steps_sum), prec
            assert np.array_equal(r.raw1, ref.raw1), prec
            print("ok", prec, flush=True)
    dist.barrier(); dist.destroy_process_group()
""")


def test_nccl_sharded_equals_single(tmp_path):
    from paper_2409_03686_b200 import _native

    n = _native.device_count()
    assert n >= 1
    w = tmp_path / "worker.py"
    w.write_text(WORKER)
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29583", str(w), str(ROOT)]
    res = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-3000:]
    assert res.stdout.count("ok ") == 2
