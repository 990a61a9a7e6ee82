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


@pytest.mark.parametrize("scaling", ["strong", "weak"])
def test_bench_multi_rank_path_self_test(scaling):
    """bench.py's N > 1 path end to end with 2 ranks on this one GPU
    (EXITMEASURE_B200_DEVICE=0; the ranks' kernels are independent and the
    exchange runs over gloo on the host -- a harness self-test, not a
    measurement): row shards / replicate ranges, the all-gather and
    un-permute (strong) or row sum (weak), max-over-ranks timing, the e2e
    path, one JSON line from rank 0 with n_gpus 2."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["EXITMEASURE_B200_DEVICE"] = "0"
    res = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--dist-backend",
                          "gloo", "--scaling", scaling, "--config", "2", "--steps", "2",
                          "--warmup", "3", "--no-cpu-baseline"], capture_output=True, text=True,
                         env=env, timeout=900)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-4000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == scaling
    assert d["value"] > 0 and d["e2e"]["value"] > 0
    if scaling == "weak":
        assert "row sums ok" in d["config"]["parallelism"]
