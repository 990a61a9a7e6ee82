"""Host-side logic without a GPU: the C ABI library loads and exports what
the header declares with the layout ctypes assumes, the packers reproduce
the reference's own packing, the BASELINE configs are well formed, the
product path fails loudly without a device, and the row-sharding exchange
reassembles the full matrix across 2 gloo ranks."""

import os
import subprocess
import sys
import textwrap
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "oracle" / "_ref"


def _reference_available():
    return (REF / "exitmeasure").exists()


@pytest.fixture(scope="module")
def native():
    from paper_2409_03686_b200 import _native
    from paper_2409_03686_b200.build_native import build, lib_path

    if not lib_path().exists():
        build()
    return _native


def test_library_exports_every_declared_symbol(native):
    names = native.exported_symbols()
    assert len(names) >= 15
    missing = [n for n, ok in names if not ok]
    assert not missing, missing


def test_build_info_reports_production_knobs(native):
    """The loaded library was built with the production knobs (a stray
    environment variable at build time cannot change them silently)."""
    from paper_2409_03686_b200.build_native import KNOB_DEFAULTS

    info = native.build_info()
    assert info["arch"] == "sm_100a" and info["debug"] == "0" and info["abi"] == "1"
    for k, v in KNOB_DEFAULTS.items():
        assert info[k] == v, (k, info[k], v)


def test_ctypes_layout_matches_c_header(native, tmp_path):
    """Compile a probe against include/exitmeasure_b200.h and compare struct
    sizes/offsets with the ctypes mirrors in _native.py."""
    import ctypes

    src = tmp_path / "probe.c"
    src.write_text(textwrap.dedent("""
        #include <stdio.h>
        #include <stddef.h>
        #include "exitmeasure_b200.h"
        int main(void) {
          printf("%zu %zu %zu %zu\\n", sizeof(em_geometry), sizeof(em_side),
                 sizeof(em_options), sizeof(em_outputs));
          printf("%zu %zu %zu %zu\\n", offsetof(em_side, wkind), offsetof(em_side, blk_phase),
                 offsetof(em_outputs, err_pole), offsetof(em_geometry, ksqrt));
          return 0;
        }"""))
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    c_sizes = [int(v) for v in out]
    py = [ctypes.sizeof(native.EmGeometry), ctypes.sizeof(native.EmSide),
          ctypes.sizeof(native.EmOptions), ctypes.sizeof(native.EmOutputs),
          native.EmSide.wkind.offset, native.EmSide.blk_phase.offset,
          native.EmOutputs.err_pole.offset, native.EmGeometry.ksqrt.offset]
    assert c_sizes == py


def test_no_device_fails_loudly(native):
    """No CPU fallback: without a GPU the product path raises NativeError."""
    from paper_2409_03686_b200 import backend, configs
    from paper_2409_03686_b200.errors import NativeError

    if native.device_count() > 0:
        pytest.skip("a CUDA device is present")
    cfg = configs.get(1).subset(2, 10)
    s0 = backend.pack_side(cfg.fam0, 2, cfg.eps)
    s1 = backend.pack_side(cfg.fam1, 2, cfg.eps)
    with pytest.raises(NativeError):
        backend.run_accumulate(cfg.dom, cfg.kt.k_sqrt, cfg.poles, 1, cfg.eps, 10**6, 10, s0, s1)


@pytest.mark.skipif(not _reference_available(), reason="oracle/_ref not built")
def test_packing_matches_reference_packer():
    """pack_geometry / pack_side on the reference's own objects give the
    reference's arrays (S/backend.py:71-126)."""
    sys.path.insert(0, str(REF))
    from exitmeasure import backend as rb
    from exitmeasure.geometry import catalog, side_points

    from paper_2409_03686_b200 import backend as B

    for key in ("disc", "annulus", "disc_five_holes", "square_hole", "shell3d"):
        dom = catalog(key)
        g_ref = rb.pack_geometry(dom)
        g = B.pack_geometry(dom)
        assert np.array_equal(g.gi, g_ref.gi) and np.array_equal(g.gf, g_ref.gf)
        assert np.array_equal(g.comp_side, g_ref.comp_side)
        for side in ("gamma0", "gamma1"):
            comps = dom.gamma0 if side == "gamma0" else dom.gamma1
            if not comps:
                continue
            for eps in (1e-8, 0.2):
                pts = side_points(dom, side, [40] * len(comps))
                a = rb.pack_side(pts, dom.dimension, eps)
                b = B.pack_side(pts, dom.dimension, eps)
                assert np.array_equal(a.anchors, b.anchors)
                assert np.array_equal(a.blk, b.blk) and np.array_equal(a.blkf, b.blkf)
                assert np.all(b.blk_phase == 0.0)


def test_baseline_configs_well_formed():
    from paper_2409_03686_b200 import backend, configs
    from paper_2409_03686_b200.geometry import dist_to_boundary

    expect = {1: (32, 128), 2: (256, 512), 3: (1024, 1024), 4: (1024, 2048), 5: (4096, 8146)}
    for idx, (m, nbins) in expect.items():
        cfg = configs.get(idx)
        assert cfg.n_poles == m
        s0 = backend.pack_side(cfg.fam0, cfg.d, cfg.eps)
        s1 = backend.pack_side(cfg.fam1, cfg.d, cfg.eps)
        assert s0.size + s1.size == nbins
        a0, a1 = cfg.split(np.zeros((m, s0.size)), np.zeros((m, s1.size)))
        assert a0.shape[1] + a1.shape[1] == nbins
        dmin = min(dist_to_boundary(cfg.dom, p) for p in cfg.poles)
        assert dmin > cfg.eps
        assert np.allclose(np.linalg.eigvalsh(cfg.kt.k).max(), 1.0)
    # cfg4's two hemisphere lattices are exact mirror images
    c4 = configs.get(4)
    up, lo = c4.fam1.points[:1024], c4.fam1.points[1024:]
    assert np.array_equal(up[:, :2], lo[:, :2]) and np.array_equal(up[:, 2], -lo[:, 2])
    # cfg5: notch faces carry 2 x 2048 squares of side 1/64, outer faces 4050 of 1/30
    c5 = configs.get(5)
    assert c5.fam0.points.shape == (4050, 3) and c5.fam1.points.shape == (4096, 3)
    assert np.all(np.isclose(c5.fam1.points[:, 0], 0.5) | np.isclose(c5.fam1.points[:, 1], 0.5))


def test_conductivity_normalisation_matches_reference():
    if not _reference_available():
        pytest.skip("oracle/_ref not built")
    sys.path.insert(0, str(REF))
    from exitmeasure.conductivity import make_tensor as ref_make

    from paper_2409_03686_b200.conductivity import make_tensor

    for raw in ([[2.0, 0.8], [0.8, 1.0]], np.eye(3) * 5.0, [[3, 1, 0], [1, 2, .5], [0, .5, 1]],
                [[1.0, 0.3], [0.3, 0.4]]):
        a, b = make_tensor(raw), ref_make(raw)
        assert np.array_equal(a.k, b.k) and np.array_equal(a.k_sqrt, b.k_sqrt)


def test_shard_rows_partition():
    from paper_2409_03686_b200.distributed import shard_rows

    for n, w in [(10, 3), (256, 8), (3, 4), (1024, 1)]:
        parts = [shard_rows(n, w, r) for r in range(w)]
        assert np.array_equal(np.sort(np.concatenate(parts)), np.arange(n))


_GLOO_WORKER = textwrap.dedent("""
    import os, sys
    import numpy as np
    import torch, torch.distributed as dist
    sys.path.insert(0, sys.argv[1])
    from paper_2409_03686_b200.distributed import gather_rows, shard_rows
    from paper_2409_03686_b200 import backend, configs
    from oracle import oracle as O
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    cfg = configs.get(3).subset(7, 300)
    geom = backend.pack_geometry(cfg.dom)
    s0 = backend.pack_side(cfg.fam0, 2, cfg.eps); s1 = backend.pack_side(cfg.fam1, 2, cfg.eps)
    ids = shard_rows(cfg.n_poles, world, rank)
    rows = []
    for i in ids:   # the rank's rows, RNG keyed by the GLOBAL pole id
        o0 = np.zeros(s0.size); o1 = np.zeros(s1.size)
        O.accumulate_chunk(geom.gi, geom.gf, geom.comp_side, cfg.kt.k_sqrt, cfg.poles[i], int(i),
                           0, cfg.n_rep, cfg.seed, cfg.eps, 10**6, s0.anchors, s0.blk, s0.blkf, 0,
                           s0.idw_radii, 2, s1.anchors, s1.blk, s1.blkf, 0, s1.idw_radii, 2, o0, o1)
        rows.append(np.concatenate([o0, o1]))
    local = torch.as_tensor(np.array(rows, dtype=np.int64))
    full = gather_rows(local, cfg.n_poles, world).numpy()
    raw0, raw1, *_ = O.run_accumulate_packed(geom.gi, geom.gf, geom.comp_side, cfg.kt.k_sqrt,
        cfg.poles, cfg.seed, cfg.eps, 10**6, cfg.n_rep, (s0.anchors, s0.blk, s0.blkf),
        (s1.anchors, s1.blk, s1.blkf), threads=1)
    assert np.array_equal(full, np.concatenate([raw0, raw1], 1).astype(np.int64)), rank
    dist.barrier(); dist.destroy_process_group()
    print("rank", rank, "ok")
""")


def test_row_sharded_gather_gloo_two_ranks(tmp_path):
    """world_size 2 over gloo: cyclic row shards keyed by global pole ids,
    gathered, equal the single-process result exactly."""
    w = tmp_path / "worker.py"
    w.write_text(_GLOO_WORKER)
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", PYTHONPATH=str(ROOT))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29577", str(w), str(ROOT)]
    res = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-3000:]
    assert res.stdout.count("ok") == 2


def test_spectral_requires_a_device():
    """Device Gram/SVD have no CPU fallback: without CUDA they raise."""
    import torch

    from paper_2409_03686_b200 import spectral
    from paper_2409_03686_b200.errors import NativeError, ValidationError

    if torch.cuda.is_available():
        pytest.skip("a CUDA device is visible")
    with pytest.raises(NativeError):
        spectral.gram(np.ones((3, 2)), np.ones(2), np.ones(3))
    with pytest.raises(ValidationError):
        spectral.svd(np.ones(3))
    with pytest.raises(ValidationError):
        spectral.sym_eig(np.array([[1.0, 2.0], [0.0, 1.0]]))


def test_plan_cache_key_is_exact_content():
    """The run_accumulate plan cache keys on the exact bytes of every input
    (no digest): equal content -> equal key; any changed element, dtype,
    shape, scalar or option -> a different key; the reference's SidePack
    (no blk_phase field) is accepted."""
    from dataclasses import dataclass

    from paper_2409_03686_b200 import backend as B, configs

    cfg = configs.get(2)
    geom = B.pack_geometry(cfg.dom)
    s0 = B.pack_side(cfg.fam0, 2, cfg.eps)
    s1 = B.pack_side(cfg.fam1, 2, cfg.eps)
    args = (geom, cfg.kt.k_sqrt, cfg.poles, cfg.eps, 10**6, s0, s1, "fp32", "max", 0, None)
    k = B._plan_key(*args)
    assert B._plan_key(*(geom, cfg.kt.k_sqrt.copy(), cfg.poles.copy()) + args[3:]) == k
    p2 = cfg.poles.copy()
    p2[17, 1] = np.nextafter(p2[17, 1], 1.0)
    assert B._plan_key(geom, cfg.kt.k_sqrt, p2, *args[3:]) != k
    assert B._plan_key(*args[:3], cfg.eps * 2, *args[4:]) != k
    assert B._plan_key(*args[:7], "ref64", *args[8:]) != k
    assert B._plan_key(*args[:10], np.arange(cfg.n_poles)) != k
    a1 = s1.anchors.copy()
    a1[0, 0] += 1e-12
    s1b = B.SidePack(a1, s1.blk, s1.blkf, s1.weights_kind, s1.idw_radii, s1.idw_power,
                     s1.blk_phase)
    assert B._plan_key(*args[:6], s1b, *args[7:]) != k

    @dataclass(frozen=True)
    class RefSidePack:  # the reference's field set (S/backend.py:57-68)
        anchors: np.ndarray
        blk: np.ndarray
        blkf: np.ndarray
        weights_kind: int
        idw_radii: np.ndarray
        idw_power: int

    r1 = RefSidePack(s1.anchors, s1.blk, s1.blkf, s1.weights_kind, s1.idw_radii, s1.idw_power)
    assert B._plan_key(*args[:6], r1, *args[7:]) != k  # no phase -> different plan


def test_tangent_chain_resolution():
    """Which geometries walk on tangent balls (em_resolve_chain, no device):
    the BASELINE configs with K != I (cfg2 box, cfg3 concentric annulus, cfg4
    ball, cfg5 L-box) resolve "tangent" to itself, cfg1 (K = I), an annulus
    with an off-centre hole and a box with a hole to "max"; "max" / "woe"
    are kept; REF64 runs the reference chain only."""
    from paper_2409_03686_b200 import backend as B, configs
    from paper_2409_03686_b200.errors import NativeError

    for idx, want in ((1, "max"), (2, "tangent"), (3, "tangent"), (4, "tangent"),
                      (5, "tangent")):
        cfg = configs.get(idx)
        geom = B.pack_geometry(cfg.dom)
        assert B.resolve_chain(geom, cfg.kt.k_sqrt, "fp32", "tangent") == want, idx
        assert B.resolve_chain(geom, cfg.kt.k_sqrt, "fp32", "max") == "max"
        assert B.resolve_chain(geom, cfg.kt.k_sqrt, "fp32", "woe") == "woe"
        assert B.resolve_chain(geom, cfg.kt.k_sqrt, "ref64", "woe") == "woe"
        with pytest.raises(NativeError):
            B.resolve_chain(geom, cfg.kt.k_sqrt, "ref64", "tangent")
    k2 = configs.get(2).kt.k_sqrt
    off = B.GeomPack(np.array([2, 0, 1]), np.array([0.0, 0.0, 1.0, 0.1, 0.0, 0.4]),
                     np.array([0, 1], dtype=np.int8))
    assert B.resolve_chain(off, k2, "fp32", "tangent") == "max"
    conc = B.GeomPack(np.array([2, 0, 1]), np.array([0.0, 0.0, 1.0, 0.0, 0.0, 0.4]),
                      np.array([0, 1], dtype=np.int8))
    assert B.resolve_chain(conc, k2, "fp32", "tangent") == "tangent"
    holed_box = B.GeomPack(np.array([2, 1, 1]), np.array([0.0, 0.0, 1.0, 0.2, 0.0, 0.3]),
                           np.array([0, 1], dtype=np.int8))
    assert B.resolve_chain(holed_box, k2, "fp32", "tangent") == "max"
    with pytest.raises(NativeError):  # invalid geometry: dimension 4
        B.resolve_chain(B.GeomPack(np.array([4, 1, 0]), np.zeros(5), np.zeros(1, np.int8)),
                        np.eye(4), "fp32", "tangent")


_BUDGET_WORKER = textwrap.dedent("""
    import sys
    import torch.distributed as dist
    sys.path.insert(0, sys.argv[1])
    from paper_2409_03686_b200.distributed import agree_on_budget_error
    from paper_2409_03686_b200.errors import WalkBudgetError
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    # rank 0 fails at global (pole 5, rep 3), rank 1 at (pole 2, rep 7): every
    # rank must raise the lexicographically first one, (2, 7)
    cases = [({0: (5, 3), 1: (2, 7)}, (2, 7)), ({1: (4, 0)}, (4, 0)), ({}, None)]
    for errs, want in cases:
        e = WalkBudgetError(*errs[rank], 100) if rank in errs else None
        try:
            agree_on_budget_error(e, 10, 100, "cpu")
            got = None
        except WalkBudgetError as x:
            got = (x.pole, x.replicate)
            assert x.max_steps == 100
        assert got == want, (rank, got, want)
    dist.barrier(); dist.destroy_process_group()
    print("rank", rank, "ok")
""")


def test_budget_error_agreed_across_gloo_ranks(tmp_path):
    """A budget overrun on any rank is raised on EVERY rank (the global
    lexicographic minimum) before the gather, so no rank is left blocking in
    the collective."""
    w = tmp_path / "worker.py"
    w.write_text(_BUDGET_WORKER)
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", PYTHONPATH=str(ROOT))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29579", str(w), str(ROOT)]
    res = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-3000:]
    assert res.stdout.count("ok") == 2


def test_bench_gpus_flag_spawns_ranks():
    """`bench.py --gpus 2` without a torchrun environment launches two ranks
    itself (the driver's N>1 contract); the gloo harness check reports both."""
    import json

    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2",
                          "--harness-check"], capture_output=True, text=True, env=env,
                         timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    line = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(line) == 1, res.stdout
    d = json.loads(line[0])
    assert d["n_gpus"] == 2 and d["ranks"] == [0, 1]


def test_bench_rejects_world_mismatch():
    """Under torchrun, --gpus must equal WORLD_SIZE (no silent 1-GPU timing)."""
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "4"],
                         capture_output=True, text=True, env=env, timeout=600)
    assert res.returncode == 2 and "WORLD_SIZE" in res.stderr


_EXCHANGE_WORKER = textwrap.dedent("""
    import sys
    import torch, torch.distributed as dist
    sys.path.insert(0, sys.argv[1])
    from paper_2409_03686_b200.distributed import cyclic_gather_index, exchange_rows, shard_rows
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    for n_poles, row in ((7, 5), (8, 3), (1, 4)):
        ids = shard_rows(n_poles, world, rank)
        m_pad = -(-n_poles // world)
        buf = torch.full((m_pad * row + 3 * m_pad,), -1, dtype=torch.int64)
        rows = buf[: m_pad * row].view(m_pad, row)
        for j, g in enumerate(ids):  # this rank's rows hold their GLOBAL pole id
            rows[j] = torch.arange(row) + 1000 * int(g)
        gathered = torch.zeros((world, buf.numel()), dtype=torch.int64)
        out = torch.zeros((n_poles, row), dtype=torch.int64)
        exchange_rows(buf, gathered, cyclic_gather_index(n_poles, world, m_pad), m_pad, row, out)
        want = torch.arange(row)[None, :] + 1000 * torch.arange(n_poles)[:, None]
        assert torch.equal(out, want), (rank, n_poles, out)
    dist.barrier(); dist.destroy_process_group()
    print("rank", rank, "ok")
""")


def test_strong_scaling_exchange_gloo_two_ranks(tmp_path):
    """The bench's per-step exchange (one all-gather of the flat blocks, the
    un-permute to pole order) reassembles cyclic row shards -- ragged shards
    and an empty shard included -- on 2 gloo ranks."""
    w = tmp_path / "worker.py"
    w.write_text(_EXCHANGE_WORKER)
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", PYTHONPATH=str(ROOT))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29581", str(w), str(ROOT)]
    res = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-3000:]
    assert res.stdout.count("ok") == 2
