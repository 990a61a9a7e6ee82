"""All-pole entry-wise parity at BASELINE scale (GPU box; evidence run, too
long for the suite): every pole of cfg3 / cfg4 at 1e6 FP32 walks against
1e5 walks per pole of the reference itself (oracle/_ref, all host threads),
cfg5's 4096 poles at 1e6 against 1e4 C-oracle walks per pole.  SURVEY
Appendix B statistics (exact conditional tails) into
gpurun_out/fullscale_allpoles_cfgC.json.
    python tools/fullscale_parity.py [3 4 5]"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle import oracle as O  # noqa: E402  (test infrastructure: the checker)
from paper_2409_03686_b200 import _native, backend as B, configs  # noqa: E402
import test_gpu_fullscale as F  # noqa: E402

_native.require_device(0)
O.lib()
for idx in [int(a) for a in sys.argv[1:]] or [3, 4, 5]:
    cfg = configs.get(idx)
    n_ref = 10**4 if idx == 5 else 10**5
    t0 = time.perf_counter()
    gpu = F._gpu_counts(B, cfg, 10**6, cfg.seed)
    t1 = time.perf_counter()
    ref = F.reference_counts(cfg, n_ref, cfg.seed + 1, O)
    t2 = time.perf_counter()
    s = F.appendix_b(gpu, 10**6, ref, n_ref, f"allpoles_cfg{idx}")
    ok = (s["exceed_z4"] <= s["exceed_z4_q999"] and s["max_abs_z_equiv"] <= s["bonferroni_z"]
          and s["row_chi2_min_p"] > 1e-4 / s["rows"] and s["row_chi2_ks_uniform_p"] > 1e-3)
    print(f"cfg{idx}: {cfg.n_poles} poles, GPU 1e6 walks/pole ({t1 - t0:.1f} s) vs reference "
          f"{n_ref:.0e} ({t2 - t1:.1f} s): |z|>4 {s['exceed_z4']} (q999 {s['exceed_z4_q999']}), "
          f"max |z| {s['max_abs_z_equiv']:.2f} (Bonferroni {s['bonferroni_z']:.2f}), row chi2 KS p "
          f"{s['row_chi2_ks_uniform_p']:.3f}, min row p {s['row_chi2_min_p']:.2e} -> "
          f"{'PASS' if ok else 'FAIL'}", flush=True)
