"""Where does the one-shot API call spend its time? (GPU box)
python tools/e2e_profile.py [cfg]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2409_03686_b200 import _native as N, backend as B, configs  # noqa: E402

cfg = configs.get(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
lib = N.lib()
tim = {}


def wrap(name):
    f = getattr(lib, name)

    class W:
        def __call__(self, *a):
            t = time.perf_counter()
            r = f(*a)
            tim[name] = tim.get(name, 0.0) + time.perf_counter() - t
            return r

        def __getattr__(self, k):
            return getattr(f, k)
    setattr(lib, name, W())


for n in ("em_plan_create", "em_plan_run_host", "em_plan_destroy", "em_plan_last_stats"):
    wrap(n)
for it in range(6):
    tim.clear()
    t0 = time.perf_counter()
    geom = B.pack_geometry(cfg.dom)
    s0 = B.pack_side(cfg.fam0, cfg.d, cfg.eps)
    s1 = B.pack_side(cfg.fam1, cfg.d, cfg.eps)
    t1 = time.perf_counter()
    plan = B.Plan(geom, cfg.kt.k_sqrt, cfg.poles, cfg.eps, 10**6, s0, s1, precision="fp32")
    t2 = time.perf_counter()
    r = plan.run(cfg.seed, cfg.n_rep)
    t3 = time.perf_counter()
    plan.close()
    t4 = time.perf_counter()
    c = {k: 1e3 * v for k, v in tim.items()}
    print(f"iter {it}: pack {1e3*(t1-t0):.3f} ms, plan {1e3*(t2-t1):.3f} ms "
          f"(C {c.get('em_plan_create', 0):.3f}), run {1e3*(t3-t2):.3f} ms "
          f"(C {c.get('em_plan_run_host', 0):.3f}, kernel {r.kernel_ms:.3f}), "
          f"close {1e3*(t4-t3):.3f} ms, total {1e3*(t4-t0):.3f} ms")
t0 = time.perf_counter()
for _ in range(5):
    r = B.run_accumulate(cfg.dom, cfg.kt.k_sqrt, cfg.poles, cfg.seed, cfg.eps, 10**6, cfg.n_rep,
                         B.pack_side(cfg.fam0, cfg.d, cfg.eps), B.pack_side(cfg.fam1, cfg.d, cfg.eps),
                         precision="fp32")
print(f"run_accumulate: {1e3*(time.perf_counter()-t0)/5:.3f} ms per call (kernel {r.kernel_ms:.3f})")

if len(sys.argv) > 2 and sys.argv[2] == "prof":
    import cProfile
    import pstats

    s0 = B.pack_side(cfg.fam0, cfg.d, cfg.eps)
    s1 = B.pack_side(cfg.fam1, cfg.d, cfg.eps)
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(50):
        B.run_accumulate(cfg.dom, cfg.kt.k_sqrt, cfg.poles, cfg.seed, cfg.eps, 10**6, cfg.n_rep,
                         s0, s1, precision="fp32", cache=False)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)

# the reference's entry point with the plugin installed (bench.py's e2e path)
ref = Path(__file__).resolve().parents[1] / "oracle" / "_ref"
if (ref / "exitmeasure").exists():
    sys.path.insert(0, str(ref))
    from paper_2409_03686_b200 import plugin

    rb = plugin.install(precision="fp32", cache=False)
    s0 = B.pack_side(cfg.fam0, cfg.d, cfg.eps)
    s1 = B.pack_side(cfg.fam1, cfg.d, cfg.eps)
    for it in range(4):
        t0 = time.perf_counter()
        r = B.run_accumulate(cfg.dom, cfg.kt.k_sqrt, cfg.poles, cfg.seed, cfg.eps, 10**6,
                             cfg.n_rep, s0, s1, precision="fp32", cache=False)
        t1 = time.perf_counter()
        a0, a1 = r.raw0, r.raw1
        t2 = time.perf_counter()
        rr = rb.run_accumulate(cfg.dom, cfg.kt.k_sqrt, cfg.poles, cfg.seed, cfg.eps, 10**6,
                               cfg.n_rep, s0, s1)
        t3 = time.perf_counter()
        print(f"plugin path: backend.run_accumulate {1e3*(t1-t0):.3f} ms (kernel "
              f"{r.kernel_ms:.3f}), raw0/raw1 float64 {1e3*(t2-t1):.3f} ms, reference entry "
              f"point total {1e3*(t3-t2):.3f} ms")
    plugin.uninstall(rb)
