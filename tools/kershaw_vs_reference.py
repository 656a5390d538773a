"""The reference's own benchmark driver (tmopbench.bench.run_benchmark,
bench.py:171-241; reference CLI defaults: Kershaw 12^3, p = 2, n_q = 6,
mu_303, Jacobi-MINRES) on the host cores vs this package's GPU driver
(paper_2205_12721_b200.kershaw_bench.run_benchmark) on the same
configuration, both writing the reference's CSV row.  Run on the GPU box:

    python tools/kershaw_vs_reference.py --out profiles/round2_kershaw12_vs_reference.json
"""
import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import os, sys, json, time
sys.path.insert(0, sys.argv[1])
import tmopbench.bench as rb
cfg = rb.BenchConfig(nx=int(sys.argv[2]), ny=int(sys.argv[2]), nz=int(sys.argv[2]), order=int(sys.argv[3]),
                     n_quad=int(sys.argv[4]), csv_path=sys.argv[5])
rep = rb.run_benchmark(cfg)
print(json.dumps({"total_s": rep.times["total"], "newton": rep.newton_iterations, "minres": rep.minres_iterations,
                  "status": rep.status, "f_final": rep.f_final, "max_dev_uniform": rep.max_dev_uniform,
                  "hessian_apply_s": rep.times["hessian_apply"]}))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=12)
    ap.add_argument("--order", type=int, default=2)
    ap.add_argument("--nq", type=int, default=6)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    sys.path.insert(0, ROOT)
    from paper_2205_12721_b200 import kershaw_bench as KB
    tmp = tempfile.mkdtemp()
    cores = len(os.sched_getaffinity(0))
    env = dict(os.environ, NUMBA_NUM_THREADS=str(cores), OMP_NUM_THREADS=str(cores),
               OPENBLAS_NUM_THREADS=str(cores), PYTHONDONTWRITEBYTECODE="1",
               NUMBA_CACHE_DIR=os.path.join(tmp, "numba"))
    ref_csv = os.path.join(tmp, "ref.csv")
    t = time.perf_counter()
    r = subprocess.run([sys.executable, "-c", CHILD, os.path.join(ROOT, "baseline", "_ref"), str(a.n), str(a.order),
                        str(a.nq), ref_csv], env=env, capture_output=True, text=True, timeout=3600)
    if r.returncode != 0:
        raise SystemExit(r.stderr[-3000:])
    ref = json.loads(r.stdout.strip().splitlines()[-1])
    ref["wall_incl_jit_s"] = time.perf_counter() - t
    gpu_csv = os.path.join(tmp, "gpu.csv")
    KB.run_benchmark(KB.BenchConfig(nx=a.n, ny=a.n, nz=a.n, order=a.order, n_quad=a.nq))      # warm-up
    rep = KB.run_benchmark(KB.BenchConfig(nx=a.n, ny=a.n, nz=a.n, order=a.order, n_quad=a.nq, csv_path=gpu_csv))
    fused = KB.run_benchmark(KB.BenchConfig(nx=a.n, ny=a.n, nz=a.n, order=a.order, n_quad=a.nq), fused=True)
    out = {"config": f"Kershaw eps 0.3, {a.n}^3 hexes, p={a.order}, n_q={a.nq}, mu_303, Jacobi-MINRES "
                     f"(the reference CLI defaults)",
           "reference_cpu": dict(ref, cores=cores, csv=KB.read_csv_row(ref_csv)),
           "gpu_kernel_timer": {"total_s": rep.times["total"], "newton": rep.newton_iterations,
                                "minres": rep.minres_iterations, "status": rep.status, "f_final": rep.f_final,
                                "max_dev_uniform": rep.max_dev_uniform, "hessian_apply_s": rep.times["hessian_apply"],
                                "csv": KB.read_csv_row(gpu_csv)},
           "gpu_fused": {"total_s": fused.times["total"], "newton": fused.newton_iterations,
                         "minres": fused.minres_iterations, "status": fused.status,
                         "max_dev_uniform": fused.max_dev_uniform},
           "speedup_total": ref["total_s"] / fused.times["total"]}
    with open(a.out, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps({k: out[k] for k in ("config", "speedup_total")}))


if __name__ == "__main__":
    main()
