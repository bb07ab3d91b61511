"""bench.py's reference arm (the oracle timed on the host) runs on CPU:
one complete, measured oracle solve per step on a bounded sample, the contract's JSON
keys, n/nnz from the closed forms, and it never loads the product library."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROBE = r"""
import runpy, sys, json
sys.argv = ["bench.py", "--impl", "reference", "--steps", "2", "--warmup", "1", "--ref-c", "12"]
try:
    runpy.run_path("bench.py", run_name="__main__")
except SystemExit:
    pass
print("LOADED_PRODUCT=" + json.dumps(any(m.startswith("paper_2201_05413_b200") for m in sys.modules)))
"""


def test_reference_arm_measures_the_oracle_without_the_product():
    env = dict(os.environ, OMP_NUM_THREADS="2")
    out = subprocess.run([sys.executable, "-c", PROBE], cwd=ROOT, capture_output=True, text=True, env=env,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    d = json.loads(lines[-1])
    assert d["impl"] == "reference" and d["metric"] == "pcg_time_to_solution" and d["unit"] == "s"
    assert d["higher_is_better"] is False and d["steps"] == 2 and d["warmup"] == 1
    assert d["config"]["n"] == 511 ** 3 and d["config"]["nnz"] == 7 * 511 ** 3 - 6 * 511 ** 2
    assert "c=12" in d["config"]["timed_sample"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["value"] == d["value"] and cb["cores"] == 1 and cb["host_cores"] >= 1
    assert "measured, not scaled" in cb["sample"] and cb["all_cores"]["cores"] == 2
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert 0 < d["value"] < 60
    assert "LOADED_PRODUCT=false" in out.stdout


def test_bench_k1a_byte_accounting(monkeypatch):
    """bench.py's K1a bytes per row over the deferred x update's cycle M follow the
    passes' loads and stores: M - 1 holds read z and p and write p (24),
    the apply reads z, the M directions and x and writes p and x (8 (M + 2) + 16);
    PCG_XDEFER is parsed as the library parses it (atoi: 0 / 2 / 4, other numbers 4,
    no number 0)."""
    import runpy
    g = runpy.run_path(os.path.join(ROOT, "bench.py"), run_name="bench_module")
    for m, v in g["K1A_BYTES"].items():
        want = 40.0 if m == 0 else ((m - 1) * 24 + 8 * (m + 2) + 16) / m
        assert v == want, (m, v, want)
    for env, m in ((None, 4), ("0", 0), ("2", 2), ("4", 4), ("1", 4), ("7", 4), ("x", 0), (" 2", 2)):
        if env is None:
            monkeypatch.delenv("PCG_XDEFER", raising=False)
        else:
            monkeypatch.setenv("PCG_XDEFER", env)
        assert g["xdefer_cycle"]() == m, env
