"""bench.py keeps the driver's JSON-line contract: our arm on the GPU (short run) and the reference
arm (the reference's own CPU T2C engine from oracle/_ref) on the host."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRIC = "MLUPS (D3Q19 fp64 BGK) vs porosity; % of HBM peak GB/s; at 1/2/4/8 B200"


def run_bench(*args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                         capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.gpu
def test_our_arm_line():
    d = run_bench("--steps", "8", "--warmup", "3", "--no-sweep", "--no-other", "--no-cpu")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "gpu_launches", "clocks",
              "e2e"):
        assert k in d, k
    assert d["metric"] == METRIC and d["unit"] == "MLUPS" and d["higher_is_better"] is True
    assert d["n_gpus"] == 1 and d["steps"] == 8 and d["warmup"] == 3 and d["dtype"] == "f64"
    assert d["value"] > 0 and d["gpu_launches"] > 0 and "workload" in d["config"]
    sys.path.insert(0, ROOT)
    import bench
    assert d["config"] == bench.workload_config(1, 2032128)  # same dict as the reference arm's
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    c = d["clocks"]
    assert c["sm_mhz"] > 0 and c["sm_max_mhz"] > 0 and isinstance(c["reasons"], list)
    e = d["e2e"]
    assert e["value"] > 0 and e["unit"] == "MLUPS" and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0


def test_reference_arm_line():
    if not any(f.startswith("libsplbm_ref") for f in os.listdir(os.path.join(ROOT, "oracle", "_ref"))
               if os.path.isdir(os.path.join(ROOT, "oracle", "_ref"))):
        pytest.skip("oracle/_ref not built")
    d = run_bench("--impl", "reference", "--steps", "2", "--warmup", "1")
    assert d["impl"] == "reference" and d["metric"] == METRIC and d["unit"] == "MLUPS"
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "MLUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_loads_no_product_code():
    """The reference arm runs the reference's engine only: the product library must not be mapped
    into its process, and its `config` equals the one our arm prints for the same N."""
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libsplbm_ref.so")):
        pytest.skip("oracle/_ref not built")
    code = ("import sys, json; sys.argv=['bench.py','--impl','reference','--steps','1','--warmup','1'];"
            "sys.path.insert(0, '.'); import bench; bench.main();"
            "maps=open('/proc/self/maps').read();"
            "print(json.dumps({'product_loaded': 'libsplbm_b200' in maps,"
            " 'product_imported': any(m.startswith('paper_1703_08015_b200') for m in sys.modules),"
            " 'config': bench.workload_config(1, 2032128)}))")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 2
    line, probe = lines
    assert probe["product_loaded"] is False and probe["product_imported"] is False
    assert line["config"] == probe["config"]
