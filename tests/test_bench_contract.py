"""bench.py contract on the CPU: the reference arm (--impl reference, the
oracle port of the reference's CPU path) prints one JSON line with the
driver's keys; ranks other than 0 exit without output."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=600, env=e, cwd=ROOT)


def test_reference_arm_line():
    p = _run(["--impl", "reference", "--config", "cfg0", "--steps", "2", "--warmup", "1"])
    assert p.returncode == 0, p.stderr
    lines = [l for l in p.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 1
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"]["workload"] == "cfg0"
    cb = d["cpu_baseline"]
    assert cb["value"] == d["value"] and cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["sample"]
    e2e = d["e2e"]
    assert e2e["value"] == d["value"] and e2e["unit"] == d["unit"]
    assert e2e["h2d_bytes_per_step"] == 0 and e2e["d2h_bytes_per_step"] == 0


def test_reference_arm_other_ranks_are_silent():
    p = _run(["--impl", "reference", "--config", "cfg0", "--steps", "1", "--warmup", "1"],
             env={"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert p.returncode == 0, p.stderr
    assert p.stdout.strip() == ""


def test_both_arms_report_the_same_config():
    """The driver compares the two arms' config dicts: both come from
    bench.static_config, and the reference arm runs the reference's own code
    (oracle/_ref) when it is built."""
    sys.path.insert(0, ROOT)
    import bench

    p = _run(["--impl", "reference", "--config", "cfg0", "--steps", "1", "--warmup", "1", "--no-accuracy"])
    assert p.returncode == 0, p.stderr
    d = json.loads(p.stdout.strip().splitlines()[-1])
    assert d["config"] == bench.static_config("cfg0", 1)
    src = open(os.path.join(ROOT, "bench.py")).read()
    assert '"config": static_config(args.config, world)' in src  # the GPU arm
    if os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libmidbf_ref.so")):
        assert d["cpu_baseline"]["kind"] == "reference"
