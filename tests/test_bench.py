"""bench.py plumbing on CPU: the N-rank self-launch and the reference arm's
independence from the product library."""

from __future__ import annotations

import json
import os
import subprocess
import sys

from conftest import ROOT


def _json_line(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out
    return json.loads(lines[0])


def test_gpus_flag_launches_ranks():
    """`bench.py --gpus 2` outside torchrun spawns two ranks itself (VERDICT r1
    missing #4); the winner exchange over the process group picks np.argmax."""
    env = dict(os.environ, VMI_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--dist-selftest", "--poses", "1001"], capture_output=True, text=True,
                       env=env, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _json_line(r.stdout)
    assert d["n_gpus"] == 2 and d["index"] == d["want_index"]


def test_world_mismatch_fails_loudly():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4",
                        "--dist-selftest"], capture_output=True, text=True, env=env, timeout=120)
    assert r.returncode != 0 and "WORLD_SIZE" in (r.stderr + r.stdout)


def test_reference_arm_never_loads_the_product_library():
    """The reference arm times the oracle only: libvmi.so must stay unloaded
    (product pose matrices voided vs_reference)."""
    code = (
        "import sys; sys.argv=['bench.py','--impl','reference','--config','c1','--steps','1',"
        "'--warmup','0']; sys.path.insert(0, %r); import bench; bench.main();"
        "from paper_1709_06948_b200 import _lib; assert _lib._lib is None, 'libvmi loaded';"
        "maps=open('/proc/self/maps').read(); assert 'libvmi.so' not in maps; print('clean')"
    ) % ROOT
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    assert r.stdout.strip().endswith("clean")
    d = _json_line(r.stdout.rsplit("\n", 2)[0])
    assert d["impl"] == "reference" and d["cpu_baseline"]["kind"] == "port"
    assert d["cpu_baseline"]["host"]["numpy"]
