"""Every libffs path on small shapes through the bounds-checked build (libffs_checked.so,
-DFFS_CHECKED: device-side checks of every data-derived index, trap on failure) -- the substitute
for compute-sanitizer, which is closed on this GPU pool (profiles/r02/compute_sanitizer_closed.log).
Runs tools/san_run.py in a subprocess with FFS_LIBRARY=checked and requires a clean exit and
oracle-identical results."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("graph", ["1", "0"])
def test_checked_build_runs_every_path(graph):
    from paper_2109_07358_b200 import build
    build.build(checked=True)
    env = dict(os.environ, FFS_LIBRARY="checked", SAN_GRAPH=graph)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "san_run.py")], env=env, capture_output=True,
                       text=True, timeout=900)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0, r.stderr[-2000:]
    assert "FFS_CHECK failed" not in r.stdout + r.stderr
    lines = [l for l in r.stdout.splitlines() if "differing" in l]
    assert len(lines) >= 10 and all(" 0 differing" in l or ": 0 differing" in l for l in lines), lines
    assert "observables ok: True" in r.stdout
