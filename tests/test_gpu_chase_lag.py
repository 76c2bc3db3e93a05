"""The lag-2 wavefront chase (default) against the lag-3 one (PEVD_CHASE_LAG=3): both execute
exactly the sequential chase's operations, so d, e and every reflector must agree bit for bit,
and reruns must too (a race would show up as a differing or varying digest).  The schedule is
chosen once per process, hence the subprocesses."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [(40, 8), (300, 16), (1000, 32), (1001, 24), (4097, 32), (9000, 32), (20001, 8)]

SNIPPET = r"""
import json, sys
sys.path.insert(0, %r)
from tools.chase_lag_check import run
for n, b in %r:
    print(json.dumps(run(n, b, 3)), flush=True)
"""


def digests(lag):
    env = dict(os.environ, PEVD_CHASE_LAG=str(lag))
    out = subprocess.run([sys.executable, "-c", SNIPPET % (ROOT, CASES)], env=env, cwd=ROOT,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]


@pytest.mark.gpu
def test_lag2_chase_bitwise_equals_lag3():
    a, b = digests(3), digests(2)
    assert len(a) == len(b) == len(CASES)
    for x, y in zip(a, b):
        assert len(x["digests"]) == 1, x          # reruns identical
        assert x["digests"] == y["digests"], (x, y)
