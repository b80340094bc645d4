"""bench.py --impl reference (the driver's reference arm) on the small shape c1:
it builds its inputs on the host, times the unmodified reference (numba, from
baseline/_ref when installed) and the C port, prints one JSON line, and never
loads the product library."""
import json
import subprocess
import sys

from conftest import REPO


def test_reference_arm_runs_without_the_product_library():
    out = subprocess.run([sys.executable, str(REPO / "bench.py"), "--impl", "reference",
                          "--shape", "c1", "--cpu-seconds", "1"], capture_output=True, text=True,
                         timeout=600, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "s" and line["value"] > 0
    assert line["product_library_loaded"] is False
    assert line["cpu_baseline"]["kind"] in ("reference", "port")
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["reference_port"]["value"] > 0
    assert len(line["config"]["inputs_digest"]) == 32
