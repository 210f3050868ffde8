"""The reference's acceptance criteria 5 (the adaptive scheduler balances the
storage NICs, sign test over 20 seeds), 7 (model-execution bursts slowed
<= 2 % by KV traffic; the WRR floor) and 10 (online: dual-path TTFT no worse
than PE-only, arrival-rate gain >= 1.3x), restated in
tests/acceptance_criteria.cpp with the reference's scenarios, seeds and
thresholds (/root/reference/proj/tests/acceptance.cpp:274-331, :383-420,
:551-601),
compiled against this build's pdsim headers and libdualpath.so (CPU)."""

import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2602_21548_b200")


def test_acceptance_criteria_5_7_10(tmp_path):
    exe = str(tmp_path / "acceptance")
    subprocess.run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "acceptance_criteria.cpp"), "-L", LIBDIR, "-ldualpath",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True, capture_output=True, text=True)
    res = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    print(res.stdout)
    assert res.returncode == 0, res.stdout + res.stderr[-2000:]
    assert res.stdout.count("PASS") == 3
