"""Host-side logic of bench.py (CPU): the workloads, the link model, the
storage-balance metric and the reference arm's configuration."""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2602_21548_b200 as dp  # noqa: E402


class Args:
    sessions_per_gpu = 2
    workload = "c1"


def test_link_model():
    # one engine, or a box whose host links outrun the engines: the SM rate
    assert bench.link_per_engine(None, 4) == bench.PCIE_ZC_BPS
    assert bench.link_per_engine(55.6e9, 1) == bench.PCIE_ZC_BPS
    assert bench.link_per_engine(220e9, 4) == bench.PCIE_ZC_BPS
    # a shared host ceiling: its share per engine
    assert bench.link_per_engine(116e9, 4) == pytest.approx(29e9)


@pytest.mark.parametrize("wl,L,b", [("c1", 61, 576), ("c3", 64, 4096), ("c2", 61, 576)])
def test_workloads_and_cluster(wl, L, b):
    a = Args()
    a.workload = wl
    trajs, shape = bench.workload(a, 2)
    assert len(trajs) == 4 and shape["L"] == L and shape["b"] == b
    cfg = bench.cluster(shape, 1, 1, 0.0, None, 29e9)
    cfg.validate()
    assert cfg.node_storage_bandwidth() == pytest.approx(29e9)
    capped = bench.cluster(shape, 1, 1, 6.25e9)
    assert capped.node_storage_bandwidth() == pytest.approx(6.25e9)
    asym = bench.cluster(shape, 1, 1, 0.0, [6.25e9, 3.125e9])
    assert asym.node_storage_bandwidth(1) == pytest.approx(3.125e9)


def test_c1_is_the_baseline_generator():
    # BASELINE config 1: 20 turns, append 429, gen 500, ~95 % token-weighted hit
    a = Args()
    a.sessions_per_gpu = 64
    trajs, _ = bench.workload(a, 1)
    assert all(len(t.rounds) == 20 for t in trajs)
    hit = sum(dp.context_before(t, r) for t in trajs for r in range(len(t.rounds)))
    prompt = sum(dp.context_before(t, r) + t.rounds[r].append_tokens for t in trajs for r in range(len(t.rounds)))
    assert 0.94 < hit / prompt < 0.97


def test_storage_balance_metric():
    # two engines, one reads twice the other's bytes in every window
    spans = {0: [(0.0, 1.0, 2_000_000)], 1: [(0.0, 1.0, 1_000_000)]}
    res = bench.storage_balance(spans, None, 2, width=0.1, window=2)
    assert res["bytes_max_avg"] == pytest.approx(2 / 1.5, abs=1e-4)  # rounded to 4 places
    # normalised by caps 2:1 the utilisation is balanced
    res = bench.storage_balance(spans, [2.0, 1.0], 2, width=0.1, window=2)
    assert res["utilisation_max_avg"] == pytest.approx(1.0, abs=1e-4)
    assert bench.storage_balance({}, None, 2) is None


def test_trace_workload(tmp_path):
    p = str(tmp_path / "t.tsv")
    dp.save_trace(p, dp.synthesize(max_len=8000, count=7, seed=2))
    a = Args()
    a.trace, a.sessions_per_gpu = p, 2
    trajs, shape = bench.workload(a, 2)
    assert [t.id for t in trajs] == [t.id for t in dp.load_trace(p)[:4]]
    assert shape["L"] == 61


@pytest.mark.parametrize("wl", ["c1", "c2", "c3"])
def test_trace_stats_match_the_exec_plan(wl):
    """The config dict both arms print (requests, hit bytes, prompt tokens)
    is computed from the trace alone and equals the executor plan's."""
    a = Args()
    a.workload = wl
    a.sessions_per_gpu = 3
    trajs, shape = bench.workload(a, 1)
    stats = bench.trace_stats([[(r.append_tokens, r.gen_tokens) for r in t.rounds] for t in trajs], shape)
    cfg = bench.cluster(shape, 1, 1, 0.0)
    planned = dp.plan(cfg, trajs, policy="pe_only", **bench.PLAN_KW)
    xp = dp.build_exec_plan(cfg, trajs, planned, dp.ExecOptions())
    assert stats == (xp.requests, xp.hit_bytes, xp.prompt_tokens)


@pytest.mark.parametrize("wl", ["c1", "c2"])
def test_reference_trace_is_the_product_trace(tmp_path, wl):
    """The reference arm builds its trace with the reference's own generator
    (oracle/_ref): identical rounds to the product's synthesize."""
    from oracle import refpy
    if not refpy.ref_available():
        pytest.skip("oracle/_ref not built")
    a = Args()
    a.workload = wl
    a.trace = ""
    rounds = bench.reference_trace(a, wl, 5, str(tmp_path / "t.tsv"))
    trajs, _ = bench.workload(a, 1, sessions=5)
    assert rounds == [[(r.append_tokens, r.gen_tokens) for r in t.rounds] for t in trajs]


def test_reference_arm_loads_no_repo_library():
    """bench.py --impl reference times the CPU port on the same config and
    never loads the product (libdualpath.so / _core)."""
    import json
    import subprocess
    from oracle import refpy
    if not refpy.ref_available():
        pytest.skip("oracle/_ref not built")
    code = ("import sys, json; sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '0',"
            " '--sessions-per-gpu', '2']; import bench; a = bench.parse(); line = bench.reference_arm(a);"
            " maps = open('/proc/self/maps').read();"
            " print(json.dumps({'line': line, 'product': ('libdualpath' in maps) or ('_core.cpython' in maps)}))")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, check=True)
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["product"] is False
    line = res["line"]
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "port"
    assert line["config"]["sessions"] == 2 and line["config"]["requests"] == 40
    assert line["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] == 0


def _bench_fixtures():
    import glob
    return sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "bench_*.json")))


@pytest.mark.parametrize("path", _bench_fixtures(), ids=lambda p: os.path.basename(p)[6:-5])
def test_bench_plans_match_reference_fixtures(path):
    """Every configuration bench.py measures: the product planner's decisions
    (request -> PE, DE, read path) and makespan are the reference simulator's
    own, bit for bit (fixtures from oracle/_ref, tests/golden/make_golden.py)."""
    import json
    from paper_2602_21548_b200 import dist as dpdist
    with open(path) as f:
        want = json.load(f)
    a = Args()
    a.workload = want["workload"]
    a.trace = ""
    trajs, shape = bench.workload(a, 1, sessions=want["sessions"])
    cfg = bench.cluster(shape, want["P"], want["D"], want["cap_gbps"] * 1e9)
    planned = dp.plan(cfg, trajs, policy=want["policy"], **bench.PLAN_KW)
    assert bench.golden_key(want["workload"], want["sessions"], want["P"], want["D"], want["policy"],
                            want["cap_gbps"], bench.PCIE_ZC_BPS) == want["key"]
    assert len(planned["decisions"]) == want["decisions"]
    assert sum(1 for d in planned["decisions"] if d[4] == 1) == want["de_path"]
    assert dpdist.plan_digest(planned) == want["decisions_digest"]
    assert planned["makespan"] == want["makespan"]
