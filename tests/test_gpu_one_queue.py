"""The executor's ACTUAL enqueues under the worst case the deadlock model
assumes (tests/test_enqueue_model.py): every stream of a device on ONE
hardware queue.  CUDA_DEVICE_MAX_CONNECTIONS=1 makes the driver multiplex
all streams of a device onto a single channel, so a cross-stream wait (event
or spin kernel) enqueued in front of its producer would hang the device.
The pipelines run in a subprocess with that setting (it only takes effect
before CUDA initialises) on two GPUs -- one engine per device, as in
production -- under a timeout; they must finish and verify their pools.
This checks the runtime's real enqueue order, not a restatement of it."""

import os
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
sys.path.insert(0, {root!r})
sys.path.insert(0, {tests!r})
import paper_2602_21548_b200 as dp
from test_gpu_engine import cluster, small_trace, handoff_engines, verify_prompt_pool, STORAGE_BOUND
cfg = cluster(1, 1, L=4)
trajs = small_trace(count=8, turns=5, seed=6)
planned = dp.plan(cfg, trajs, policy="dual_path", **STORAGE_BOUND)
opt = dp.ExecOptions()
opt.seed = 9
opt.handoff = True
opt.prefill = {prefill}
opt.persist = {persist}
opt.handoff_layerwise = {layerwise}
opt.compute_quota = 5e-4
opt.prefill_cost = (2e-10, 1e-9, 4e-7, 1e-5)
opt.k1_mode, opt.k2_mode, opt.k3_mode = {k1}, {k2}, {k3}
opt.wait_timeout_ms = 20000
xp = dp.build_exec_plan(cfg, trajs, planned, opt)
opt.pool_slots, opt.de_pool_slots = xp.peak_slots, xp.de_peak_slots   # tight: slot reuse waits
xp = dp.build_exec_plan(cfg, trajs, planned, opt)
rts = handoff_engines(xp, 2, [0, 1])
for _ in range(2):
    for rt in rts:
        rt.reset_counters()
    res = dp.run_step_all(rts)
    assert sum(r.bytes_read for r in res) == xp.hit_bytes
assert verify_prompt_pool(rts[0], xp, cfg) > 0
print("ok")
"""


@pytest.mark.parametrize("prefill,persist,layerwise,k1,k2,k3", [
    (False, False, False, 0, 0, 0), (False, True, False, 3, 2, 1),
    (True, False, False, 0, 0, 1), (True, True, False, 3, 2, 1), (True, False, True, 0, 0, 0),
    (True, False, True, 3, 2, 1)])  # layerwise copy-engine K3: stream waits on the forward rows
def test_pipeline_on_one_hardware_queue_per_device(two_gpus, prefill, persist, layerwise, k1, k2, k3):
    env = dict(os.environ, CUDA_DEVICE_MAX_CONNECTIONS="1", CUDA_VISIBLE_DEVICES=os.environ.get(
        "CUDA_VISIBLE_DEVICES", "0,1"))
    code = SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"), prefill=prefill, persist=persist,
                         layerwise=layerwise, k1=k1, k2=k2, k3=k3)
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=240)
    assert p.returncode == 0 and p.stdout.strip().endswith("ok"), p.stdout[-2000:] + p.stderr[-4000:]
