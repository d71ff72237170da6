"""bench.py's multi-GPU launcher on a one-GPU box (-m gpu): `bench.py --gpus 2` without a launcher
re-runs itself under torch.distributed.run with two ranks; with --comm host both ranks share cuda:0
and exchange through the library's host-mediated communicator (gloo), so the launcher, the
drug-range sharding, the max-over-ranks timing and the data-parallel library path all run, and the
JSON line reports n_gpus = 2 ("never report a world size the caller did not ask for")."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _json_line(text):
    lines = [ln for ln in text.splitlines() if ln.startswith("{")]
    assert lines, text[-2000:]
    return json.loads(lines[-1])


@pytest.mark.parametrize("workload,exchange", [("C1", 2), ("C3", 0)])
def test_bench_gpus2_host_comm(workload, exchange):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--workload", workload, "--comm", "host",
           "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-gather-regime", "--exchange", str(exchange)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = _json_line(r.stdout)
    assert line["n_gpus"] == 2 and line["steps"] == 2 and line["warmup"] == 3
    assert line["value"] > 0 and line["config"]["comm"] == "host"
    assert line["runtime"]["exchange_used"] == ("u-reduce" if exchange == 2 else "S-allgather")
    assert line["runtime"]["collectives"] > 0
    assert line["gpu_launches"] > 0
