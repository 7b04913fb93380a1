"""bench.py driver contract on CPU: the multi-GPU launcher and the
reference arm's JSON line (same config object as our arm's)."""

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def _env():
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    return env


def test_gpus_n_relaunches_under_torchrun():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "4", "--steps", "7", "--print-launcher"],
                         capture_output=True, text=True, env=_env(), timeout=120, check=True).stdout
    cmd = json.loads(out.strip().splitlines()[-1])["launcher"]
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-4:] == ["--gpus", "4", "--steps", "7"] and cmd[-5].endswith("bench.py")


def test_reference_arm_under_the_launcher():
    """--gpus 2 outside torchrun: two ranks start, rank 0 alone prints the
    reference arm's line with n_gpus 2 and the full config block."""
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2", "--config",
                        "c1", "--steps", "1", "--warmup", "0"], capture_output=True, text=True, env=_env(),
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    line = lines[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    sys.path.insert(0, str(ROOT))
    import bench
    assert line["config"] == bench.config_block("c1", "csr", 64 ** 3, 190 ** 3, 2)
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
