"""bench.py's reference arm (the CPU oracle port timed on host cores) runs without
a GPU and prints one well-formed JSON line; the GPU arm's contract keys are
checked on the GPU box by the driver."""

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_prints_contract_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config",
                          "cfg1", "--steps", "1", "--warmup", "0", "--ref-seconds", "0.05"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "cpu_baseline", "e2e", "config"):
        assert key in line
    assert line["value"] > 0 and line["cpu_baseline"]["kind"] == "port"
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    cb = line["cpu_baseline"]
    assert cb["host_dram_copy_gbs"] > 0 and cb["kv_read_gbs"] > 0
    assert abs(cb["frac_of_host_dram"] - cb["kv_read_gbs"] / cb["host_dram_copy_gbs"]) < 1e-9


def test_reference_arm_under_torchrun_prints_once():
    """Launched like the driver's N>1 run (torchrun, 2 ranks): rank 0 alone runs the
    CPU arm and prints one line; rank 1 exits 0 without output."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node=2", "--master-addr", "127.0.0.1", "--master-port",
                          str(port), str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--config", "cfg1", "--steps", "1", "--warmup", "0", "--ref-seconds", "0.05"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2
