"""bench.py's multi-rank launch (`--gpus N` must not silently time one GPU).

CPU: the torchrun command `python bench.py --gpus N` re-executes itself under (one rank per GPU, 127.0.0.1
rendezvous, the caller's flags passed through). GPU: `--gpus 2 --fabric` runs the N-rank path (two ranks on
one GPU through the in-process fabric) end to end and prints one line with n_gpus = 2."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_launch_command_is_torchrun_one_rank_per_gpu():
    sys.path.insert(0, ROOT)
    import bench
    cmd = bench.launch_cmd(["--gpus", "4", "--steps", "5", "--config", "c3"], 4, 29555)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--nnodes=1" in cmd
    assert "--master-addr=127.0.0.1" in cmd and "--master-port=29555" in cmd
    i = cmd.index(os.path.abspath(os.path.join(ROOT, "bench.py")))
    assert cmd[i + 1:] == ["--gpus", "4", "--steps", "5", "--config", "c3"]


def test_bench_self_launch_reaches_ranks_with_world_size(tmp_path):
    """The re-executed ranks see WORLD_SIZE / RANK (gloo stand-in for the rendezvous: a tiny script is
    launched through the same command builder)."""
    sys.path.insert(0, ROOT)
    import bench
    probe = tmp_path / "probe.py"
    probe.write_text("import os; print('RANK', os.environ['RANK'], 'WORLD', os.environ['WORLD_SIZE'])\n")
    cmd = bench.launch_cmd([], 2, 29556)
    cmd[cmd.index(os.path.abspath(os.path.join(ROOT, "bench.py")))] = str(probe)
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    ranks = sorted(line for line in out.stdout.splitlines() if line.startswith("RANK"))
    assert ranks == ["RANK 0 WORLD 2", "RANK 1 WORLD 2"]


@pytest.mark.gpu
def test_bench_two_ranks_on_the_fabric():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--fabric", "--config", "c1",
                          "--steps", "4", "--warmup", "3"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    line = lines[0]
    assert line["n_gpus"] == 2 and line["value"] > 0 and "fabric" in line
    assert all(r["world"] == 2 and r["collective_rows"] > 0 for r in line["ranks"])
    assert line["ranks"][0]["loss"] > 0.0
