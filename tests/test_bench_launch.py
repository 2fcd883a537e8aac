"""bench.py's N-GPU entry point (`--gpus N` must start N ranks itself).

`python bench.py --gpus 2` outside torchrun re-launches itself under
torch.distributed.run with two ranks on 127.0.0.1, as the driver does; the
SISPH_BENCH_RANKFILE hook makes every rank record `rank/world` and the
DRYRUN hook stops it there (no GPU here)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gpus_2_starts_two_ranks(tmp_path):
    rf = tmp_path / "ranks.txt"
    env = dict(os.environ, SISPH_BENCH_RANKFILE=str(rf), SISPH_BENCH_DRYRUN="1")
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1",
                        "--warmup", "0"], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert sorted(rf.read_text().split()) == ["0/2", "1/2"]


def test_gpus_mismatch_with_world_size_fails_loudly(tmp_path):
    env = dict(os.environ, WORLD_SIZE="3", RANK="0", SISPH_BENCH_DRYRUN="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0 and "WORLD_SIZE=3" in r.stderr
