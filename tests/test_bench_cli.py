"""bench.py's multi-GPU entry: `--gpus N` re-launches itself as N ranks under
torch.distributed.run, and refuses loudly (non-zero exit, no JSON line) when
the node has fewer than N GPUs -- it never falls back to one GPU."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gpus_more_than_present_fails_loudly():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode != 0
    assert "refusing to run" in r.stderr and "--gpus 2" in r.stderr
    assert r.stdout.strip() == ""


def test_world_size_mismatch_fails():
    env = dict(os.environ, WORLD_SIZE="4", RANK="0", LOCAL_RANK="0", CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode != 0 and "WORLD_SIZE=4" in r.stderr
