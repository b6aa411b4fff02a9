"""CPU tests of bench.py's multi-GPU launch path: `python bench.py --gpus N`
re-launches itself as N ranks under torch.distributed.run (127.0.0.1), every
rank takes its shard of the batch (no data-path collective; R:include/ternkit/
linalg.hpp:278-291 row partition), and rank 0 prints one line.  --dry-run
swaps NCCL for gloo and skips the kernels so the plumbing runs here."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args, env_extra=None, timeout=180):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=timeout, env=env, cwd=ROOT)


def _line(proc):
    lines = [ln for ln in proc.stdout.splitlines() if ln.startswith("{")]
    assert proc.returncode == 0, proc.stderr[-2000:]
    assert len(lines) == 1, proc.stdout  # rank 0 alone prints
    return json.loads(lines[0])


@pytest.mark.parametrize("gpus,workload,shards", [
    (2, "resnet50", [[0, 512], [512, 512]]),            # cfg5 strong scaling: 1024 split
    (2, "resnet18", [[0, 256], [256, 256]]),            # cfg4 weak scaling: 256 per GPU
    (4, "resnet50", [[0, 256], [256, 256], [512, 256], [768, 256]]),
])
def test_gpus_n_self_launches_n_ranks(gpus, workload, shards):
    d = _line(_bench("--gpus", str(gpus), "--dry-run", "--workload", workload))
    assert d["n_gpus"] == gpus and d["ranks"] == gpus
    assert d["shards"] == shards
    assert sum(c for _, c in d["shards"]) == d["global_batch"]


def test_world_size_mismatch_is_an_error():
    p = _bench("--gpus", "2", "--dry-run", env_extra={"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert p.returncode != 0 and "WORLD_SIZE=1" in (p.stderr + p.stdout)


def test_single_gpu_is_not_relaunched():
    d = _line(_bench("--gpus", "1", "--dry-run", "--workload", "resnet18"))
    assert d["n_gpus"] == 1 and d["shards"] == [[0, 256]]


def test_reference_arm_line():
    """--impl reference: the reference's own CPU code (oracle/_ref) on the
    workload, one JSON line with impl/value/unit/cpu_baseline/e2e (cfg2, the
    cheapest workload; needs the reference build, made by build())."""
    from oracle.oracle import reference_lib_path
    if reference_lib_path() is None:
        pytest.skip("oracle/_ref not built on this host")
    d = _line(_bench("--impl", "reference", "--workload", "conv", "--steps", "2", "--warmup", "1", timeout=600))
    assert d["impl"] == "reference" and d["unit"] == "Tops/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
