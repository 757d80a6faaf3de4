"""Multi-process sharded path with the DEVICE kernels: two ranks
each run the histogram kernel on their chunk-aligned shard, all-reduce the
256 x u64 counts (NCCL when two GPUs are visible, else gloo with both ranks
on cuda:0), quantize on the device, encode their chunks and gather the
shard streams onto rank 0. The gathered ICH1 stream must equal the 1-GPU
encode byte for byte and the all-reduced counts must equal np.bincount of
the whole message (reference cli.py:31-37). Also: ``bench.py --gpus 2``
launches two ranks itself and reports n_gpus = 2."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_1402_3392_b200 import _lib

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

N_BYTES = 9_000_011
CHUNK = 65536


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if _lib.device_count() == 0:
        pytest.fail("no CUDA device: the -m gpu suite must run on a B200")


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out, backend):
    import torch
    import torch.distributed as dist

    from paper_1402_3392_b200.dist import ShardedCodec
    from paper_1402_3392_b200.synth import synth_device

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = torch.device("cuda", rank % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    sc = ShardedCodec(N_BYTES, rank, world, CHUNK, 32, 12, device=dev)
    d = synth_device(sc.shard.n_bytes, 1.1, 77, first=sc.shard.byte_lo, device=dev)
    sc.build_global_model(d)
    sc.encode(d)
    back = torch.empty_like(d)
    sc.decode(back)
    torch.cuda.synchronize(dev)
    ok = bool(torch.equal(back[: sc.shard.n_bytes], d[: sc.shard.n_bytes]))
    cc = sc.gather(N_BYTES)
    np.savez(out / f"rank{rank}.npz", counts=sc.codec.counts.cpu().numpy().view(np.uint64),
             ok=ok, container=np.frombuffer(cc.to_bytes(), np.uint8) if cc is not None
             else np.zeros(0, np.uint8))
    dist.destroy_process_group()


def test_two_ranks_device_kernels_gather_equals_single_gpu(tmp_path):
    import torch
    import torch.multiprocessing as mp

    from paper_1402_3392_b200.chunked import encode_chunked
    from paper_1402_3392_b200.synth import synth_host

    backend = "nccl" if torch.cuda.device_count() >= 2 else "gloo"
    world = 2
    mp.spawn(_worker, args=(world, free_port(), tmp_path, backend), nprocs=world, join=True)
    msg = synth_host(N_BYTES, 1.1, 77)
    full = np.bincount(msg, minlength=256).astype(np.uint64)
    parts = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    for p in parts:
        assert bool(p["ok"])  # each rank decodes its own shard
        assert np.array_equal(p["counts"], full)  # all-reduced == whole-message bincount
    single = encode_chunked(msg, None, 32, CHUNK, 12).to_bytes()
    assert parts[0]["container"].tobytes() == single
    assert len(parts[1]["container"]) == 0


def test_bench_gpus_2_launches_two_ranks():
    import torch

    backend = "nccl" if torch.cuda.device_count() >= 2 else "gloo"
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "3",
                        "--warmup", "3", "--mib", "32", "--no-e2e", "--no-cpu",
                        "--dist-backend", backend],
                       capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2
    assert line["value"] > 0
    assert line["config"]["global_bytes"] == 2 * 32 * (1 << 20)


def test_bench_gpus_beyond_visible_is_an_error():
    import torch

    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    n = torch.cuda.device_count() + 1
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", str(n), "--steps", "3",
                        "--warmup", "3", "--mib", "16", "--no-e2e", "--no-cpu"],
                       capture_output=True, text=True, env=env, timeout=300, cwd=ROOT)
    assert r.returncode != 0
    assert "visible" in r.stderr
