"""Multi-process host logic of the sharded path, world_size 2 over gloo on
CPU: chunk-aligned shards tile the message exactly, the histogram
all-reduce equals the whole-message histogram, and the per-shard chunk
streams concatenate to the 1-GPU stream (chunk boundaries do not depend on
the GPU count). The oracle stands in for the device kernels here."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1402_3392_b200.dist import allreduce_counts, shard_for
from paper_1402_3392_b200.synth import synth_host

N_BYTES = 300_001
CHUNK = 16384


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shards_tile_message():
    for n in (0, 1, CHUNK, CHUNK + 1, N_BYTES, 10 * CHUNK):
        for world in (1, 2, 3, 4, 8):
            shards = [shard_for(n, r, world, CHUNK) for r in range(world)]
            assert shards[0].byte_lo == 0 and shards[-1].byte_hi == n
            for a, b in zip(shards, shards[1:]):
                assert a.byte_hi == b.byte_lo and a.chunk_hi == b.chunk_lo
            for s in shards:
                assert s.byte_lo % CHUNK == 0 or s.n_bytes == 0
            sizes = [s.n_chunks for s in shards]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_for(10, 2, 2)


def _worker(rank, world, port, out):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
    import oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    msg = synth_host(N_BYTES, 1.1, seed=5)
    sh = shard_for(N_BYTES, rank, world, CHUNK)
    local, _ = oracle.histogram(msg[sh.byte_lo:sh.byte_hi])
    counts = torch.from_numpy(local.view(np.int64).copy())
    allreduce_counts(counts)
    total = counts.numpy().view(np.uint64)
    alpha = int(np.nonzero(total)[0].max()) + 1
    freqs = oracle.quantize(total[:alpha], 12)
    f, cum, _ = oracle.table_views(freqs, 12)
    payload, offs, states = oracle.encode_chunks_u16(msg[sh.byte_lo:sh.byte_hi], CHUNK, f, cum,
                                                     12, 32)
    np.savez(out / f"rank{rank}.npz", total=total, freqs=np.asarray(freqs), payload=payload,
             offsets=offs, states=states)
    # the cross-rank framing step: global word base and the gathered stream
    from paper_1402_3392_b200.dist import gather_stream, global_word_base
    from paper_1402_3392_b200.rans import SymbolTable

    base, total_words = global_word_base(int(offs[-1]))
    cc = gather_stream(torch.from_numpy(payload.view(np.int16).copy()),
                       torch.from_numpy(offs.astype(np.int64)),
                       torch.from_numpy(states.reshape(-1).view(np.int32).copy()),
                       sh, N_BYTES, CHUNK, 32, SymbolTable(list(freqs), 12), dst=0)
    np.savez(out / f"frame{rank}.npz", base=base, total_words=total_words,
             container=np.frombuffer(cc.to_bytes(), np.uint8) if cc is not None
             else np.zeros(0, np.uint8))
    dist.destroy_process_group()


def test_gloo_world2_histogram_allreduce_and_shard_streams(tmp_path):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
    import oracle

    world = 2
    mp.spawn(_worker, args=(world, free_port(), tmp_path), nprocs=world, join=True)
    msg = synth_host(N_BYTES, 1.1, seed=5)
    full, alpha = oracle.histogram(msg)
    freqs = oracle.quantize(full[:alpha], 12)
    f, cum, _ = oracle.table_views(freqs, 12)
    payload, offs, states = oracle.encode_chunks_u16(msg, CHUNK, f, cum, 12, 32)
    parts = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    for p in parts:  # every rank built the identical global model
        assert np.array_equal(p["total"], full)
        assert p["freqs"].tolist() == freqs
    # concatenated shard streams == the single-GPU stream
    assert np.array_equal(np.concatenate([p["payload"] for p in parts]), payload)
    assert np.array_equal(np.concatenate([p["states"] for p in parts]), states)
    k0 = len(parts[0]["offsets"]) - 1
    assert np.array_equal(parts[0]["offsets"], offs[: k0 + 1])
    assert np.array_equal(parts[1]["offsets"] + offs[k0], offs[k0:])
    # gathered on rank 0: byte-identical to the single-GPU ICH1 stream
    from paper_1402_3392_b200.chunked import ChunkedContainer
    from paper_1402_3392_b200.rans import SymbolTable

    frames = [np.load(tmp_path / f"frame{r}.npz") for r in range(world)]
    assert [int(fr["base"]) for fr in frames] == [0, int(offs[k0])]
    assert all(int(fr["total_words"]) == int(offs[-1]) for fr in frames)
    single = ChunkedContainer(32, CHUNK, N_BYTES, SymbolTable(freqs, 12), states,
                              offs.astype(np.uint64), payload)
    assert frames[0]["container"].tobytes() == single.to_bytes()
    assert len(frames[1]["container"]) == 0
