"""Multi-GPU sharding: one process per GPU, chunk-aligned contiguous shards.

SURVEY 8e. Chunk boundaries depend only on the chunk length, so the encoded
stream is identical for 1, 2, 4 or 8 GPUs: rank r owns chunks
[k0, k1) = an even split of ceil(n / C) chunks and encodes them with the
GLOBAL model. The only exchange on the path is one all-reduce (sum) of the
256 x u64 byte histogram (2 KiB; NCCL over NVLink when the tensor is on a
GPU, gloo for the CPU tests) before the replicated, deterministic quantize;
decode needs no communication at all.
"""

from __future__ import annotations

from dataclasses import dataclass

from .chunked import DEFAULT_CHUNK, n_chunks_for


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    chunk_lo: int   # first chunk index owned
    chunk_hi: int   # one past the last chunk owned
    byte_lo: int    # message byte range [byte_lo, byte_hi)
    byte_hi: int

    @property
    def n_bytes(self) -> int:
        return self.byte_hi - self.byte_lo

    @property
    def n_chunks(self) -> int:
        return self.chunk_hi - self.chunk_lo


def shard_for(n: int, rank: int, world: int, chunk_len: int = DEFAULT_CHUNK) -> Shard:
    """Contiguous, chunk-aligned shard of an n-byte message for `rank`.
    Chunks are split as evenly as possible (the first n_chunks % world ranks
    get one extra)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    k = n_chunks_for(n, chunk_len)
    per, extra = divmod(k, world)
    lo = rank * per + min(rank, extra)
    hi = lo + per + (1 if rank < extra else 0)
    return Shard(rank, world, lo, hi, min(n, lo * chunk_len), min(n, hi * chunk_len))


def allreduce_counts(counts, group=None) -> None:
    """In-place SUM of the 256-bin histogram across ranks (int64 tensor; the
    device kernels write u64, and two's-complement addition is identical)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)


class ShardedCodec:
    """One rank's part of a multi-GPU chunked encode / decode.

    build_global_model(): local histogram of this rank's shard ->
    all-reduce -> quantize + tables (identical on every rank).
    encode()/decode(): purely local over the shard's chunks.
    """

    def __init__(self, n_total: int, rank: int, world: int, chunk_len: int = DEFAULT_CHUNK,
                 lane_count: int = 32, scale_bits: int = 14, device=None, group=None):
        from .chunked import DeviceCodec

        self.shard = shard_for(n_total, rank, world, chunk_len)
        self.group = group
        self.codec = DeviceCodec(max(16, self.shard.n_bytes), chunk_len, lane_count,
                                 scale_bits, device)

    def build_global_model(self, d_shard):
        self.codec.histogram(d_shard, self.shard.n_bytes)
        allreduce_counts(self.codec.counts, self.group)
        self.codec.build_table_from_counts()

    def encode(self, d_shard, frame: bool = True):
        self.codec.encode(d_shard, self.shard.n_bytes, frame)

    def decode(self, d_out, payload=None, offsets=None, states=None):
        self.codec.decode(d_out, self.shard.n_bytes, payload, offsets, states)
