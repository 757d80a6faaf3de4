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


def global_word_base(local_words: int, group=None) -> tuple[int, int]:
    """(first global word of this rank's payload, total words of the stream):
    an exclusive prefix over ranks of the per-rank payload sizes -- one
    all-gather of one int64 per rank. Adding the base to a shard's local word
    offsets gives its chunks' offsets in the whole message's stream."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return 0, int(local_words)
    dev = torch.device("cuda", torch.cuda.current_device()) \
        if dist.get_backend(group) == "nccl" else torch.device("cpu")
    world = dist.get_world_size(group)
    mine = torch.tensor([int(local_words)], dtype=torch.int64, device=dev)
    sizes = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(sizes, mine, group=group)
    sizes = [int(t.item()) for t in sizes]
    rank = dist.get_rank(group)
    return sum(sizes[:rank]), sum(sizes)


def gather_stream(payload, offsets, states, shard: Shard, n_total: int, chunk_len: int,
                  lane_count: int, table, dst: int = 0, group=None):
    """Assemble the whole message's chunked stream (an ICH1
    ChunkedContainer) on rank ``dst`` from every rank's shard stream, given
    as torch tensors on the backend's device: ``payload`` (16-bit words),
    ``offsets`` (the shard's local word offsets, n_chunks + 1) and
    ``states`` (n_chunks x N). One all-gather of the sizes, then padded
    all-gathers of payloads, offsets and states. Returns the container on
    ``dst`` and None elsewhere. Chunk boundaries never depend on the rank
    count, so the result is byte-identical to a single-GPU encode."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from .chunked import ChunkedContainer

    single = not (dist.is_available() and dist.is_initialized())
    world = 1 if single else dist.get_world_size(group)
    rank = 0 if single else dist.get_rank(group)
    dev = payload.device
    k = shard.n_chunks
    if world == 1:
        words = int(offsets[k].item()) if k else 0
        return ChunkedContainer(
            lane_count, chunk_len, n_total, table,
            states.reshape(-1)[: k * lane_count].cpu().numpy().view(np.uint32)
            .reshape(-1, lane_count),
            offsets[: k + 1].cpu().numpy().astype(np.uint64),
            payload[:words].cpu().numpy().view(np.uint16).copy())
    words = int(offsets[k].item()) if k else 0
    meta = torch.tensor([words, k], dtype=torch.int64, device=dev)
    metas = [torch.zeros(2, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(metas, meta, group=group)
    metas = [(int(m[0].item()), int(m[1].item())) for m in metas]
    wmax = max(1, max(w for w, _ in metas))
    kmax = max(c for _, c in metas)

    def padded(t, size, dtype):
        out = torch.zeros(max(1, size), dtype=dtype, device=dev)
        if t.numel():
            out[: t.numel()] = t.reshape(-1).view(dtype)
        return out

    # payload words travel as int32 pairs (gloo has no 16-bit collectives)
    pay16 = padded(payload[:words], wmax + (wmax & 1), torch.int16)
    bufs = (pay16.view(torch.int32),
            padded(offsets[: k + 1], kmax + 1, torch.int64),
            padded(states.reshape(-1)[: k * lane_count], kmax * lane_count, torch.int32))
    gathered = []
    for b in bufs:
        parts = [torch.empty_like(b) for _ in range(world)]
        dist.all_gather(parts, b, group=group)
        gathered.append(parts)
    if rank != dst:
        return None
    pays, offs, sts = gathered
    payload_all = np.concatenate(
        [p.cpu().numpy().view(np.uint16)[:w] for p, (w, _) in zip(pays, metas)])
    states_all = np.concatenate(
        [s[: c * lane_count].cpu().numpy().view(np.uint32) for s, (_, c) in zip(sts, metas)])
    offsets_all = [np.zeros(1, dtype=np.uint64)]
    base = 0
    for o, (w, c) in zip(offs, metas):
        offsets_all.append(o[1: c + 1].cpu().numpy().astype(np.uint64) + np.uint64(base))
        base += w
    return ChunkedContainer(lane_count, chunk_len, n_total, table,
                            states_all.reshape(-1, lane_count), np.concatenate(offsets_all),
                            payload_all)


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

    def gather(self, n_total: int, dst: int = 0):
        """The whole message's ICH1 stream on rank ``dst`` (after encode with
        framing): every rank's shard payload, offsets and states gathered
        over the process group (NVLink for NCCL)."""
        c = self.codec
        k = self.shard.n_chunks
        return gather_stream(c.payload, c.offsets[: k + 1], c.states[: k * c.lane_count],
                             self.shard, n_total, c.chunk_len, c.lane_count, c.read_table(),
                             dst, self.group)
