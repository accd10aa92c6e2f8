"""Host-side rank plumbing for multi-process C3 worlds (one process per GPU,
torchrun): CUDA-IPC handle exchange, barriers and max-over-ranks timing.
Transport is torch.distributed over gloo (host objects only — no device data
moves through it; the collectives themselves run over NVLink in libc3cuda).
"""
import os


class Dist:
    """Rank plumbing (torch.distributed, gloo for host objects). Single
    process when WORLD_SIZE is unset."""

    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        if self.world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group("gloo", rank=self.rank, world_size=self.world)
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def allgather_bytes(self, blob):
        if not self.pg:
            return [blob]
        out = [None] * self.world
        self.pg.all_gather_object(out, blob)
        return out

    def max_list(self, values):
        """Elementwise max over ranks of a list of floats."""
        if not self.pg:
            return list(values)
        import torch
        t = torch.tensor(values, dtype=torch.float64)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return t.tolist()

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


def join_handles(blobs, blob_bytes):
    """Concatenate per-rank handle blobs in rank order (c3_session_import layout)."""
    for i, b in enumerate(blobs):
        if len(b) != blob_bytes:
            raise ValueError(f"rank {i}: handle blob is {len(b)} bytes, want {blob_bytes}")
    return b"".join(blobs)
