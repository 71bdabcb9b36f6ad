"""Frame sharding across ranks: frames are independent, so each
rank runs its own pipeline over its own contiguous frame range and the data
path has no collective.  torch.distributed is used only to align the timed
region (barrier) and to take the slowest rank's time.
"""
from __future__ import annotations


def shard(rank: int, world: int, per_rank: int) -> range:
    """Weak scaling: rank r processes frames [r*per_rank, (r+1)*per_rank)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    return range(rank * per_rank, (rank + 1) * per_rank)


def split(n: int, rank: int, world: int) -> range:
    """Strong scaling: a fixed batch of n frames split into contiguous shards
    whose sizes differ by at most one."""
    base, rem = divmod(n, world)
    start = rank * base + min(rank, rem)
    return range(start, start + base + (1 if rank < rem else 0))


def max_over_ranks(values, device=None):
    """Element-wise max of a list of floats over all ranks (identity when not
    distributed)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


class HostGather:
    """The batch's results in ONE host buffer shared by the ranks of a node
    ("results are gathered to the host", no collective).

    Rank 0 creates a file in /dev/shm sized for the whole batch; every rank
    maps it and copies its own contiguous shard's results (device-to-host)
    straight into its slice, so after a barrier rank 0 holds the batch's
    results in frame order.  With CUDA the mapping is page-locked
    (cudaHostRegister), so those copies are asynchronous DMA like any
    pinned-buffer copy.  `rows` is this rank's range of the leading axis.
    """

    def __init__(self, tag: str, shape, dtype, rows: range, rank: int, barrier, pin: bool = True,
                 single_process: bool = False):
        import mmap
        import os

        import numpy as np

        self.rank = rank
        self.shape, self.dtype = tuple(int(s) for s in shape), np.dtype(dtype)
        self.nbytes = int(np.prod(self.shape, dtype=np.int64)) * self.dtype.itemsize
        self.path = f"/dev/shm/hogb200_{tag}"
        if single_process:
            self.path = None  # one process: a private page-locked mapping is the same gather
        if rank == 0 and self.path:
            with open(self.path, "wb") as f:
                f.truncate(max(self.nbytes, 1))
        barrier()
        if self.path:
            fd = os.open(self.path, os.O_RDWR)
            try:
                self._mm = mmap.mmap(fd, max(self.nbytes, 1), mmap.MAP_SHARED,
                                     mmap.PROT_READ | mmap.PROT_WRITE)
            finally:
                os.close(fd)
        else:
            self._mm = mmap.mmap(-1, max(self.nbytes, 1))
        self.array = np.frombuffer(self._mm, dtype=self.dtype,
                                   count=int(np.prod(self.shape, dtype=np.int64))).reshape(self.shape)
        self.rows = rows
        self._registered = False
        self._barrier = barrier
        if pin:
            import torch

            if torch.cuda.is_available() and self.nbytes:
                ptr = self.array.ctypes.data
                err = torch.cuda.cudart().cudaHostRegister(ptr, self.nbytes, 0)
                if int(err) != 0:
                    raise RuntimeError(f"cudaHostRegister failed ({err})")
                self._registered = True
        import torch

        self.tensor = torch.from_numpy(self.array)  # whole batch (host)

    def local(self):
        """This rank's slice (a host tensor view of the shared buffer)."""
        return self.tensor[self.rows.start: self.rows.stop]

    def close(self):
        """Unpin and unmap; rank 0 removes the file after every rank is done."""
        import os

        if self._registered:
            import torch

            torch.cuda.cudart().cudaHostUnregister(self.array.ctypes.data)
            self._registered = False
        del self.tensor, self.array
        try:
            self._mm.close()
        except BufferError:  # views still held by the caller: unmapped when they go
            pass
        self._barrier()
        if self.rank == 0 and self.path:
            try:
                os.unlink(self.path)
            except FileNotFoundError:
                pass
