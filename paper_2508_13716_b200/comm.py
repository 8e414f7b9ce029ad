"""Inter-device plumbing: barriers, the K7 gradient all-reduce, peer pointers.

One process per GPU.  ``SoloComm`` is the single-device case (all partitions
co-resident; "peer" reads are local HBM reads).  ``DistComm`` runs over an
initialised torch.distributed process group:

* peer buffers are exchanged as CUDA IPC handles (cudaIpcGetMemHandle +
  allocation offset) and opened in every process, so the K3 staging kernel
  pulls halo rows straight out of the owner's HBM over NVLink (one-sided,
  no NCCL on the data path);
* ``barrier()`` is stream-ordered: kernels queued after it on this rank's
  stream cannot start before every rank's preceding kernels (the owners'
  layer outputs) have completed -- no host sync.  By default it is a
  point-to-point flag exchange (``cg_flag_signal`` / ``cg_flag_wait``: each
  rank bumps its own IPC-mapped flag word with a stream write and its stream
  waits for every peer's word to reach the same generation; stream memory
  operations, no kernel, no collective).  CG_PEER_SYNC=nccl selects a
  1-element NCCL all-reduce instead; without CUDA (gloo on CPU) it is a host
  barrier;
* ``allreduce_`` is the K7 weight-gradient (+ loss) all-reduce.

The global cache tier is one POSIX shared-memory segment per node, mapped
and registered as pinned, portable, device-mapped memory in every rank.
"""

from __future__ import annotations

import ctypes as C
import os
import uuid

import numpy as np

from ._lib import call


class SoloComm:
    rank = 0
    world = 1

    def barrier(self) -> None:
        pass

    def host_barrier(self) -> None:
        pass

    def allreduce_(self, t) -> None:
        pass

    def exchange_pointers(self, local_ptr: int, device: int) -> list[int]:
        return [int(local_ptr)]

    def broadcast_obj(self, obj):
        return obj

    def close(self) -> None:
        pass


class DistComm:
    def __init__(self, device: int):
        import torch
        import torch.distributed as dist
        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.device = device
        self.backend = dist.get_backend()
        dev = torch.device("cuda", device) if self.backend == "nccl" else torch.device("cpu")
        self._flag = torch.zeros(1, dtype=torch.float32, device=dev)
        self._cuda = torch.cuda.is_available()
        self._opened: list[int] = []
        mode = os.environ.get("CG_PEER_SYNC", "flags")
        self.sync = ("flags" if self._cuda and mode == "flags" else
                     "nccl" if self.backend == "nccl" else "host")
        if self.sync == "flags":
            # one 32-bit generation counter per rank, read by every peer
            self._gen = 0
            self._word = torch.zeros(16, dtype=torch.int32, device=torch.device("cuda", device))
            ptrs = self.exchange_pointers(self._word.data_ptr(), device)
            self._words = np.array(ptrs, np.uint64)

    def barrier(self) -> None:
        if self.sync == "flags":
            import torch
            self._gen += 1
            st = torch.cuda.current_stream(self.device).cuda_stream
            call("cg_flag_signal", self._word.data_ptr(), self._gen, st)
            call("cg_flag_wait", self._words.ctypes.data, self.world, self.rank, self._gen, st)
        elif self.sync == "nccl":
            self.dist.all_reduce(self._flag)   # stream-ordered device barrier
        else:
            import torch
            if self._cuda:
                torch.cuda.current_stream().synchronize()
            self.dist.barrier()

    def host_barrier(self) -> None:
        self.dist.barrier()

    def allreduce_(self, t) -> None:
        if self.backend == "nccl":
            self.dist.all_reduce(t)
        elif not t.is_cuda:
            self.dist.all_reduce(t)
        else:
            import torch
            torch.cuda.current_stream().synchronize()
            h = t.cpu()
            self.dist.all_reduce(h)
            t.copy_(h)

    def broadcast_obj(self, obj):
        box = [obj]
        self.dist.broadcast_object_list(box, src=0)
        return box[0]

    def exchange_pointers(self, local_ptr: int, device: int) -> list[int]:
        handle = (C.c_uint8 * 64)()
        off = C.c_int64(0)
        call("cg_ipc_get_handle", local_ptr, C.addressof(handle), C.addressof(off))
        mine = (bytes(handle), off.value)
        allh = [None] * self.world
        self.dist.all_gather_object(allh, mine)
        ptrs = []
        for r, (h, o) in enumerate(allh):
            if r == self.rank:
                ptrs.append(int(local_ptr))
                continue
            buf = (C.c_uint8 * 64).from_buffer_copy(h)
            p = C.c_void_p()
            call("cg_ipc_open_handle", C.addressof(buf), device, C.addressof(p))
            self._opened.append(p.value)
            ptrs.append(p.value + o)
        return ptrs

    def close(self) -> None:
        for p in self._opened:
            try:
                call("cg_ipc_close_handle", p)
            except Exception:  # noqa: BLE001
                pass
        self._opened.clear()


class HostTier:
    """The global cache level: pinned, mapped host memory (zero-copy over UVA)."""

    def __init__(self, nbytes: int, comm=None):
        self.nbytes = max(int(nbytes), 16)
        self._shm = None
        self._registered = False
        if comm is None or comm.world == 1:
            p = C.c_void_p()
            call("cg_host_tier_alloc", self.nbytes, C.addressof(p))
            self.ptr = p.value
            self._owned = True
            return
        from multiprocessing import shared_memory
        name = comm.broadcast_obj(f"capgnn_{uuid.uuid4().hex[:12]}" if comm.rank == 0 else None)
        if comm.rank == 0:
            self._shm = shared_memory.SharedMemory(name=name, create=True, size=self.nbytes)
        comm.host_barrier()
        if comm.rank != 0:
            self._shm = shared_memory.SharedMemory(name=name, create=False)
        buf = np.frombuffer(self._shm.buf, dtype=np.uint8)
        self.ptr = buf.ctypes.data
        self._keep = buf
        call("cg_host_tier_register", self.ptr, self.nbytes)
        self._registered = True
        self._owned = False
        self._rank = comm.rank
        comm.host_barrier()

    def close(self) -> None:
        if self.ptr is None:
            return
        if self._owned:
            call("cg_host_tier_free", self.ptr)
        else:
            if self._registered:
                call("cg_host_tier_unregister", self.ptr)
            del self._keep
            self._shm.close()
            if self._rank == 0:
                try:
                    self._shm.unlink()
                except FileNotFoundError:
                    pass
        self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def local_rank_device() -> int:
    return int(os.environ.get("LOCAL_RANK", "0"))
