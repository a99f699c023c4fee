"""Host side of the λPipe multicast engine (wraps ``lp_mc_*`` of the C ABI).

:class:`MulticastEngine` owns one ``lp_mc`` handle: the block table of a
packed image, a node table (device-visible image + signal area per node) and a
compiled schedule.  :class:`Cluster` is the set of node images one process
can address:

* ``Cluster.local(...)``   — every node's image on ONE GPU, executed by one
  kernel launch (test / single-GPU emulation; the guide's rule for fewer GPUs
  than ranks);
* ``Cluster.distributed(...)`` — one process per GPU under torchrun; images
  are exchanged as CUDA-IPC handles so each rank pushes straight into its
  peers' HBM over NVLink;
* an optional HOST node: pinned (page-locked, device-mapped) host memory that
  receivers pull from over PCIe (config C3).  In the distributed case it lives
  in a POSIX shared-memory segment that every rank maps and registers.
"""

from __future__ import annotations

import contextlib
import ctypes as C
import mmap
import os
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .errors import InvalidArgumentError, NativeError
from .image import fill_args

LP_NODE_GPU, LP_NODE_HOST = 0, 1
DEFAULT_TILE = 512 * 1024


class _CudaArray:
    """Minimal ``__cuda_array_interface__`` view of a raw device pointer."""

    def __init__(self, ptr: int, shape: tuple, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def device_view(ptr: int, nbytes: int, device: int, dtype=None, shape=None):
    """A torch tensor aliasing ``nbytes`` of device memory at ``ptr`` (no copy)."""
    import torch
    dtype = dtype or torch.uint8
    base = torch.int16 if dtype == torch.bfloat16 else dtype
    typestr = {torch.uint8: "|u1", torch.int16: "<i2", torch.float16: "<f2", torch.float32: "<f4",
               torch.int32: "<i4", torch.int64: "<i8"}[base]
    n = nbytes // torch.empty((), dtype=base).element_size()
    with torch.cuda.device(device):
        t = torch.as_tensor(_CudaArray(ptr, (n,), typestr), device=f"cuda:{device}")
    if dtype == torch.bfloat16:
        t = t.view(torch.bfloat16)
    return t.view(shape) if shape is not None else t


# copy-engine streams per node for the hybrid executor's pinned-host DMA (its
# blocks alternate between them); LP_HOST_DMA_STREAMS overrides
HOST_DMA_STREAMS = int(os.environ.get("LP_HOST_DMA_STREAMS", "1"))


class MulticastEngine:
    """One compiled λPipe multicast over a fixed block table."""

    def __init__(self, n_nodes: int, block_offsets, block_lengths, tile_bytes=DEFAULT_TILE):
        """``tile_bytes``: one size, or one per block (lp_mc_create_tiled)."""
        lib = N.lib()
        self.n_nodes = n_nodes
        self.n_blocks = len(block_offsets)
        self.block_offsets = list(block_offsets)
        self.block_lengths = list(block_lengths)
        self.tile_bytes = tile_bytes
        h = C.c_void_p()
        if isinstance(tile_bytes, (list, tuple)):
            if len(tile_bytes) != self.n_blocks:
                raise ValueError("one tile size per block")
            N.check(lib.lp_mc_create_tiled(C.byref(h), n_nodes, self.n_blocks, N.i64_array(block_offsets),
                                           N.i64_array(block_lengths), N.i64_array(tile_bytes)),
                    "lp_mc_create_tiled")
        else:
            N.check(lib.lp_mc_create(C.byref(h), n_nodes, self.n_blocks, N.i64_array(block_offsets),
                                     N.i64_array(block_lengths), tile_bytes), "lp_mc_create")
        self._h = h
        sb = C.c_int64()
        N.check(lib.lp_mc_signal_bytes(h, C.byref(sb)), "lp_mc_signal_bytes")
        self.signal_bytes = sb.value

    def close(self):
        if self._h:
            N.lib().lp_mc_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

    def set_node(self, node: int, kind: int, image: int, signals: int = 0, ready: int = 0):
        N.call("lp_mc_set_node", self._h, node, kind, C.c_void_p(image), C.c_void_p(signals or None),
               C.c_void_p(ready or None))

    def set_schedule(self, rows, sources):
        self._rows = [tuple(int(v) for v in r) for r in rows]
        flat = [int(v) for r in rows for v in r]
        arr = N.i32_array(flat) if flat else (C.c_int32 * 1)()
        N.call("lp_mc_set_schedule", self._h, arr, len(rows), N.i32_array(list(sources)), len(sources))

    def configure(self, direction: int = 1, push_mode: int = 1, pull_mode: int = 1, chunk_bytes: int = 16384,
                  window: int = 3):
        """direction 0 = senders push, 1 = receivers pull; copy engine per role:
        0 = LDG/STG vectors, 1 = TMA bulk pipeline; window = ops an LDG CTA may interleave."""
        N.call("lp_mc_configure", self._h, direction, push_mode, pull_mode, chunk_bytes, window)
        self.cfg = (direction, push_mode, pull_mode, chunk_bytes, window)

    def set_option(self, name: str, value: int):
        N.call("lp_mc_set_option", self._h, name.encode(), int(value))

    def reset_signals(self, node: int, stream: int = 0):
        N.call("lp_mc_reset_signals", self._h, node, C.c_void_p(stream or None))

    def run(self, exec_nodes, epoch: int, push_ctas: int, pull_ctas: int, stream: int = 0):
        N.call("lp_mc_run", self._h, N.i32_array(list(exec_nodes)), len(exec_nodes), epoch,
               push_ctas, pull_ctas, C.c_void_p(stream or None))

    def run_ce(self, node: int, epoch: int, streams: list, block_events: list | None = None):
        """Enqueue ``node``'s receives on copy engines (see lp_mc_run_ce)."""
        arr = (C.c_void_p * len(streams))(*[int(x) for x in streams])
        evs = None
        if block_events is not None:
            evs = (C.c_void_p * self.n_blocks)(*[int(e) if e else None for e in block_events])
        N.call("lp_mc_run_ce", self._h, node, epoch, len(streams), arr, evs)

    def run_host_dma(self, node: int, epoch: int, streams: list, block_events: list | None = None):
        """Enqueue ``node``'s HOST-sourced receives on copy engines (hybrid
        executor, option host_dma = 1; see lp_mc_run_host_dma)."""
        arr = (C.c_void_p * len(streams))(*[int(x) for x in streams])
        evs = None
        if block_events is not None:
            evs = (C.c_void_p * self.n_blocks)(*[int(e) if e else None for e in block_events])
        N.call("lp_mc_run_host_dma", self._h, node, epoch, len(streams), arr, evs)

    def landing_events(self, node: int, epoch: int, stream: int, block_events: list):
        """Record block_events[b] on ``stream`` once ``node`` holds block b
        (waits on the node's own counters; see lp_mc_landing_events)."""
        evs = (C.c_void_p * self.n_blocks)(*[int(e) if e else None for e in block_events])
        N.call("lp_mc_landing_events", self._h, node, epoch, C.c_void_p(stream), evs)

    def received_blocks(self, node: int) -> list:
        """Blocks ``node`` receives under the current schedule, in step order."""
        return [r[3] for r in sorted(getattr(self, "_rows", [])) if r[2] == node]

    def verify(self, node: int, epoch: int, sums_ptr: int, stream: int = 0, ctas: int = 32):
        """Checksum ``node``'s received blocks as they land (lp_mc_verify)
        into ``n_blocks`` uint64 at device pointer ``sums_ptr``: enqueue it
        after the run's producers; ``stream`` parks in stream-ordered waits on
        the node's block counters and launches one checksum kernel per block."""
        N.call("lp_mc_verify", self._h, node, epoch, ctas, C.c_void_p(sums_ptr), C.c_void_p(stream or None))

    def node_ops(self, node: int) -> tuple:
        """(in-kernel ops, host-DMA ops) ``node`` executes."""
        k, d = C.c_int(), C.c_int()
        N.call("lp_mc_node_ops", self._h, node, C.byref(k), C.byref(d))
        return k.value, d.value

    def status(self, stream: int = 0) -> None:
        code = C.c_int()
        N.call("lp_mc_status", self._h, C.c_void_p(stream or None), C.byref(code))

    def arrivals_ns(self, node: int) -> list:
        out = (C.c_uint64 * self.n_blocks)()
        N.call("lp_mc_arrivals", self._h, node, out)
        return list(out)

    def complete(self, node: int, epoch: int) -> list:
        out = (C.c_int32 * self.n_blocks)()
        N.call("lp_mc_block_complete", self._h, node, epoch, out)
        return [bool(x) for x in out]


def schedule_rows(schedule) -> list:
    """(step, sender, receiver, block) rows of a MulticastSchedule or its lines."""
    if isinstance(schedule, (list, tuple)) and schedule and isinstance(schedule[0], str):
        return [tuple(int(x) for x in ln.split(",")) for ln in schedule]
    return [(t.step, t.sender, t.receiver, t.block_id) for row in schedule.steps for t in row]


@dataclass
class NodeBuffer:
    node: int
    kind: int
    device: int              # CUDA device holding it (-1 for host)
    image: int               # device-visible pointer in this process
    signals: int = 0
    owned: list = field(default_factory=list)   # (kind, ptr) to free


class HostImage:
    """Page-locked, device-mapped host copy of a packed image (a HOST node).

    ``shm_name`` backs it with a POSIX shared-memory file so every rank of a
    torchrun job maps the same pages (``/dev/shm``); otherwise anonymous.
    """

    def __init__(self, nbytes: int, shm_name: str | None = None, create: bool = True):
        self.nbytes = nbytes
        self.shm_path = None
        if shm_name:
            self.shm_path = f"/dev/shm/{shm_name}"
            flags = os.O_RDWR | (os.O_CREAT if create else 0)
            fd = os.open(self.shm_path, flags, 0o600)
            if create:
                os.ftruncate(fd, nbytes)
            self._mm = mmap.mmap(fd, nbytes, mmap.MAP_SHARED, mmap.PROT_READ | mmap.PROT_WRITE)
            os.close(fd)
        else:
            self._mm = mmap.mmap(-1, nbytes, mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS,
                                 mmap.PROT_READ | mmap.PROT_WRITE)
        self.array = np.frombuffer(self._mm, dtype=np.uint8)
        self.host_ptr = self.array.ctypes.data
        alias = C.c_void_p()
        N.call("lp_host_register", C.c_void_p(self.host_ptr), nbytes, C.byref(alias))
        self.device_ptr = alias.value

    def close(self, unlink: bool = False):
        if self.device_ptr:
            N.lib().lp_host_unregister(C.c_void_p(self.host_ptr))
            self.device_ptr = 0
        self.array = None
        try:
            self._mm.close()
        except BufferError:
            pass
        if unlink and self.shm_path and os.path.exists(self.shm_path):
            os.unlink(self.shm_path)


@contextlib.contextmanager
def on_device(device: int):
    """Make ``device`` current for the calls inside (the library shares the
    CUDA runtime with torch, so this is torch's device context)."""
    import torch
    with torch.cuda.device(device):
        yield


def dev_malloc(device: int, nbytes: int) -> int:
    p = C.c_void_p()
    N.call("lp_malloc", device, nbytes, C.byref(p))
    return p.value


def dev_free(device: int, ptr: int):
    N.call("lp_free", device, C.c_void_p(ptr))


def ipc_handle(ptr: int) -> bytes:
    buf = (C.c_char * 64)()
    N.call("lp_ipc_get", C.c_void_p(ptr), buf)
    return bytes(buf)


def ipc_open(device: int, handle: bytes) -> int:
    p = C.c_void_p()
    buf = (C.c_char * 64).from_buffer_copy(handle)
    N.call("lp_ipc_open", device, buf, C.byref(p))
    return p.value


def fill_image(device_ptr: int, layout, seed: int, stream: int = 0):
    """Write the synthetic weights of ``layout`` into an image on the device."""
    off, numel, kind, sexp, _ = fill_args(layout)
    n = len(off)
    N.call("lp_fill_tensors", C.c_void_p(device_ptr), n, N.i64_array(off), N.i64_array(numel),
           N.i32_array(kind), N.i32_array(sexp), C.c_uint64(seed), C.c_void_p(stream or None))


def block_checksums(device_ptr: int, offsets, lengths, stream: int = 0) -> list:
    out = (C.c_uint64 * len(offsets))()
    N.call("lp_block_checksums", C.c_void_p(device_ptr), len(offsets), N.i64_array(offsets),
           N.i64_array(lengths), out, C.c_void_p(stream or None))
    return list(out)


def _fit_ctas(device: int, n_exec: int, push_ctas: int, pull_ctas: int) -> tuple:
    """Scale per-node CTA counts so ``n_exec`` nodes fit one CTA per SM."""
    import torch
    sms = torch.cuda.get_device_properties(device).multi_processor_count
    per = push_ctas + pull_ctas
    if n_exec * per <= sms:
        return push_ctas, pull_ctas
    room = sms // max(1, n_exec)
    if room < (push_ctas > 0) + (pull_ctas > 0):
        raise ValueError(f"{n_exec} nodes on device {device} leave {room} CTAs each: too few for the "
                         f"push and pull roles")
    push = max(1, (push_ctas * room) // per) if push_ctas else 0
    pull = room - push if pull_ctas else 0
    if pull_ctas and pull < 1:
        push, pull = push - 1, 1
    return push, pull


class Cluster:
    """Node images addressable from this process + the engine that moves them."""

    def __init__(self, engine: MulticastEngine, nodes: list, exec_nodes: list, rank: int = 0,
                 world: int = 1, host: HostImage | None = None):
        self.engine = engine
        self.nodes = nodes
        self.exec_nodes = exec_nodes
        self.rank, self.world = rank, world
        self.host = host
        self.epoch = 0

    # -- construction ---------------------------------------------------------

    @classmethod
    def local(cls, n_gpu_nodes: int, block_offsets, block_lengths, image_bytes: int, device: int = 0,
              host_node: bool = False, tile_bytes=DEFAULT_TILE):
        """All GPU nodes on one device (node ids 1.. if a host node 0 exists)."""
        n_nodes = n_gpu_nodes + (1 if host_node else 0)
        with on_device(device):
            eng = MulticastEngine(n_nodes, block_offsets, block_lengths, tile_bytes)
        nodes = []
        host = None
        first = 0
        if host_node:
            host = HostImage(image_bytes)
            eng.set_node(0, LP_NODE_HOST, host.device_ptr)
            nodes.append(NodeBuffer(0, LP_NODE_HOST, -1, host.device_ptr))
            first = 1
        for i in range(first, n_nodes):
            img = dev_malloc(device, image_bytes)
            sig = dev_malloc(device, eng.signal_bytes)
            nb = NodeBuffer(i, LP_NODE_GPU, device, img, sig, [("dev", img), ("dev", sig)])
            eng.set_node(i, LP_NODE_GPU, img, sig)
            eng.reset_signals(i)
            nodes.append(nb)
        N.call("lp_sync_device", device)
        exec_nodes = [nb.node for nb in nodes if nb.kind == LP_NODE_GPU]
        return cls(eng, nodes, exec_nodes, host=host)

    @classmethod
    def distributed(cls, block_offsets, block_lengths, image_bytes: int, host_node: bool = False,
                    tile_bytes=DEFAULT_TILE, shm_name: str = "lambdapipe_host_image"):
        """One GPU node per torchrun rank (node id = rank, +1 with a host node 0)."""
        import torch
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
        device = torch.cuda.current_device()
        off = 1 if host_node else 0
        n_nodes = world + off
        eng = MulticastEngine(n_nodes, block_offsets, block_lengths, tile_bytes)
        img = dev_malloc(device, image_bytes)
        sig = dev_malloc(device, eng.signal_bytes)
        mine = (ipc_handle(img), ipc_handle(sig))
        allh = [None] * world
        dist.all_gather_object(allh, mine)
        nodes = []
        host = None
        if host_node:
            if rank == 0:
                host = HostImage(image_bytes, shm_name, create=True)
            dist.barrier()
            if rank != 0:
                host = HostImage(image_bytes, shm_name, create=False)
            eng.set_node(0, LP_NODE_HOST, host.device_ptr)
            nodes.append(NodeBuffer(0, LP_NODE_HOST, -1, host.device_ptr))
        for r in range(world):
            node = r + off
            if r == rank:
                p_img, p_sig, owned = img, sig, [("dev", img), ("dev", sig)]
            else:
                p_img = ipc_open(device, allh[r][0])
                p_sig = ipc_open(device, allh[r][1])
                owned = [("ipc", p_img), ("ipc", p_sig)]
            eng.set_node(node, LP_NODE_GPU, p_img, p_sig)
            nodes.append(NodeBuffer(node, LP_NODE_GPU, device if r == rank else -2, p_img, p_sig, owned))
        eng.reset_signals(rank + off)
        N.call("lp_sync_device", device)
        dist.barrier()
        return cls(eng, nodes, [rank + off], rank, world, host)

    @classmethod
    def devices(cls, node_devices: list, block_offsets, block_lengths, image_bytes: int, host_node: bool = False,
                tile_bytes=DEFAULT_TILE):
        """One process driving several GPUs: GPU node i lives on device
        ``node_devices[i]`` (node ids shift by one if a host node 0 exists).
        An entry of -1 makes that node a HOST node instead (the box's
        pinned host copy, at any position — e.g. the second source of a
        tier-driven plan, GPU copies first); several HOST positions share
        one pinned copy.
        One engine per device holds the full node table; each device runs
        one kernel over its own nodes (peer access enabled both ways)."""
        node_devices = ([-1] if host_node else []) + list(node_devices)
        devs = sorted(set(d for d in node_devices if d >= 0))
        for a in devs:
            for b in devs:
                if a != b:
                    N.call("lp_enable_peer", a, b)
        n_nodes = len(node_devices)
        engines = {}
        for d in devs:
            with on_device(d):
                engines[d] = MulticastEngine(n_nodes, block_offsets, block_lengths, tile_bytes)
        nodes, host = [], None
        for i, d in enumerate(node_devices):
            if d < 0:                       # every HOST position shares the one pinned copy
                if host is None:
                    with on_device(devs[0]):
                        host = HostImage(image_bytes)
                nodes.append(NodeBuffer(i, LP_NODE_HOST, -1, host.device_ptr))
                continue
            img = dev_malloc(d, image_bytes)
            sig = dev_malloc(d, engines[d].signal_bytes)
            N.call("lp_memset", C.c_void_p(sig), 0, engines[d].signal_bytes, None)
            nodes.append(NodeBuffer(i, LP_NODE_GPU, d, img, sig, [("dev", img), ("dev", sig)]))
        for d, eng in engines.items():
            for nb in nodes:
                eng.set_node(nb.node, nb.kind, nb.image, nb.signals)
        for d in devs:
            N.call("lp_sync_device", d)
        cl = cls(engines[devs[0]], nodes, [nb.node for nb in nodes if nb.kind == LP_NODE_GPU], host=host)
        cl.per_device = engines
        return cl

    @classmethod
    def over_buffers(cls, buffers: list, block_offsets, block_lengths, tile_bytes=DEFAULT_TILE):
        """An engine over EXISTING node buffers (no allocation, nothing freed
        on close): ``buffers[i]`` is the NodeBuffer of op-local node i.  Used
        by the autoscaling server, which keeps one image + signal area per GPU
        across repeated scale-outs."""
        devs = sorted({nb.device for nb in buffers if nb.kind == LP_NODE_GPU})
        engines = {}
        for d in devs:
            with on_device(d):
                eng = MulticastEngine(len(buffers), block_offsets, block_lengths, tile_bytes)
            for i, nb in enumerate(buffers):
                eng.set_node(i, nb.kind, nb.image, nb.signals)
            engines[d] = eng
        nodes = [NodeBuffer(i, nb.kind, nb.device, nb.image, nb.signals, []) for i, nb in enumerate(buffers)]
        cl = cls(engines[devs[0]], nodes, [nb.node for nb in nodes if nb.kind == LP_NODE_GPU])
        cl.per_device = engines
        return cl

    def node(self, i: int) -> NodeBuffer:
        return self.nodes[i]

    def node_device(self, i: int) -> int:
        return self.nodes[i].device

    def set_schedule_all(self, schedule, sources):
        for d, eng in getattr(self, "per_device", {0: self.engine}).items():
            eng.set_schedule(schedule_rows(schedule), sources)

    def launch_devices(self, streams: dict, push_ctas: int = 0, pull_ctas: int = 64) -> int:
        """Multi-device launch: one kernel per device over that device's nodes."""
        self.epoch += 1
        self._mc_streams = {d: (st if isinstance(st, int) else st.cuda_stream) for d, st in streams.items()}
        streams = self._mc_streams
        for d, eng in self.per_device.items():
            mine = [nb.node for nb in self.nodes if nb.kind == LP_NODE_GPU and nb.device == d]
            # every CTA of the dataflow must be co-resident: several nodes on
            # one device (tests, host-fed boxes) share its SMs
            push, pull = _fit_ctas(d, len(mine), push_ctas, pull_ctas)
            with on_device(d):
                eng.run(mine, self.epoch, push, pull, streams[d])
        return self.epoch

    def launch_devices_ce(self, streams: dict) -> int:
        """Multi-device launch on copy engines: every GPU node's ops enqueued
        on its device's stream (``streams``: device -> torch stream).

        Always in the PUSH direction (senders' copy engines write into the
        receivers, waits on the sender's OWN flags): with one process owning
        every GPU, a stream waiting (cuStreamWaitValue32) on another device's
        native allocation deadlocks once relays wait on each other across
        devices — GPU0 -> 3 peers hung in the pull direction and completes in
        push (tools/relay_check.py; one process per GPU, whose peers' flags
        are IPC mappings, pulls fine)."""
        self.epoch += 1
        self._mc_streams = {}
        for d, eng in self.per_device.items():
            cfg = getattr(eng, "cfg", (1, 0, 0, 16384, 3))
            if cfg[0] != 0:
                eng.configure(0, *cfg[1:])
            st = streams[d]
            sts = list(st) if isinstance(st, (list, tuple)) else [st]     # several: ops round-robin
            ptrs = [x if isinstance(x, int) else x.cuda_stream for x in sts]
            with on_device(d):
                for nb in self.nodes:
                    if nb.kind == LP_NODE_GPU and nb.device == d:
                        eng.run_ce(nb.node, self.epoch, ptrs)
        return self.epoch

    def wait_devices(self) -> None:
        """Synchronise every per-device multicast launch; raise on a watchdog expiry."""
        for d, eng in getattr(self, "per_device", {}).items():
            with on_device(d):
                eng.status(getattr(self, "_mc_streams", {}).get(d, 0))

    def complete_nodes(self, epoch: int | None = None) -> dict:
        """node -> per-block complete flags (reads each node's counters)."""
        ep = self.epoch if epoch is None else epoch
        out = {}
        for nb in self.nodes:
            if nb.kind != LP_NODE_GPU:
                continue
            eng = getattr(self, "per_device", {}).get(nb.device, self.engine)
            out[nb.node] = eng.complete(nb.node, ep)
        return out

    def close(self):
        for nb in self.nodes:
            for kind, ptr in nb.owned:
                if kind == "dev":
                    dev_free(max(nb.device, 0), ptr)
                else:
                    N.lib().lp_ipc_close(C.c_void_p(ptr))
            nb.owned = []
        if self.host is not None:
            self.host.close(unlink=self.rank == 0 and self.host.shm_path is not None)
            self.host = None
        for eng in getattr(self, "per_device", {}).values():
            eng.close()
        self.engine.close()

    # -- execution ------------------------------------------------------------

    def set_schedule(self, schedule, sources):
        self.engine.set_schedule(schedule_rows(schedule), sources)

    def launch(self, push_ctas: int = 32, pull_ctas: int = 0, stream: int = 0, epoch: int | None = None):
        """Launch one multicast epoch (async on ``stream``); returns the epoch."""
        if epoch is None:
            self.epoch += 1
            epoch = self.epoch
        else:
            self.epoch = epoch
        if push_ctas < 0 or pull_ctas < 0 or push_ctas + pull_ctas < 1:
            raise InvalidArgumentError("need at least one CTA")
        self.engine.run(self.exec_nodes, epoch, push_ctas, pull_ctas, stream)
        return epoch

    def ce_streams(self, node: int, count: int = 1) -> list:
        """Per-node torch streams the copy-engine executor enqueues on."""
        import torch
        if not hasattr(self, "_ce"):
            self._ce = {}
        if node not in self._ce or len(self._ce[node]) != count:
            dev = torch.cuda.current_device()
            self._ce[node] = [torch.cuda.Stream(device=dev) for _ in range(count)]
        return self._ce[node]

    def launch_ce(self, streams_per_node: int = 1, epoch: int | None = None, after=None) -> int:
        """One epoch on copy engines for every exec node; ``after`` = a torch
        event the CE streams wait for first.  Returns the epoch."""
        if epoch is None:
            self.epoch += 1
            epoch = self.epoch
        else:
            self.epoch = epoch
        for node in self.exec_nodes:
            streams = self.ce_streams(node, streams_per_node)
            if after is not None:
                for st in streams:
                    st.wait_event(after)
            self.engine.run_ce(node, epoch, [st.cuda_stream for st in streams])
        return epoch

    def launch_hybrid(self, stream, push_ctas: int = 0, pull_ctas: int = 64, epoch: int | None = None) -> tuple:
        """One epoch with the hybrid executor: every exec node's HOST-sourced
        receives run as pinned DMA on its copy-engine stream, the NVLink relays
        run in the multicast kernel on ``stream`` (only launched when the node
        has kernel ops).  ``stream`` (torch stream) ends up waiting for both.
        Returns (epoch, kernel launches)."""
        import torch
        if epoch is None:
            self.epoch += 1
            epoch = self.epoch
        else:
            self.epoch = epoch
        self.engine.set_option("host_dma", 1)
        start = torch.cuda.Event()
        start.record(stream)
        run_kernel = []
        for node in self.exec_nodes:
            k_ops, d_ops = self.engine.node_ops(node)
            if d_ops:
                sts = self.ce_streams(node, HOST_DMA_STREAMS)
                for st in sts:
                    st.wait_event(start)
                self.engine.run_host_dma(node, epoch, [st.cuda_stream for st in sts])
            if k_ops:
                run_kernel.append(node)
        if run_kernel:
            self.engine.run(run_kernel, epoch, push_ctas, pull_ctas, stream.cuda_stream)
        self.join_ce(stream)
        return epoch, int(bool(run_kernel)) * (2 if pull_ctas > 0 else 1)   # (+ counter re-base kernel)

    def join_ce(self, stream) -> None:
        """Make ``stream`` wait for every CE stream of this process."""
        import torch
        for node in self.exec_nodes:
            for st in getattr(self, "_ce", {}).get(node, []):
                ev = torch.cuda.Event()
                ev.record(st)
                stream.wait_event(ev)

    def wait(self, stream: int = 0):
        try:
            self.engine.status(stream)
        except NativeError:
            raise


def load_source_image(cluster: "Cluster", node: int, layout, seed: int, device: int = 0):
    """Materialise the synthetic weights on a source node (GPU fill; host
    nodes get a device fill copied down over PCIe)."""
    nb = cluster.node(node)
    if nb.kind == LP_NODE_GPU:
        with on_device(nb.device if nb.device >= 0 else device):
            fill_image(nb.image, layout, seed)
        return
    scratch = dev_malloc(device, layout.weights_bytes)
    try:
        with on_device(device):
            fill_image(scratch, layout, seed)
        N.call("lp_memcpy", C.c_void_p(cluster.host.host_ptr), C.c_void_p(scratch), layout.weights_bytes,
               None)
        N.call("lp_sync_device", device)
    finally:
        dev_free(device, scratch)
