"""Python binding of the out-of-core training-step executor (pooch_ctx).

Argument marshalling only: profiling (Sec. 4.2), classification (Sec. 4.4) and
execution (fwd / bwd with swap and recompute, update) all run in libpooch.so.
PyTorch is used by callers for device memory, pinned host memory, streams and
process groups; this module only passes their raw pointers through the C ABI.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import P, IODesc, LayerDesc, PlanReport, ProfileT, SearchCfg, check, lib
from .planning import STRATEGIES

NETS = {"tiny": 0, "resnet50": 1, "resnet50v1": 2, "unet3d": 3, "alexnet": 4, "resnext3d": 5, "resnext50_3d": 6}
KINDS = ["conv", "bnrelu", "tail_proj", "tail_id", "maxpool", "avgpool", "fc_ce", "upconv", "head_ce", "bnrelu_conv",
         "conv_relu", "lrn", "fc_relu_drop"]
FAMILIES = ["conv_fwd", "conv_dgrad", "conv_wgrad", "bn_fwd", "bn_bwd", "pool", "fc_ce", "sgd",
            "swap_out", "swap_in", "allreduce", "other", "stall", "gconv_fwd", "gconv_dgrad", "gconv_wgrad"]


FUSE_BNRELU = 16   # POOCH_NET_FUSE_BNRELU: BN-ReLU on the consuming conv's operand load


def build_net(name: str, in_hw: int, classes: int, width: int = 32, fuse: bool = False):
    """Layer descriptors of a built-in workload (pooch_build_net); fuse=True merges every
    conv-feeding BN-ReLU into its conv (POOCH_L_BNRELU_CONV)."""
    which = NETS[name] | (FUSE_BNRELU if fuse else 0)
    n = C.c_int32(0)
    check(lib.pooch_build_net(which, in_hw, classes, width, None, C.byref(n)))
    arr = (LayerDesc * n.value)()
    check(lib.pooch_build_net(which, in_hw, classes, width, arr, C.byref(n)))
    return arr


class PinnedHost:
    """Page-locked host arena of exactly `nbytes` (numpy pages registered with
    cudaHostRegister; torch's pinned allocator rounds up to a power of two, which
    turns 157 GB into 256 GB). The caller owns it (pooch_set_budget's host arena)."""

    def __init__(self, nbytes: int):
        import torch
        self.nbytes = int(nbytes)
        self.buf = np.empty(self.nbytes, np.uint8)
        self.cudart = torch.cuda.cudart()
        err = self.cudart.cudaHostRegister(self.buf.ctypes.data, self.nbytes, 0)
        if int(err) != 0:
            raise RuntimeError("cudaHostRegister(%d bytes) failed: %s" % (self.nbytes, err))

    def data_ptr(self):
        return self.buf.ctypes.data

    def numel(self):
        return self.nbytes

    def __del__(self):
        try:
            self.cudart.cudaHostUnregister(self.buf.ctypes.data)
        except Exception:
            pass


def _ptr(x):
    """Raw address of a torch tensor / int / None."""
    if x is None:
        return None
    if isinstance(x, int):
        return C.c_void_p(x)
    if hasattr(x, "data_ptr"):
        return C.c_void_p(x.data_ptr())
    if hasattr(x, "cuda_stream"):
        return C.c_void_p(x.cuda_stream)
    raise TypeError(type(x))


class Context:
    def __init__(self, layers, batch: int, in_c: int, in_h: int, in_w: int, classes: int, device: int = 0,
                 in_d: int = 0):
        self.layers = layers
        self.n = len(layers)
        self.batch, self.in_c, self.in_h, self.in_w, self.classes = batch, in_c, in_h, in_w, classes
        self.in_d = in_d
        io = IODesc(batch, in_c, in_h, in_w, classes, in_d)
        h = C.c_void_p()
        check(lib.pooch_create(layers, len(layers), C.byref(io), device, C.byref(h)))
        self.h = h
        self._keep = []

    @classmethod
    def builtin(cls, name, batch, in_hw=None, classes=None, width=32, device=0, fuse=False):
        if name == "unet3d":   # config 4: in_hw^3 volume, input channels padded 1 -> 32
            in_hw = in_hw or 256
            classes = classes or 2
            return cls(build_net(name, in_hw, classes, width, fuse), batch, 32, in_hw, in_hw, classes, device,
                       in_d=in_hw)
        if name in ("resnext3d", "resnext50_3d"):   # in_hw = H = W, width = D; input channels 3 -> 4
            classes = classes or 400
            return cls(build_net(name, in_hw, classes, width, fuse), batch, 4, in_hw, in_hw, classes, device,
                       in_d=width)
        in_hw = in_hw or {"tiny": 32, "alexnet": 227}.get(name, 224)
        classes = classes or (10 if name == "tiny" else 1000)
        return cls(build_net(name, in_hw, classes, width, fuse), batch, 4, in_hw, in_hw, classes, device)

    def close(self):
        if self.h:
            lib.pooch_destroy(self.h)
            self.h = None
        self._keep = []          # release the caller's arenas held for the context's lifetime

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, st):
        check(st, self.h)

    # ---------------------------------------------------------------- setup
    def resident_bytes(self) -> int:
        v = C.c_uint64()
        self._chk(lib.pooch_resident_bytes(self.h, C.byref(v)))
        return v.value

    def set_budget(self, dev, dev_bytes, host=None, host_bytes=0):
        self._keep = [dev, host]
        self._chk(lib.pooch_set_budget(self.h, _ptr(dev), int(dev_bytes), _ptr(host), int(host_bytes)))

    def set_streams(self, compute, d2h, h2d, comm=None):
        self._streams = (compute, d2h, h2d, comm)
        self._chk(lib.pooch_set_streams(self.h, _ptr(compute), _ptr(d2h), _ptr(h2d), _ptr(comm)))

    def set_precision(self, precision: int):
        """0 = TF32, 1 = 3xTF32 (default)."""
        self._chk(lib.pooch_set_precision(self.h, int(precision)))

    def set_comm(self, unique_id: bytes, rank: int, world: int):
        buf = C.create_string_buffer(bytes(unique_id), 128)
        self._chk(lib.pooch_set_comm(self.h, buf, rank, world))

    def peer_open(self, rank: int, world: int) -> bytes:
        """Allocate this rank's IPC-exported exchange buffer for the peer-memory allreduce;
        returns its 64-byte cudaIpcMemHandle (all-gather them, then set_peers)."""
        h = C.create_string_buffer(64)
        nb = C.c_uint64(0)
        self._chk(lib.pooch_peer_open(self.h, int(rank), int(world), h, C.byref(nb)))
        self.peer_bytes = nb.value
        return bytes(h.raw)

    def set_peers(self, handles):
        """Map every rank's exchange buffer (handles in rank order)."""
        buf = C.create_string_buffer(b"".join(bytes(x) for x in handles), 64 * len(handles))
        self._chk(lib.pooch_set_peers(self.h, buf))

    def allreduce_buckets(self):
        """[(lo, hi, close_task)] float ranges of the gradient region allreduced per bucket."""
        n = C.c_int32(0)
        self._chk(lib.pooch_allreduce_buckets(self.h, C.byref(n), None, None, None))
        lo, hi = np.zeros(n.value, np.uint64), np.zeros(n.value, np.uint64)
        ct = np.zeros(n.value, np.int32)
        self._chk(lib.pooch_allreduce_buckets(self.h, C.byref(n), lo.ctypes.data, hi.ctypes.data, ct.ctypes.data))
        return [(int(a), int(b), int(t)) for a, b, t in zip(lo, hi, ct)]

    def set_rng(self, seed: int, step: int):
        """(seed, step) of the counter-based dropout masks (pooch_set_rng)."""
        self._chk(lib.pooch_set_rng(self.h, seed & 0xFFFFFFFF, step & 0xFFFFFFFF))

    def input_slot(self):
        x, l = C.c_void_p(), C.c_void_p()
        self._chk(lib.pooch_input_slot(self.h, C.byref(x), C.byref(l)))
        return x.value, l.value

    # ---------------------------------------------------------------- parameters
    def params(self):
        n = C.c_int32()
        self._chk(lib.pooch_num_params(self.h, C.byref(n)))
        out = []
        buf = C.create_string_buffer(64)
        for i in range(n.value):
            k = C.c_int64()
            self._chk(lib.pooch_param_info(self.h, i, buf, C.byref(k)))
            out.append((buf.value.decode(), k.value))
        return out

    def set_param(self, i, arr, which=0):
        a = np.ascontiguousarray(arr, dtype=np.float32).ravel()
        self._chk(lib.pooch_set_param(self.h, i, which, a.ctypes.data_as(P(C.c_float)), a.size))

    def get_param(self, i, which=0):
        k = self.params()[i][1]
        a = np.empty(k, np.float32)
        self._chk(lib.pooch_get_param(self.h, i, which, a.ctypes.data_as(P(C.c_float)), k))
        return a

    # ---------------------------------------------------------------- profile / plan / step
    PROFILE_MODES = {"auto": 0, "isolated": 1, "all_swap": 2}

    def set_profile_mode(self, mode: str):
        """'auto' (all-swap iterations when they fit, else isolated), 'isolated' or 'all_swap'."""
        self._chk(lib.pooch_set_profile_mode(self.h, self.PROFILE_MODES[mode]))

    def profile(self, iters=3):
        pr = ProfileT()
        self._chk(lib.pooch_profile(self.h, iters, C.byref(pr)))
        n = pr.n
        g = lambda p: [int(p[i]) for i in range(n)] if p else None
        return dict(fwd=g(pr.fwd_ns), bwd=g(pr.bwd_ns), rec=g(pr.rec_ns), d2h=g(pr.d2h_ns), h2d=g(pr.h2d_ns),
                    bytes=g(pr.bytes), tail=int(pr.tail_ns), resident=int(pr.resident_bytes),
                    d2h_gbs=pr.d2h_gbs, h2d_gbs=pr.h2d_gbs, duplex_gbs=pr.duplex_gbs,
                    mode={1: "isolated", 2: "all_swap"}.get(int(pr.mode), str(pr.mode)),
                    d2h_issue=g(pr.d2h_issue_ns), h2d_issue=g(pr.h2d_issue_ns), step_ns=int(pr.step_ns))

    def comm_info(self):
        """(nranks, rank, cuda device) of the library's NCCL communicator (ncclCommCount etc.)."""
        a, b, d = C.c_int32(), C.c_int32(), C.c_int32()
        self._chk(lib.pooch_comm_info(self.h, C.byref(a), C.byref(b), C.byref(d)))
        return a.value, b.value, d.value

    def set_profile(self, fwd, bwd, rec, d2h, h2d, tail):
        arrs = [np.asarray(v, np.int64) for v in (fwd, bwd, rec, d2h, h2d)]
        self._chk(lib.pooch_set_profile(self.h, *[a.ctypes.data_as(P(C.c_int64)) for a in arrs], int(tail)))

    def set_link(self, d2h_gbs, h2d_gbs, duplex_gbs):
        """Override the probed host-link rates (GB/s) the planner's link model uses (Reading 51)."""
        self._chk(lib.pooch_set_link(self.h, float(d2h_gbs), float(h2d_gbs), float(duplex_gbs)))

    def plan(self, strategy="pooch", li_cap=16, threads=0, sched=0, fixed=None):
        out = np.zeros(self.n, np.uint8)
        rep = PlanReport()
        fx = None if fixed is None else np.asarray(fixed, np.uint8)
        self._chk(lib.pooch_plan(self.h, STRATEGIES[strategy], C.byref(SearchCfg(li_cap, threads, sched)),
                                 None if fx is None else fx.ctypes.data_as(P(C.c_uint8)),
                                 out.ctypes.data_as(P(C.c_uint8)), C.byref(rep)))
        rd = {k: getattr(rep, k) for k, _ in PlanReport._fields_}
        return [int(v) for v in out], rd

    def train_step(self, lr: float, sync_loss: bool = True):
        if sync_loss:
            loss = C.c_float()
            self._chk(lib.pooch_train_step(self.h, lr, C.byref(loss)))
            return loss.value
        self._chk(lib.pooch_train_step(self.h, lr, None))
        return None

    def step_was_graph(self) -> bool:
        """Whether the last train_step ran as one captured CUDA graph launch."""
        v = C.c_int32()
        self._chk(lib.pooch_step_graph(self.h, C.byref(v)))
        return bool(v.value)

    def read_buffer(self, which, m, nbytes):
        a = np.empty(nbytes // 4, np.float32)
        self._chk(lib.pooch_read_buffer(self.h, which, m, a.ctypes.data, nbytes))
        return a

    def loss_slot(self):
        p = C.c_void_p()
        self._chk(lib.pooch_loss_slot(self.h, C.byref(p)))
        return p.value

    def set_timing(self, on: bool):
        self._chk(lib.pooch_set_timing(self.h, 1 if on else 0))

    def last_timing(self):
        arrs = [np.zeros(self.n, np.int64) for _ in range(5)]
        step = C.c_int64()
        self._chk(lib.pooch_last_timing(self.h, *[a.ctypes.data_as(P(C.c_int64)) for a in arrs], C.byref(step)))
        return dict(zip(("fwd", "bwd", "rec", "d2h", "h2d"), arrs), step_ns=step.value)

    def last_trace(self, simulated=False):
        """Measured timeline of the last instrumented step (simulated=True: the current plan's
        simulated one): [(lane, kind, id, start_ns, end_ns)]."""
        fn = lib.pooch_plan_trace if simulated else lib.pooch_last_trace
        n = C.c_int32(0)
        self._chk(fn(self.h, C.byref(n), None, None, None, None, None))
        a = [np.zeros(n.value, np.int32) for _ in range(3)] + [np.zeros(n.value, np.int64) for _ in range(2)]
        self._chk(fn(self.h, C.byref(n), *[x.ctypes.data for x in a]))
        lanes = ("COMPUTE", "D2H", "H2D")
        return [(lanes[int(l)], chr(int(k)), int(i), int(s), int(e)) for l, k, i, s, e in zip(*a)]

    def timing_segments(self):
        """Per-launch-group (family, ms, flops, bytes) of the last instrumented step."""
        n = C.c_int32(0)
        self._chk(lib.pooch_timing_segments(self.h, C.byref(n), None, None, None, None))
        fam = np.zeros(n.value, np.int32)
        arr = [np.zeros(n.value, np.float64) for _ in range(3)]
        self._chk(lib.pooch_timing_segments(self.h, C.byref(n), fam.ctypes.data, *[a.ctypes.data for a in arr]))
        return [(FAMILIES[int(f)], float(m), float(fl), float(b)) for f, m, fl, b in zip(fam, *arr)]

    def family_stats(self):
        out = {}
        for f, name in enumerate(FAMILIES):
            t, l, fl, by = C.c_double(), C.c_int64(), C.c_double(), C.c_double()
            self._chk(lib.pooch_family_stats(self.h, f, C.byref(t), C.byref(l), C.byref(fl), C.byref(by)))
            out[name] = dict(ms=t.value, launches=l.value, flops=fl.value, bytes=by.value)
        return out
