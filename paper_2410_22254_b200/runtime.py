"""ctypes binding of libtlk.so (the C ABI in include/tlk.h).

No CPU fallback: if the library is missing or the device is not an sm_100a
B200, every entry point raises ``TlkError`` -- the packed path never
silently degrades.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

LIB_PATH = os.environ.get("TLK_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libtlk.so")

TLK_OK, TLK_EINVAL, TLK_ECUDA, TLK_EOOM, TLK_ESTATE = 0, -1, -2, -3, -4
MODEL_MLP, MODEL_CNN, MODEL_XFORMER, MODEL_GPT, MODEL_RESNET18 = 1, 2, 3, 4, 5
MODELS = {"mlp": MODEL_MLP, "cnn": MODEL_CNN, "xformer": MODEL_XFORMER, "gpt": MODEL_GPT,
          "resnet18": MODEL_RESNET18}
OPT_ADAM, OPT_ADAMW, OPT_SGD = 1, 2, 3
OPTIMIZERS = {"adam": OPT_ADAM, "adamw": OPT_ADAMW, "sgd": OPT_SGD}
PACK_WRITE_ALL_GRADS = 1
PACK_SNAPSHOTS = 2
PACK_OWN_STREAM = 4
PACK_PERSISTENT = 8
BUF_PARAMS, BUF_GRADS, BUF_MOM1, BUF_MOM2, BUF_WBF16, BUF_LOSS, BUF_PIXELS, BUF_LABELS, BUF_ACTS = range(9)

EXPORTS = (
    "tlk_abi_version", "tlk_last_error", "tlk_model_query", "tlk_model_tensor", "tlk_open",
    "tlk_close", "tlk_sync", "tlk_stream", "tlk_set_mem_limit", "tlk_mem_in_use", "tlk_pack_create",
    "tlk_pack_destroy", "tlk_pack_stream", "tlk_lane_load", "tlk_lane_release",
    "tlk_run", "tlk_step_host", "tlk_pack_host_input_bytes", "tlk_step_host_blob", "tlk_step_host_async", "tlk_step_host_wait", "tlk_lane_status_get", "tlk_lane_losses", "tlk_lane_params",
    "tlk_pack_tensor", "tlk_pack_named", "tlk_pack_info", "tlk_pack_launches_per_step", "tlk_profile_step",
    "tlk_selftest_gemm",
    "tlk_selftest_datagen",
    "tlk_selftest_optimizer", "tlk_cnn_ktrace",
)


class TlkError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"tlk error {code}: {msg}")
        self.code = code
        self.oom = code == TLK_EOOM or "out of memory" in msg


class JobDesc(C.Structure):
    _fields_ = [("task_id", C.c_int64), ("slot_index", C.c_int32), ("steps", C.c_int32),
                ("optimizer", C.c_int32), ("lr", C.c_float), ("beta1", C.c_float),
                ("beta2", C.c_float), ("eps", C.c_float), ("weight_decay", C.c_float),
                ("momentum", C.c_float), ("seed", C.c_uint64)]


class PackDesc(C.Structure):
    _fields_ = [("model", C.c_int32), ("batch", C.c_int32), ("lanes", C.c_int32),
                ("max_steps", C.c_int32), ("host_input", C.c_int32), ("flags", C.c_int32),
                ("layers", C.c_int32), ("d_model", C.c_int32), ("heads", C.c_int32),
                ("seq_len", C.c_int32), ("vocab", C.c_int32)]


class ModelInfo(C.Structure):
    _fields_ = [("param_count", C.c_int64), ("param_stride", C.c_int64),
                ("flops_per_sample", C.c_int64), ("num_tensors", C.c_int32)]


class LaneStatus(C.Structure):
    _fields_ = [("active", C.c_int32), ("steps_done", C.c_int32), ("steps", C.c_int32),
                ("error", C.c_int32)]


_lib = None
_lock = threading.Lock()


def lib():
    """Load libtlk.so once; raise (never fall back) when it is absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise TlkError(TLK_ESTATE, f"{LIB_PATH} missing: run `python -m paper_2410_22254_b200.build`")
            L = C.CDLL(LIB_PATH)
            for name in EXPORTS:
                getattr(L, name).restype = C.c_int
            L.tlk_last_error.restype = C.c_char_p
            _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != TLK_OK:
        raise TlkError(rc, lib().tlk_last_error().decode("utf-8", "replace"))


def model_info(model: int) -> ModelInfo:
    info = ModelInfo()
    check(lib().tlk_model_query(model, 64, C.byref(info)))
    return info


def model_tensors(model: int):
    """[(offset, count, fan_in)] per tensor, from the library's layout table."""
    info = model_info(model)
    out = []
    for t in range(info.num_tensors):
        off, cnt, fan = C.c_int64(), C.c_int64(), C.c_int32()
        check(lib().tlk_model_tensor(model, t, C.byref(off), C.byref(cnt), C.byref(fan)))
        out.append((off.value, cnt.value, fan.value))
    return out


class _CudaArray:
    """__cuda_array_interface__ view of a device buffer (zero-copy torch handoff)."""

    def __init__(self, ptr: int, shape, typestr: str, owner):
        self.__cuda_array_interface__ = {
            "shape": tuple(shape), "typestr": typestr, "data": (ptr, False), "version": 3,
            "strides": None,
        }
        self._owner = owner


class Context:
    """One per GPU: the device-resident home of every packed lane on it."""

    def __init__(self, device: int = 0):
        self._ctx = C.c_void_p()
        check(lib().tlk_open(int(device), C.byref(self._ctx)))
        self.device = device

    def close(self):
        if self._ctx:
            lib().tlk_close(self._ctx)
            self._ctx = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def sync(self):
        check(lib().tlk_sync(self._ctx))

    @property
    def stream_handle(self) -> int:
        s = C.c_void_p()
        check(lib().tlk_stream(self._ctx, C.byref(s)))
        return s.value or 0

    def set_mem_limit(self, nbytes: int) -> None:
        """Admission budget for pack memory (0 = device memory only)."""
        check(lib().tlk_set_mem_limit(self._ctx, C.c_int64(int(nbytes))))

    def mem_in_use(self) -> int:
        n = C.c_int64()
        check(lib().tlk_mem_in_use(self._ctx, C.byref(n)))
        return n.value

    def pack(self, model: int, batch: int, lanes: int, max_steps: int, host_input: bool = False,
             flags: int = 0, **cfg):
        return Pack(self, model, batch, lanes, max_steps, host_input, flags, **cfg)


class Pack:
    """K co-resident training lanes of one model (tlk_pack_*)."""

    def __init__(self, ctx: Context, model: int, batch: int, lanes: int, max_steps: int,
                 host_input: bool = False, flags: int = 0, layers: int = 0, d_model: int = 0,
                 heads: int = 0, seq_len: int = 0, vocab: int = 0):
        self.ctx, self.model, self.batch, self.lanes = ctx, model, batch, lanes
        self.max_steps, self.host_input = max_steps, host_input
        desc = PackDesc(model, batch, lanes, max_steps, int(host_input), int(flags), layers, d_model,
                        heads, seq_len, vocab)
        pid = C.c_int32()
        check(lib().tlk_pack_create(ctx._ctx, C.byref(desc), C.byref(pid)))
        self.id = pid.value
        self.info = ModelInfo()
        check(lib().tlk_pack_info(ctx._ctx, self.id, C.byref(self.info)))

    def load(self, lane: int, *, seed: int, steps: int, optimizer: int = OPT_ADAM, lr: float = 1e-3,
             beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8, weight_decay: float = 0.0,
             momentum: float = 0.0, task_id: int = 0, slot_index: int = 0):
        d = JobDesc(task_id, slot_index, steps, optimizer, lr, beta1, beta2, eps, weight_decay,
                    momentum, seed & 0xFFFFFFFFFFFFFFFF)
        check(lib().tlk_lane_load(self.ctx._ctx, self.id, lane, C.byref(d)))

    def release(self, lane: int):
        check(lib().tlk_lane_release(self.ctx._ctx, self.id, lane))

    def destroy(self):
        """Free the pack's device memory (tlk_pack_destroy); the pack is unusable after."""
        if self.id >= 0:
            check(lib().tlk_pack_destroy(self.ctx._ctx, self.id))
            self.id = -1

    @property
    def stream_handle(self) -> int:
        s = C.c_void_p()
        check(lib().tlk_pack_stream(self.ctx._ctx, self.id, C.byref(s)))
        return s.value or 0

    def run(self, steps: int):
        check(lib().tlk_run(self.ctx._ctx, self.id, int(steps)))

    def step_host(self, pixels, labels, losses_out=None):
        """One end-to-end step from host numpy buffers (uint8 [L,B,784], int32 [L,B])."""
        import numpy as np

        px = np.ascontiguousarray(pixels, dtype=np.uint8)
        lb = np.ascontiguousarray(labels, dtype=np.int32)
        assert px.shape == (self.lanes, self.batch, 784) and lb.shape == (self.lanes, self.batch)
        out = losses_out if losses_out is not None else np.empty(self.lanes, np.float32)
        check(lib().tlk_step_host(self.ctx._ctx, self.id, px.ctypes.data_as(C.c_void_p),
                                  lb.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p)))
        return out

    def host_input_bytes(self) -> int:
        n = C.c_int64()
        check(lib().tlk_pack_host_input_bytes(self.ctx._ctx, self.id, C.byref(n)))
        return n.value

    def step_host_blob(self, blob, losses_out=None):
        """One end-to-end step from a host blob (any model; layout in tlk.h)."""
        blob = np.ascontiguousarray(blob)
        out = losses_out if losses_out is not None else np.empty(self.lanes, np.float32)
        check(lib().tlk_step_host_blob(self.ctx._ctx, self.id, blob.ctypes.data_as(C.c_void_p),
                                       C.c_int64(blob.nbytes), out.ctypes.data_as(C.c_void_p)))
        return out

    def step_host_async(self, pixels, labels, losses_out) -> int:
        """Pipelined end-to-end step (tlk_step_host_async): returns a ticket at once;
        the buffers (pinned numpy views) must stay alive until step_host_wait(ticket)."""
        assert pixels.dtype == np.uint8 and labels.dtype == np.int32 and losses_out.dtype == np.float32
        assert pixels.shape == (self.lanes, self.batch, 784) and labels.shape == (self.lanes, self.batch)
        assert pixels.flags.c_contiguous and labels.flags.c_contiguous and losses_out.size >= self.lanes
        t = C.c_int64(0)
        check(lib().tlk_step_host_async(self.ctx._ctx, self.id, pixels.ctypes.data_as(C.c_void_p),
                                        labels.ctypes.data_as(C.c_void_p), losses_out.ctypes.data_as(C.c_void_p),
                                        C.byref(t)))
        return t.value

    def step_host_wait(self, ticket: int) -> None:
        check(lib().tlk_step_host_wait(self.ctx._ctx, self.id, C.c_int64(ticket)))

    def status(self, lane: int) -> LaneStatus:
        s = LaneStatus()
        check(lib().tlk_lane_status_get(self.ctx._ctx, self.id, lane, C.byref(s)))
        return s

    def losses(self, lane: int, n: int):
        import numpy as np

        out = np.zeros(n, np.float32)
        check(lib().tlk_lane_losses(self.ctx._ctx, self.id, lane,
                                    out.ctypes.data_as(C.c_void_p), int(n)))
        return out

    def params(self, lane: int):
        import numpy as np

        out = np.zeros(self.info.param_stride, np.float32)
        check(lib().tlk_lane_params(self.ctx._ctx, self.id, lane, out.ctypes.data_as(C.c_void_p),
                                    int(self.info.param_stride)))
        return out

    def launches_per_step(self) -> int:
        n = C.c_int32()
        check(lib().tlk_pack_launches_per_step(self.ctx._ctx, self.id, C.byref(n)))
        return n.value

    def profile_step(self, iters: int = 5):
        """[(kernel name, mean ms)] for one step, measured with CUDA events on
        the context stream (un-graphed; advances the lanes by `iters` steps)."""
        cap, nlen = 1024, 32768
        ms = (C.c_float * cap)()
        names = C.create_string_buffer(nlen)
        n = C.c_int32()
        check(lib().tlk_profile_step(self.ctx._ctx, self.id, int(iters), ms, names, nlen, cap,
                                     C.byref(n)))
        labels = names.value.decode().split(",")
        return [(labels[k], float(ms[k])) for k in range(n.value)]

    def named(self, name: str, dtype: str = "f4"):
        """Zero-copy torch view of a named model buffer (tlk_pack_named)."""
        import torch

        ptr, nbytes = C.c_void_p(), C.c_int64()
        check(lib().tlk_pack_named(self.ctx._ctx, self.id, name.encode(), C.byref(ptr), C.byref(nbytes)))
        itemsize = {"f4": 4, "u2": 2, "i4": 4}[dtype]
        return torch.as_tensor(_CudaArray(ptr.value, (nbytes.value // itemsize,), "<" + dtype, self),
                               device=f"cuda:{self.ctx.device}")

    def tensor(self, which: int):
        """Zero-copy torch view of a pack buffer (TLK_BUF_*)."""
        import torch

        ptr, nbytes = C.c_void_p(), C.c_int64()
        check(lib().tlk_pack_tensor(self.ctx._ctx, self.id, which, C.byref(ptr), C.byref(nbytes)))
        typestr, itemsize = {BUF_WBF16: ("<u2", 2), BUF_ACTS: ("<u2", 2), BUF_PIXELS: ("|u1", 1),
                             BUF_LABELS: ("<i4", 4)}.get(which, ("<f4", 4))
        n = nbytes.value // itemsize
        t = torch.as_tensor(_CudaArray(ptr.value, (n,), typestr, self), device=f"cuda:{self.ctx.device}")
        return t


def selftest_gemm(a_mn: bool, b_mn: bool, bn: int, A, B, Cout, batch, M, N, K, stream=0):
    check(lib().tlk_selftest_gemm(int(a_mn), int(b_mn), int(bn), C.c_void_p(A.data_ptr()),
                                  C.c_void_p(B.data_ptr()), C.c_void_p(Cout.data_ptr()),
                                  int(batch), int(M), int(N), int(K), C.c_void_p(stream)))


def selftest_optimizer(kind: int, seed: int, n: int) -> int:
    """Bit mismatches of the packed optimizer update vs its library-intrinsic form."""
    out = C.c_uint64(0)
    check(lib().tlk_selftest_optimizer(int(kind), C.c_uint64(seed), C.c_int64(n), C.byref(out)))
    return out.value


def selftest_datagen(seed: int, step: int, batch: int, px, labels, stream=0):
    check(lib().tlk_selftest_datagen(C.c_uint64(seed), int(step), int(batch),
                                     C.c_void_p(px.data_ptr()), C.c_void_p(labels.data_ptr()),
                                     C.c_void_p(stream)))
