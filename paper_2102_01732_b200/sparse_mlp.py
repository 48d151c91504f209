"""Thin ctypes binding of libsparse_mlp.so (include/sparse_mlp.h): argument marshalling only.

Every call maps 1:1 onto a C-ABI function of the same name; every step of the training path runs
in the library's sm_100a kernels.  There is no CPU fallback: if the library is missing the import
fails, and every call on a machine without a CUDA device fails in the library.

PyTorch is used for plumbing only: device tensors (raw pointers are passed), the current stream,
and (optionally) the caching allocator the library allocates through.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SMLP_LIB") or os.path.join(_PKG, "lib", "libsparse_mlp.so")   # SMLP_LIB: A/B builds

SMLP_MAX_LAYERS = 16
ACTIVATIONS = {"relu": 0, "all_relu": 1}
INITS = {"normal": 0, "xavier": 1, "he_uniform": 2}
ERRORS = {0: "OK", -1: "E_ARG", -2: "E_NOMEM", -3: "E_CUDA", -4: "E_SHAPE", -5: "E_STALE", -6: "E_DATA",
          -7: "E_STATE", -8: "E_STRUCT"}
PRUNE_OUTGOING = 1

# the symbols include/sparse_mlp.h declares (checked by tests/test_abi.py)
EXPORTED = [
    "sparse_mlp_create", "sparse_mlp_destroy", "sparse_mlp_set_stream", "sparse_mlp_forward",
    "sparse_mlp_backward", "sparse_mlp_step", "sparse_mlp_train_step_host", "sparse_mlp_train_step_host_async",
    "sparse_mlp_sync", "sparse_mlp_gradient_flow", "sparse_mlp_export_positions", "sparse_mlp_union_average_layer",
    "sparse_mlp_retain_valid_updates", "sparse_mlp_wait_layer", "sparse_mlp_view_layout", "sparse_mlp_grad_view",
    "sparse_mlp_param_view", "sparse_mlp_evolve_topology", "sparse_mlp_prune_neurons",
    "sparse_mlp_importance", "sparse_mlp_info", "sparse_mlp_export_layer", "sparse_mlp_import_layer",
    "sparse_mlp_export_bias", "sparse_mlp_import_bias", "sparse_mlp_export_alive",
    "sparse_mlp_import_alive", "sparse_mlp_export_trace", "sparse_mlp_last_error", "sparse_mlp_version",
    "sparse_mlp_profile", "sparse_mlp_profile_read", "sparse_mlp_set_step_counter",
    "sparse_mlp_params_updated", "sparse_mlp_plan_chunks", "sparse_mlp_join", "sparse_mlp_params_averaged",
]
KERNEL_KINDS = {0: "stage_input", 1: "fwd", 2: "fwd_finish", 3: "softmax_ce", 4: "bwd", 5: "bwd_finish",
                6: "sgd_update", 7: "fwd_bits", 8: "bwd_bits", 9: "layer_update", 10: "mirror_values",
                11: "persist_fwd", 12: "persist_bwd"}


class SparseMLPError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)


class smlp_allocator(C.Structure):
    _fields_ = [("alloc", ALLOC_FN), ("free", FREE_FN), ("ctx", C.c_void_p)]


class smlp_config(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("sizes", C.POINTER(C.c_int64)), ("epsilon", C.c_double),
                ("activation", C.c_int32), ("alpha", C.c_float), ("dropout", C.c_float),
                ("init", C.c_int32), ("seed", C.c_uint64), ("rank", C.c_int32), ("max_batch", C.c_int32),
                ("chunk_batch", C.c_int32), ("device", C.c_int32), ("stream", C.c_void_p),
                ("allocator", C.POINTER(smlp_allocator)), ("input_kind", C.c_int32)]


class smlp_sgd(C.Structure):
    _fields_ = [("lr", C.c_float), ("momentum", C.c_float), ("weight_decay", C.c_float),
                ("grad_scale", C.c_float)]


class smlp_kernel_stat(C.Structure):
    _fields_ = [("kind", C.c_int32), ("layer", C.c_int32), ("launches", C.c_int64), ("total_ms", C.c_double),
                ("bytes_per_launch", C.c_double), ("flops_per_launch", C.c_double)]


class smlp_info(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("chunk_batch", C.c_int32), ("version", C.c_uint64),
                ("sizes", C.c_int64 * SMLP_MAX_LAYERS), ("alive", C.c_int64 * SMLP_MAX_LAYERS),
                ("nnz", C.c_int64 * SMLP_MAX_LAYERS), ("cap", C.c_int64 * SMLP_MAX_LAYERS),
                ("dense_capped", C.c_int32 * SMLP_MAX_LAYERS), ("val_offset", C.c_int64 * SMLP_MAX_LAYERS),
                ("bias_offset", C.c_int64 * SMLP_MAX_LAYERS), ("param_count", C.c_int64),
                ("launches", C.c_int64), ("fwd_chunk_batch", C.c_int32), ("implicit_delta", C.c_int32)]


_lib = None


def plan_chunks(sizes, max_batch: int, chunk_batch: int = 0, l2_bytes: int = 126 << 20):
    """(chunk_batch, fwd_chunk_batch) sparse_mlp_create would pick (host-only C call)."""
    L = load_library()
    arr = (C.c_int64 * len(sizes))(*[int(n) for n in sizes])
    cb, cbf = C.c_int32(), C.c_int32()
    rc = L.sparse_mlp_plan_chunks(arr, len(sizes), int(max_batch), int(chunk_batch), int(l2_bytes),
                                  C.byref(cb), C.byref(cbf))
    if rc != 0:
        raise ValueError(L.sparse_mlp_last_error(None).decode())
    return cb.value, cbf.value


def load_library(path: str = LIB_PATH):
    """Load libsparse_mlp.so (raises if it has not been built: no fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not found; build it with `python -m paper_2102_01732_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(path)
    P, VP, I32, I64, U64, D, F = C.POINTER, C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_float
    sig = {
        "sparse_mlp_create": (I32, [P(smlp_config), P(VP)]),
        "sparse_mlp_plan_chunks": (I32, [P(I64), I32, I32, I32, I64, P(I32), P(I32)]),
        "sparse_mlp_join": (I32, [VP]),
        "sparse_mlp_destroy": (I32, [VP]),
        "sparse_mlp_set_stream": (I32, [VP, VP]),
        "sparse_mlp_forward": (I32, [VP, VP, VP, I32, I32, U64, VP]),
        "sparse_mlp_backward": (I32, [VP, VP, VP, VP, P(smlp_sgd)]),
        "sparse_mlp_step": (I32, [VP, P(smlp_sgd)]),
        "sparse_mlp_train_step_host": (I32, [VP, VP, VP, I32, U64, P(smlp_sgd), VP]),
        "sparse_mlp_train_step_host_async": (I32, [VP, VP, VP, I32, U64, P(smlp_sgd), VP]),
        "sparse_mlp_sync": (I32, [VP]),
        "sparse_mlp_gradient_flow": (I32, [VP, VP]),
        "sparse_mlp_export_positions": (I32, [VP, I32, VP, VP]),
        "sparse_mlp_union_average_layer": (I32, [VP, I32, I32, VP, VP, I64, I64, VP]),
        "sparse_mlp_retain_valid_updates": (I32, [VP, I32, VP, VP, I64, VP]),
        "sparse_mlp_wait_layer": (I32, [VP, I32, VP]),
        "sparse_mlp_view_layout": (I32, [VP, VP, VP, VP]),
        "sparse_mlp_grad_view": (I32, [VP, P(VP), P(I64), P(U64)]),
        "sparse_mlp_param_view": (I32, [VP, P(VP), P(I64), P(U64)]),
        "sparse_mlp_evolve_topology": (I32, [VP, D, U64, VP]),
        "sparse_mlp_prune_neurons": (I32, [VP, D, I32, VP, VP]),
        "sparse_mlp_importance": (I32, [VP, I32, VP, I32]),
        "sparse_mlp_info": (I32, [VP, P(smlp_info)]),
        "sparse_mlp_export_layer": (I32, [VP, I32, VP, VP, VP, VP, I32]),
        "sparse_mlp_import_layer": (I32, [VP, I32, I64, VP, VP, VP, VP]),
        "sparse_mlp_export_bias": (I32, [VP, I32, VP, VP]),
        "sparse_mlp_import_bias": (I32, [VP, I32, VP, VP]),
        "sparse_mlp_export_alive": (I32, [VP, I32, VP]),
        "sparse_mlp_import_alive": (I32, [VP, I32, VP]),
        "sparse_mlp_export_trace": (I32, [VP, I32, I32, VP]),
        "sparse_mlp_profile": (I32, [VP, I32]),
        "sparse_mlp_profile_read": (I32, [VP, P(smlp_kernel_stat), I32, P(I32)]),
        "sparse_mlp_set_step_counter": (I32, [VP, VP]),
        "sparse_mlp_params_updated": (I32, [VP]),
        "sparse_mlp_params_averaged": (I32, [VP, I32, I32]),
        "sparse_mlp_last_error": (C.c_char_p, [VP]),
        "sparse_mlp_version": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


@dataclass
class SGD:
    """Eq. 1 hyper-parameters: lr eta, momentum mu, weight decay lambda."""
    lr: float
    momentum: float = 0.9
    weight_decay: float = 0.0
    grad_scale: float = 1.0

    def c(self) -> smlp_sgd:
        return smlp_sgd(self.lr, self.momentum, self.weight_decay, self.grad_scale)


def _ptr(t) -> int:
    """Raw data pointer of a torch tensor / numpy array / int / None."""
    if t is None:
        return 0
    if isinstance(t, int):
        return t
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


class _CudaArray:
    """Zero-copy __cuda_array_interface__ wrapper so torch.as_tensor can view library memory."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False),
                                         "version": 3, "strides": None}


class SparseMLP:
    """A truly sparse MLP on one GPU: the handle of libsparse_mlp.so."""

    def __init__(self, sizes: Sequence[int], epsilon: float, activation: str = "all_relu", alpha: float = 0.5,
                 dropout: float = 0.0, init: str = "he_uniform", seed: int = 0, rank: int = 0,
                 max_batch: int = 128, chunk_batch: int = 0, device: Optional[int] = None,
                 use_torch_allocator: bool = True, input_kind: int = 0):
        import torch
        self._torch = torch
        self.lib = load_library()
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.sizes = [int(s) for s in sizes]
        self.L = len(self.sizes)
        self._sizes_c = (C.c_int64 * self.L)(*self.sizes)
        self._alloc = None
        alloc_p = None
        if use_torch_allocator:
            dev = self.device

            def _a(nbytes, stream, ctx):
                try:
                    return torch.cuda.caching_allocator_alloc(int(nbytes), dev, int(stream or 0))
                except Exception:   # out of memory -> NULL -> SMLP_E_NOMEM
                    return None

            def _f(p, nbytes, stream, ctx):
                torch.cuda.caching_allocator_delete(int(p))

            self._alloc_fns = (ALLOC_FN(_a), FREE_FN(_f))
            self._alloc = smlp_allocator(self._alloc_fns[0], self._alloc_fns[1], None)
            alloc_p = C.pointer(self._alloc)
        with torch.cuda.device(self.device):
            stream = torch.cuda.current_stream().cuda_stream
            cfg = smlp_config(self.L, self._sizes_c, float(epsilon), ACTIVATIONS[activation], float(alpha),
                              float(dropout), INITS[init], int(seed) & (2**64 - 1), int(rank), int(max_batch),
                              int(chunk_batch), self.device, C.c_void_p(stream), alloc_p, int(input_kind))
            h = C.c_void_p()
            rc = self.lib.sparse_mlp_create(C.byref(cfg), C.byref(h))
        if rc != 0:
            raise SparseMLPError(rc, self.lib.sparse_mlp_last_error(None).decode())
        self.h = h
        self.max_batch = int(max_batch)

    # -------------------------------------------------------------------------------- helpers
    def _check(self, rc: int):
        if rc != 0:
            raise SparseMLPError(rc, self.lib.sparse_mlp_last_error(self.h).decode())

    def _sync_stream(self):
        self._check(self.lib.sparse_mlp_set_stream(self.h, C.c_void_p(self._torch.cuda.current_stream().cuda_stream)))

    def close(self):
        if getattr(self, "h", None):
            self.lib.sparse_mlp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -------------------------------------------------------------------------------- hot path
    def sparse_mlp_forward(self, x, B: Optional[int] = None, x_idx=None, train: bool = True, step: int = 0,
                           probs=None):
        B = int(x.shape[0] if (B is None and x_idx is None) else (B if B is not None else x_idx.shape[0]))
        self._sync_stream()
        self._check(self.lib.sparse_mlp_forward(self.h, _ptr(x), _ptr(x_idx), B, int(bool(train)), int(step),
                                                _ptr(probs)))

    def sparse_mlp_backward(self, labels, y_idx=None, loss=None, fused: Optional[SGD] = None):
        self._sync_stream()
        f = C.byref(fused.c()) if fused is not None else None
        self._check(self.lib.sparse_mlp_backward(self.h, _ptr(labels), _ptr(y_idx), _ptr(loss), f))

    def sparse_mlp_step(self, sgd: SGD):
        self._sync_stream()
        self._check(self.lib.sparse_mlp_step(self.h, C.byref(sgd.c())))

    def sparse_mlp_train_step_host(self, x_host, y_host, B: int, step: int, sgd: SGD) -> float:
        self._sync_stream()
        out = C.c_float(0.0)
        self._check(self.lib.sparse_mlp_train_step_host(self.h, _ptr(x_host), _ptr(y_host), int(B), int(step),
                                                        C.byref(sgd.c()), C.byref(out)))
        return float(out.value)

    def sparse_mlp_train_step_host_async(self, x_host, y_host, B: int, step: int, sgd: SGD, loss_host=None):
        """Pipelined host-buffer step (pinned x_host / y_host / loss_host tensors); no sync."""
        self._sync_stream()
        self._check(self.lib.sparse_mlp_train_step_host_async(self.h, _ptr(x_host), _ptr(y_host), int(B), int(step),
                                                              C.byref(sgd.c()), _ptr(loss_host)))

    def sparse_mlp_sync(self):
        self._check(self.lib.sparse_mlp_sync(self.h))

    def sparse_mlp_join(self):
        """Rejoin the library's side-stream work (deferred mirror refreshes) on the handle's stream;
        call before ending a CUDA-graph capture that contains a training step."""
        self._check(self.lib.sparse_mlp_join(self.h))

    def sparse_mlp_gradient_flow(self) -> float:
        """Squared L2 norm of the pending (unfused) gradient."""
        self._sync_stream()
        out = C.c_double(0.0)
        self._check(self.lib.sparse_mlp_gradient_flow(self.h, C.byref(out)))
        return float(out.value)

    def sparse_mlp_export_positions(self, l: int):
        """(pos uint64 as int64 tensor, val float32 tensor) of W^(l) on the device, canonical order."""
        torch = self._torch
        nnz = self.sparse_mlp_info()["nnz"][l - 1]
        pos = torch.empty(max(nnz, 1), dtype=torch.int64, device=f"cuda:{self.device}")
        val = torch.empty(max(nnz, 1), dtype=torch.float32, device=f"cuda:{self.device}")
        self._sync_stream()
        self._check(self.lib.sparse_mlp_export_positions(self.h, int(l), _ptr(pos), _ptr(val)))
        return pos[:nnz], val[:nnz]

    def sparse_mlp_union_average_layer(self, l: int, K: int, pos_all, val_all, target: int) -> int:
        """WASAP phase-2 union averaging of W^(l) (see include/sparse_mlp.h); returns the kept count."""
        kept = C.c_int64(0)
        self._sync_stream()
        self._check(self.lib.sparse_mlp_union_average_layer(self.h, int(l), int(K), _ptr(pos_all), _ptr(val_all),
                                                            int(pos_all.numel()), int(target), C.byref(kept)))
        return int(kept.value)

    def sparse_mlp_retain_valid_updates(self, l: int, stale_pos, stale_g) -> int:
        """Map a stale gradient of W^(l) (device tensors: sorted positions, values) onto the current
        support, into the grad view (RetainValidUpdates); returns the intersection size."""
        out = C.c_int64(0)
        self._sync_stream()
        self._check(self.lib.sparse_mlp_retain_valid_updates(self.h, int(l), _ptr(stale_pos), _ptr(stale_g),
                                                             int(stale_pos.numel()), C.byref(out)))
        return int(out.value)

    def sparse_mlp_wait_layer(self, l: int, stream):
        """`stream` (torch.cuda.Stream) waits until W^(l)'s gradient of the last backward is final."""
        self._check(self.lib.sparse_mlp_wait_layer(self.h, int(l), C.c_void_p(stream.cuda_stream)))

    def sparse_mlp_view_layout(self):
        """([(val_off, cap) for W^(2)..W^(L)], bias_base) in floats of the grad / param views."""
        n = self.L - 1
        off, cap, bb = (C.c_int64 * n)(), (C.c_int64 * n)(), C.c_int64()
        self._check(self.lib.sparse_mlp_view_layout(self.h, off, cap, C.byref(bb)))
        return [(int(off[i]), int(cap[i])) for i in range(n)], int(bb.value)

    def sparse_mlp_grad_view(self):
        p, n, v = C.c_void_p(), C.c_int64(), C.c_uint64()
        self._check(self.lib.sparse_mlp_grad_view(self.h, C.byref(p), C.byref(n), C.byref(v)))
        return self._torch.as_tensor(_CudaArray(p.value, n.value), device=f"cuda:{self.device}"), v.value

    def sparse_mlp_param_view(self):
        p, n, v = C.c_void_p(), C.c_int64(), C.c_uint64()
        self._check(self.lib.sparse_mlp_param_view(self.h, C.byref(p), C.byref(n), C.byref(v)))
        return self._torch.as_tensor(_CudaArray(p.value, n.value), device=f"cuda:{self.device}"), v.value

    def sparse_mlp_params_updated(self):
        """Call after writing the param view in place (averaging): refreshes the mirror copy."""
        self._sync_stream()
        self._check(self.lib.sparse_mlp_params_updated(self.h))

    # -------------------------------------------------------------------------------- topology
    def sparse_mlp_params_averaged(self, K: int, biases_only: bool = False):
        """Eq. 2's division by K after the caller's SUM allreduce of the param view (or its bias
        block) + mirror refresh, in the library."""
        self._sync_stream()
        self._check(self.lib.sparse_mlp_params_averaged(self.h, int(K), int(bool(biases_only))))

    def sparse_mlp_evolve_topology(self, zeta: float, evolve_idx: int):
        out = (C.c_int64 * self.L)()
        self._sync_stream()
        self._check(self.lib.sparse_mlp_evolve_topology(self.h, float(zeta), int(evolve_idx), out))
        return list(out)

    def sparse_mlp_prune_neurons(self, percentile: float, outgoing: bool = True):
        pr = (C.c_int64 * self.L)()
        rm = (C.c_int64 * self.L)()
        self._sync_stream()
        self._check(self.lib.sparse_mlp_prune_neurons(self.h, float(percentile), PRUNE_OUTGOING if outgoing else 0,
                                                      pr, rm))
        return list(pr), list(rm)

    def sparse_mlp_importance(self, l: int) -> np.ndarray:
        out = np.zeros(self.sizes[l - 1], np.float64)
        self._check(self.lib.sparse_mlp_importance(self.h, int(l), out.ctypes.data, 1))
        return out

    # -------------------------------------------------------------------------------- state I/O
    def sparse_mlp_info(self) -> dict:
        inf = smlp_info()
        self._check(self.lib.sparse_mlp_info(self.h, C.byref(inf)))
        L = inf.n_layers
        return {"n_layers": L, "chunk_batch": inf.chunk_batch, "version": inf.version,
                "sizes": list(inf.sizes[:L]), "alive": list(inf.alive[:L]), "nnz": list(inf.nnz[:L]),
                "cap": list(inf.cap[:L]), "dense_capped": list(inf.dense_capped[:L]),
                "val_offset": list(inf.val_offset[:L]), "bias_offset": list(inf.bias_offset[:L]),
                "param_count": inf.param_count, "launches": inf.launches,
                "fwd_chunk_batch": inf.fwd_chunk_batch, "implicit_delta": inf.implicit_delta}

    def sparse_mlp_export_layer(self, l: int) -> dict:
        nnz = self.sparse_mlp_info()["nnz"][l - 1]
        rp = np.zeros(self.sizes[l - 2] + 1, np.int32)
        col = np.zeros(max(nnz, 1), np.int32)
        val = np.zeros(max(nnz, 1), np.float32)
        mom = np.zeros(max(nnz, 1), np.float32)
        self._check(self.lib.sparse_mlp_export_layer(self.h, int(l), rp.ctypes.data, col.ctypes.data,
                                                     val.ctypes.data, mom.ctypes.data, 1))
        return {"row_ptr": rp, "col": col[:nnz], "w": val[:nnz], "v": mom[:nnz]}

    def sparse_mlp_import_layer(self, l: int, row_ptr, col, w, v=None):
        rp = np.ascontiguousarray(row_ptr, np.int32)
        cl = np.ascontiguousarray(col, np.int32)
        wv = np.ascontiguousarray(w, np.float32)
        vv = None if v is None else np.ascontiguousarray(v, np.float32)
        self._check(self.lib.sparse_mlp_import_layer(self.h, int(l), int(len(cl)), rp.ctypes.data, cl.ctypes.data,
                                                     wv.ctypes.data, None if vv is None else vv.ctypes.data))

    def sparse_mlp_export_bias(self, l: int):
        b = np.zeros(self.sizes[l - 1], np.float32)
        vb = np.zeros(self.sizes[l - 1], np.float32)
        self._check(self.lib.sparse_mlp_export_bias(self.h, int(l), b.ctypes.data, vb.ctypes.data))
        return b, vb

    def sparse_mlp_import_bias(self, l: int, b, vb=None):
        b = np.ascontiguousarray(b, np.float32)
        vb = None if vb is None else np.ascontiguousarray(vb, np.float32)
        self._check(self.lib.sparse_mlp_import_bias(self.h, int(l), b.ctypes.data,
                                                    None if vb is None else vb.ctypes.data))

    def sparse_mlp_export_alive(self, l: int) -> np.ndarray:
        a = np.zeros(self.sizes[l - 1], np.uint8)
        self._check(self.lib.sparse_mlp_export_alive(self.h, int(l), a.ctypes.data))
        return a

    def sparse_mlp_import_alive(self, l: int, alive):
        a = np.ascontiguousarray(alive, np.uint8)
        self._check(self.lib.sparse_mlp_import_alive(self.h, int(l), a.ctypes.data))

    def sparse_mlp_export_trace(self, kind: int, l: int, B: Optional[int] = None) -> np.ndarray:
        """kind 0: activations a_l [B x n_l] (l = L: logits); 1: deltas; 2: grad of W^(l) values; 3: bias grad;
        4: binary-input path flag of the last forward (1 taken, 0 not, -1 disabled)."""
        if kind == 4:
            out = np.zeros(1, np.float32)
            self._check(self.lib.sparse_mlp_export_trace(self.h, 4, 0, out.ctypes.data))
            return out
        if kind in (0, 1):
            out = np.zeros((B, self.sizes[l - 1]), np.float32)
        elif kind == 2:
            out = np.zeros(max(1, self.sparse_mlp_info()["nnz"][l - 1]), np.float32)
        else:
            out = np.zeros(self.sizes[l - 1], np.float32)
        self._check(self.lib.sparse_mlp_export_trace(self.h, int(kind), int(l), out.ctypes.data))
        if kind == 2:
            out = out[: self.sparse_mlp_info()["nnz"][l - 1]]
        return out

    # -------------------------------------------------------------------------------- timing / graphs
    def sparse_mlp_profile(self, enable: bool):
        self._check(self.lib.sparse_mlp_profile(self.h, int(bool(enable))))

    def sparse_mlp_profile_read(self) -> list:
        cap = 64
        arr = (smlp_kernel_stat * cap)()
        n = C.c_int32(0)
        self._check(self.lib.sparse_mlp_profile_read(self.h, arr, cap, C.byref(n)))
        return [{"kernel": KERNEL_KINDS.get(a.kind, str(a.kind)), "layer": a.layer, "launches": a.launches,
                 "total_ms": a.total_ms, "bytes_per_launch": a.bytes_per_launch,
                 "flops_per_launch": a.flops_per_launch} for a in arr[: min(cap, n.value)]]

    def sparse_mlp_set_step_counter(self, counter=None):
        """counter: a CUDA uint64/int64 tensor holding the dropout step (graph replay), or None."""
        self._check(self.lib.sparse_mlp_set_step_counter(self.h, _ptr(counter)))

    # short aliases
    forward = sparse_mlp_forward
    backward = sparse_mlp_backward
    step = sparse_mlp_step
    evolve_topology = sparse_mlp_evolve_topology
    prune_neurons = sparse_mlp_prune_neurons
    info = sparse_mlp_info
    export_layer = sparse_mlp_export_layer
    import_layer = sparse_mlp_import_layer
    grad_view = sparse_mlp_grad_view
    param_view = sparse_mlp_param_view
    train_step_host = sparse_mlp_train_step_host
    train_step_host_async = sparse_mlp_train_step_host_async
    wait_layer = sparse_mlp_wait_layer
    gradient_flow = sparse_mlp_gradient_flow
    params_updated = sparse_mlp_params_updated
    params_averaged = sparse_mlp_params_averaged
    export_positions = sparse_mlp_export_positions
    union_average_layer = sparse_mlp_union_average_layer
    retain_valid_updates = sparse_mlp_retain_valid_updates
    view_layout = sparse_mlp_view_layout
    sync = sparse_mlp_sync
    join = sparse_mlp_join


def from_config(cfg, seed: Optional[int] = None, rank: int = 0, max_batch: Optional[int] = None,
                chunk_batch: int = 0, device: Optional[int] = None) -> SparseMLP:
    """Build a SparseMLP from a synth.WorkloadConfig-like object (sizes, epsilon, ...)."""
    # known {0,1} inputs: checked and reported (the bit path needs max_batch <= 128, else auto);
    # known real-valued: no detection, no bit path; else auto
    b = getattr(cfg, "binary_input", None)
    mb = int(max_batch or cfg.batch)
    kind = 0 if b is None else ((2 if mb <= 128 else 0) if b else 1)
    return SparseMLP(cfg.sizes, cfg.epsilon, cfg.activation, cfg.alpha, cfg.dropout, cfg.init,
                     cfg.model_seed if seed is None else seed, rank, max_batch or cfg.batch, chunk_batch, device,
                     input_kind=kind)
