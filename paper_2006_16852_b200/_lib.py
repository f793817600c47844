"""ctypes binding of libb200sp.so (the C ABI declared in include/b200sp.h).

The library is built in-tree by ``__graft_entry__.build()`` /
``make -C paper_2006_16852_b200/csrc``. There is no CPU fallback: if the
shared object is missing every kernel call raises KernelNotImplemented.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import KernelNotImplemented, OpalgError, ParameterError, Singular, Unsupported

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libb200sp.so")

# type codes: l=int64 i=int32 u=uint64 p=pointer d=double V=value type of the suffix
_P = ctypes.c_void_p
_CT = {"l": ctypes.c_int64, "i": ctypes.c_int32, "u": ctypes.c_uint64, "p": _P,
       "d": ctypes.c_double, "s": ctypes.c_char_p}

_SPMV_TAIL = "VpVppl"          # alpha, alpha_dev, beta, beta_dev, x_in, x_in_stride
_TYPED = {
    # BLAS-1
    "fill": "liplVp",
    "copy": "liplplp",
    "scale": "liVpplp",
    "add_scaled": "liVpplplp",
    "dot": "liplplpppp",
    "norm2": "liplpppp",
    # SpMV
    "csr_spmv_classical": "lpppplpl" + _SPMV_TAIL + "ip",
    "csr_spmv_lb": "llpppplpl" + _SPMV_TAIL + "pppiip",
    "csr_spmv_stream": "llpppplpl" + _SPMV_TAIL + "iiiip",
    "csr_spmv_tma": "llpppplpl" + _SPMV_TAIL + "iiiiip",
    "coo_spmv": "lipppplpl" + _SPMV_TAIL + "pppp",
    "rows_scale": "lpplVpplp",
    "ell_spmv": "lllppplpl" + _SPMV_TAIL + "p",
    "sellp_spmv": "lippppplpl" + _SPMV_TAIL + "p",
    "dense_spmv": "llplplplp",
    "stencil3_apply": "liVVVplplp",
    # conversions
    "csr_to_ell": "lpppllppp",
    "csr_to_sellp": "lpppippppp",
    "csr_to_hybrid_coo": "lpppippppp",
    "ell_to_csr_fill": "lllpppppp",
    "sellp_to_csr_fill": "lipppppppp",
    "hybrid_coo_append": "lpppppppp",
    "dense_row_nnz": "llplpp",
    "dense_to_csr_fill": "llplpppp",
    "csr_to_dense": "lpppplp",
    # generators
    "stencil_fill": "illdllpppp",
    "powerlaw_fill": "lupppp",
    # block-Jacobi
    "jacobi_invert": "lpppppppppidpp",
    "jacobi_apply": "lppppiplplp",
    "jacobi_invert_large": "lpppppppppidpipip",
    "jacobi_apply_large": "lppppiplplp",
    # Krylov (JAC = l p p p p)
    "cg_init": "lppp" + "lpppp" + "pppp",
    "cg_step1": "lpppp",
    "cg_step1_put": "lpppippppippp",
    "peer_put": "pippppipppp",
    "cg_sigma": "lppppp",
    "cg_coop": "lpppppppppppp",
    "bicgstab_coop": "lpppppppppppppp",
    "fcg_coop": "lpppppppppppp",
    "cgs_coop": "l" + "p" * 16,
    "csr_spmv_dot": "lppppppiippp",
    "cg_step2": "lplpppp" + "lpppp" + "pppp",
    "fcg_step2": "lplppppp" + "lpppp" + "pppp",
    "cgs_step1": "lppppp" + "lpppp" + "pp",
    "cgs_step2": "lppppp" + "lpppp" + "pp",
    "cgs_step3": "lplpppppppp",
    "bicgstab_init": "lplpppppppppppp",
    "bicgstab_step1": "lpppp" + "lpppp" + "pp",
    "bicgstab_gamma": "lppppp",
    "bicgstab_step2": "lpppp" + "lpppp" + "pppp",
    "bicgstab_tst": "lppppp",
    "bicgstab_step3": "lplpppppppppp",
    "gmres_reset": "lppppp" + "ip",
    "gmres_scale_v0": "lpppp",
    "gmres_dot0": "lipppppp",
    "gmres_mgs": "lii" + "ppppppp",
    "gmres_normalize": "lipppp",
    "gmres_arnoldi_small": "lipppppp",
    "gmres_cycle_small": "l" + "p" * 9,
    "gmres_solve_tiny": "l" + "p" * 10 + "ip",
    "gmres_combine": "lppl" + "lpppp" + "ppp",
    # distributed
    "split_fill": "lpppippppppp",
    "assemble_coo": "lpppllpppppp",
    "diag": "lpppppp",
    "ilu_fill": "lppppppppppppp",
    "parilu_sweep": "lllppppppppppppp",
    "trs": "lppppiplplpippp",
    "trs_coop": "lppppplplppip",
    "gather": "lpppp",
}
_UNTYPED = {
    "last_error": ("", ctypes.c_char_p),
    "launch_count": ("", ctypes.c_longlong),
    "version": ("", ctypes.c_int),
    "device_sync": ("", ctypes.c_int),
    "reduce_workspace_elems": ("", ctypes.c_int64),
    "scan_workspace_elems": ("l", ctypes.c_int64),
    "exclusive_scan_i32": ("lpppp", ctypes.c_int),
    "exclusive_scan_i64": ("lpppp", ctypes.c_int),
    "reduce_max_i32": ("lppp", ctypes.c_int),
    "csr_lb_tile": ("ii", ctypes.c_int32),
    "csr_lb_num_tiles": ("lli", ctypes.c_int64),
    "csr_stream_capacity": ("i", ctypes.c_int32),
    "csr_tma_stage_bytes": ("iii", ctypes.c_int64),
    "csr_lb_plan": ("llpipp", ctypes.c_int),
    "csr_seg_plan": ("llppp", ctypes.c_int),
    "peer_max": ("", ctypes.c_int32),
    "gmres_small_rows": ("", ctypes.c_int32),
    "peer_wait": ("pipipp", ctypes.c_int),
    "peer_ack": ("ippp", ctypes.c_int),
    "peer_wait_plain": ("ippp", ctypes.c_int),
    "peer_allreduce": ("piiippipp", ctypes.c_int),
    "csr_row_lengths": ("lppp", ctypes.c_int),
    "csr_to_coo_rows": ("lppp", ctypes.c_int),
    "coo_to_csr_ptrs": ("llppp", ctypes.c_int),
    "sellp_slice_lengths": ("lpiipp", ctypes.c_int),
    "hybrid_overflow_counts": ("lpipp", ctypes.c_int),
    "ell_row_lengths": ("lllppp", ctypes.c_int),
    "sellp_row_lengths": ("lippppp", ctypes.c_int),
    "add_csr_lengths": ("lppp", ctypes.c_int),
    "length_histogram": ("lpipp", ctypes.c_int),
    "empty_row_flags": ("lppp", ctypes.c_int),
    "compact_flags": ("lpppp", ctypes.c_int),
    "stencil_lengths": ("illllpp", ctypes.c_int),
    "powerlaw_lengths": ("lupipp", ctypes.c_int),
    "set_guard": ("p", None),
    "set_tuning": ("si", ctypes.c_int),
    "assemble_workspace_bytes": ("l", ctypes.c_int64),
    "ilu_counts": ("lpppppp", ctypes.c_int),
    "csr_rows": ("lppp", ctypes.c_int),
    "trs_levels": ("lppippp", ctypes.c_int),
    "trs_level_hist": ("lppp", ctypes.c_int),
    "trs_order": ("lppppp", ctypes.c_int),
    "fcg_init_ctl": ("pp", ctypes.c_int),
    "cgs_mid": ("ppp", ctypes.c_int),
    "mm_header": ("plpp", ctypes.c_int),
    "mm_count": ("plpip", ctypes.c_int),
    "mm_parse": ("plpippplpp", ctypes.c_int),
    "jacobi_block_sizes_sq": ("lppp", ctypes.c_int),
    "jacobi_pack": ("lppppppp", ctypes.c_int),
    "jacobi_large_max_block": ("", ctypes.c_int64),
    "ipc_handle_bytes": ("", ctypes.c_int32),
    "ipc_export": ("ppp", ctypes.c_int),
    "ipc_open": ("plpp", ctypes.c_int),
    "ipc_close": ("p", ctypes.c_int),
    "peer_enable": ("ip", ctypes.c_int),
    "krylov_ctl_bytes": ("", ctypes.c_int64),
    "krylov_part_elems": ("", ctypes.c_int64),
    "krylov_ctl_init": ("pippiiip", ctypes.c_int),
    "krylov_status": ("pppp", ctypes.c_int),
    "krylov_force_stop": ("piip", ctypes.c_int),
    "krylov_guard": ("pi", ctypes.c_void_p),
    "gmres_workspace_elems": ("i", ctypes.c_int64),
    "gmres_backsolve": ("ppp", ctypes.c_int),
    "gmres_after_commit": ("pp", ctypes.c_int),
    "krylov_set_dist": ("pip", ctypes.c_int),
    "krylov_red_offset": ("", ctypes.c_int64),
    "cg_finish": ("ppip", ctypes.c_int),
    "flag_out_of_range": ("lpllpp", ctypes.c_int),
    "compact_cols": ("lppppp", ctypes.c_int),
    "map_cols": ("lpllplp", ctypes.c_int),
    "split_count": ("lppippp", ctypes.c_int),
}

_lock = threading.Lock()
_lib = None
_funcs = {}


def _load():
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise KernelNotImplemented(
                f"CUDA extension {LIB_PATH} is missing: build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (sig, res) in _UNTYPED.items():
            fn = getattr(lib, "b200sp_" + name)
            fn.argtypes = [_CT[c] for c in sig]
            fn.restype = res
            _funcs[name] = fn
        for name, sig in _TYPED.items():
            for suf, vt in (("f64", ctypes.c_double), ("f32", ctypes.c_float)):
                fn = getattr(lib, f"b200sp_{name}_{suf}", None)
                if fn is None:
                    continue
                fn.argtypes = [vt if c == "V" else _CT[c] for c in sig]
                fn.restype = ctypes.c_int
                _funcs[f"{name}_{suf}"] = fn
        _lib = lib
        return lib


def available():
    try:
        _load()
        return True
    except KernelNotImplemented:
        return False


def _raise(code, name):
    msg = _funcs["last_error"]().decode(errors="replace")
    text = f"b200sp_{name}: {msg}"
    if code == 1:
        raise ParameterError(text)
    if code == 3:
        raise Singular(text)
    if code == 4:
        raise Unsupported(text)
    raise OpalgError(text)


def call(name, *args):
    """Invoke b200sp_<name>; raise the mapped error on a non-zero return."""
    _load()
    fn = _funcs[name]
    rc = fn(*args)
    if fn.restype is ctypes.c_int and rc != 0:
        _raise(rc, name)
    return rc


def query(name, *args):
    """Invoke a function returning a value (not an error code)."""
    _load()
    return _funcs[name](*args)


def set_tuning(key, value):
    """Select a kernel variant / launch shape by name (benchmark sweeps)."""
    call("set_tuning", key.encode(), int(value))


TUNING_DEFAULT = -(2 ** 31)  # include/b200sp.h B200SP_TUNING_DEFAULT


def reset_tuning(key):
    """Restore a knob's built-in (measured-best) default."""
    call("set_tuning", key.encode(), TUNING_DEFAULT)


def launch_count():
    _load()
    return int(_funcs["launch_count"]())


def suffix(dtype):
    """'f64' / 'f32' for a torch or numpy float dtype."""
    s = str(dtype)
    if s.endswith("float64"):
        return "f64"
    if s.endswith("float32"):
        return "f32"
    raise Unsupported(f"value type {dtype} (supported: float64, float32)")


def exported_symbols():
    """Every b200sp_* symbol named in include/b200sp.h (for the CPU ABI test)."""
    names = ["b200sp_" + n for n in _UNTYPED]
    for n in _TYPED:
        names += [f"b200sp_{n}_f64", f"b200sp_{n}_f32"]
    return names
