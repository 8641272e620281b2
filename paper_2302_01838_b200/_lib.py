"""ctypes binding of libvmap_b200.so (include/vmap_b200.h).

The shared library is built in-tree by `__graft_entry__.build()` (make -C
paper_2302_01838_b200/csrc).  There is no fallback: if the library is missing
or CUDA is unavailable every compute entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libvmap_b200.so"

VM_OK, VM_ERR_SHAPE, VM_ERR_CUDA, VM_ERR_UNSUPPORTED = 0, 1, 3, 4
VM_MAX_LAYERS = 8
STATUS_NONE = 0x7F7F7F7F  # "no model" sentinel written into status words

c_float_p = C.c_void_p  # all device pointers travel as void*


class VmArch(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("hidden", C.c_int32), ("input_dim", C.c_int32),
                ("reserved", C.c_int32)]


class VmLayout(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("hidden_pad", C.c_int32),
                ("fo", C.c_int32 * VM_MAX_LAYERS), ("fi", C.c_int32 * VM_MAX_LAYERS),
                ("fo_pad", C.c_int32 * VM_MAX_LAYERS), ("fi_pad", C.c_int32 * VM_MAX_LAYERS),
                ("w_off", C.c_int64 * VM_MAX_LAYERS), ("b_off", C.c_int64 * VM_MAX_LAYERS),
                ("block", C.c_int64), ("n_params", C.c_int64)]


class VmStack(C.Structure):
    _fields_ = [("arch", VmArch), ("count", C.c_int32), ("capacity", C.c_int32),
                ("params", C.c_void_p), ("m", C.c_void_p), ("v", C.c_void_p), ("step", C.c_void_p),
                ("frozen", C.c_void_p), ("corr1", C.c_void_p), ("corr2", C.c_void_p),
                ("corr_len", C.c_int32),
                ("beta1f", C.c_float), ("omb1", C.c_float), ("beta2f", C.c_float), ("omb2", C.c_float),
                ("eps", C.c_float), ("lr", C.c_float), ("beta1", C.c_double), ("beta2", C.c_double)]


class VmBatch(C.Structure):
    _fields_ = [("n_models", C.c_int32), ("n_rays", C.c_int32), ("n_points", C.c_int32),
                ("input_dim", C.c_int32),
                ("encoded", C.c_void_p), ("points", C.c_void_p), ("pe_scale", C.c_void_p),
                ("t", C.c_void_p), ("target_depth", C.c_void_p), ("target_colour", C.c_void_p),
                ("target_mask", C.c_void_p), ("valid_depth", C.c_void_p), ("ray_ok", C.c_void_p),
                ("model_rays", C.c_void_p), ("work_items", C.c_void_p), ("n_work_items", C.c_int32),
                ("reserved", C.c_int32)]


class VmLossWeights(C.Structure):
    _fields_ = [("colour", C.c_float), ("occupancy", C.c_float)]


class VmKeyframe(C.Structure):
    _fields_ = [("texel_off", C.c_int64), ("u0", C.c_int32), ("v0", C.c_int32), ("u1", C.c_int32),
                ("v1", C.c_int32), ("pose", C.c_double * 12)]


class VmSampleObject(C.Structure):
    _fields_ = [("object_id", C.c_int64), ("kf_begin", C.c_int32), ("n_kf", C.c_int32),
                ("active", C.c_int32), ("n_rays", C.c_int32),
                ("box_min", C.c_double * 3), ("box_max", C.c_double * 3),
                ("center", C.c_double * 3), ("half", C.c_double * 3), ("pe_scale", C.c_double)]


class VmSampleParams(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("step", C.c_int64),
                ("n_rays", C.c_int32), ("n_stratified", C.c_int32), ("n_surface", C.c_int32),
                ("encode", C.c_int32), ("n_freq", C.c_int32), ("include_input", C.c_int32),
                ("reserved0", C.c_int32), ("reserved1", C.c_int32),
                ("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32),
                ("t_near", C.c_double), ("t_far", C.c_double), ("surface_std", C.c_double),
                ("three_std", C.c_double), ("step_dev", C.c_void_p), ("step_offset", C.c_int64)]


class VmDetection(C.Structure):
    _fields_ = [("instance_id", C.c_int32), ("n_pixels", C.c_int32), ("n_valid", C.c_int32), ("reserved", C.c_int32),
                ("u0", C.c_int32), ("v0", C.c_int32), ("u1", C.c_int32), ("v1", C.c_int32),
                ("box_min", C.c_double * 3), ("box_max", C.c_double * 3)]


class VmSampleAux(C.Structure):
    _fields_ = [("kf_idx", C.c_void_p), ("u", C.c_void_p), ("v", C.c_void_p), ("t64", C.c_void_p)]


_SIGNATURES = {
    "vm_model_layout": (C.c_int, [C.POINTER(VmArch), C.POINTER(VmLayout)]),
    "vm_train_workspace_bytes": (C.c_size_t, [C.POINTER(VmStack), C.POINTER(VmBatch), C.c_int]),
    "vm_infer_workspace_bytes": (C.c_size_t, [C.POINTER(VmArch), C.c_int64]),
    "vm_query_grid": (C.c_int, [C.POINTER(VmStack), C.c_int32, C.c_void_p, C.c_void_p, C.c_double, C.c_void_p,
                                C.c_void_p, C.c_void_p, C.c_size_t, C.c_int64, C.c_void_p]),
    "vm_eval_rays": (C.c_int, [C.POINTER(VmStack), C.c_int32, C.c_void_p, C.c_void_p, C.c_double, C.c_void_p,
                               C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_double, C.c_double,
                               C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int64,
                               C.c_void_p]),
    "vm_view_rays": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "vm_ray_box_select": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_double,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "vm_view_compose": (C.c_int, [C.c_int32, C.c_int64] + [C.c_void_p] * 6 + [C.c_double] * 3 + [C.c_int32]
                        + [C.c_void_p] * 5),
    "vm_decode_frame": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_double,
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "vm_ingest_workspace_bytes": (C.c_size_t, [C.c_int32, C.c_int32]),
    "vm_ingest_frame": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_int32,
                                  C.c_double, C.c_int32, C.c_double, C.POINTER(VmDetection), C.c_int32,
                                  C.POINTER(C.c_int32), C.c_void_p, C.POINTER(C.c_int32), C.c_void_p, C.c_size_t,
                                  C.c_void_p]),
    "vm_pack_floats": (C.c_int64, [C.POINTER(VmStack)]),
    "vm_pack_stack": (C.c_int, [C.POINTER(VmStack), C.c_void_p, C.c_int32, C.c_void_p]),
    "vm_work_items": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_int32, C.POINTER(C.c_int32)]),
    "vm_train_step": (C.c_int, [C.POINTER(VmStack), C.POINTER(VmBatch), C.c_int, VmLossWeights,
                                C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "vm_forward": (C.c_int, [C.POINTER(VmStack), C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                             C.c_void_p]),
    "vm_backward": (C.c_int, [C.POINTER(VmStack), C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                              C.c_void_p, C.c_void_p]),
    "vm_adam": (C.c_int, [C.POINTER(VmStack), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "vm_render_forward": (C.c_int, [C.c_int64, C.c_int32] + [C.c_void_p] * 8 + [C.c_void_p]),
    "vm_render_backward": (C.c_int, [C.c_int64, C.c_int32] + [C.c_void_p] * 10 + [C.c_void_p]),
    "vm_losses": (C.c_int, [C.c_int32, C.c_int32] + [C.c_void_p] * 8 + [VmLossWeights]
                  + [C.c_void_p] * 7 + [C.c_void_p]),
    "vm_sample_workspace_bytes": (C.c_size_t, [C.c_int, C.POINTER(VmSampleParams)]),
    "vm_sample": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                            C.POINTER(VmSampleParams), C.POINTER(VmBatch), C.POINTER(VmSampleAux),
                            C.c_void_p, C.c_size_t, C.c_void_p]),
    "vm_profile_enable": (C.c_int, [C.c_int]),
    "vm_profile_read": (C.c_int, [C.POINTER(C.c_int), C.POINTER(C.c_double)]),
    "vm_profile_read_tag": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_double)]),
    "vm_profile_kernels": (C.c_int, [C.POINTER(C.c_long)]),
    "vm_trace_read": (C.c_int, [C.POINTER(C.c_ulonglong), C.c_int, C.POINTER(C.c_int)]),
    "vm_profile_count_kernels": (None, [C.c_int]),
    "vm_train_grid": (C.c_int, [C.POINTER(VmStack), C.POINTER(VmBatch), C.c_int, C.POINTER(C.c_int),
                                C.POINTER(C.c_int)]),
    "vm_step_advance": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p]),
    "vm_step_finish": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int64, C.c_void_p]),
    "vm_graph_launch": (C.c_int, [C.c_void_p, C.c_void_p]),
    "vm_last_error": (C.c_char_p, []),
    "vm_version": (C.c_char_p, []),
    "vm_ffma_peak": (C.c_int, [C.c_int, C.POINTER(C.c_float), C.c_void_p]),
}

EXPORTED = tuple(_SIGNATURES)

_lib = None


def load(path: Path | None = None) -> C.CDLL:
    """Load (once) and type the C ABI.  Raises if the library is absent."""
    global _lib
    if _lib is not None:
        return _lib
    p = Path(path) if path else Path(os.environ.get("VM_LIB") or LIB_PATH)  # VM_LIB: A/B builds (scripts)
    if not p.exists():
        raise RuntimeError(
            f"libvmap_b200.so not found at {p}; build it with `python -c "
            "'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")
    lib = C.CDLL(str(p))
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc == VM_OK:
        return
    msg = load().vm_last_error().decode(errors="replace")
    if rc == VM_ERR_SHAPE:
        raise ValueError(f"{what}: {msg}")
    if rc == VM_ERR_UNSUPPORTED:
        raise NotImplementedError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: CUDA error: {msg}")


def layout(n_layers: int, hidden: int, input_dim: int) -> VmLayout:
    arch = VmArch(n_layers, hidden, input_dim, 0)
    out = VmLayout()
    check(load().vm_model_layout(C.byref(arch), C.byref(out)), "vm_model_layout")
    return out


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None passes NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr() -> int:
    import torch
    return torch.cuda.current_stream().cuda_stream
