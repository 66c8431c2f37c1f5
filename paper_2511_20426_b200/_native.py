"""ctypes binding of ``libbcb200.so`` (the C-ABI declared in include/bcb200.h).

The library is built in-tree (``make -C paper_2511_20426_b200/csrc`` or
``__graft_entry__.build()``).  Every numeric entry point runs on the GPU;
there is deliberately no Python/CPU fallback -- if the library or a CUDA
device is missing the call raises :class:`DeviceError`.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .errors import ContractViolation, DeviceError, raise_for_status

# BC_LIB: a variant build of the same library (scripts/lib_variants.sh); default: the in-tree build
LIB_PATH = os.environ.get("BC_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libbcb200.so")
MAX_ENTRIES = 16
MAX_VIS = 32

_lock = threading.Lock()
_lib = None


class NoiseTask(C.Structure):
    _fields_ = [("key", C.c_uint64 * 2), ("counter", C.c_uint64 * 4),
                ("n", C.c_int64), ("out", C.c_void_p)]


class Batch(C.Structure):
    _fields_ = [("n_entries", C.c_int32), ("block_size", C.c_int32),
                ("block_index", C.c_int32 * MAX_ENTRIES),
                ("level", C.c_double * MAX_ENTRIES),
                ("slot", C.c_int32 * MAX_ENTRIES),
                ("n_vis", C.c_int32 * MAX_ENTRIES),
                ("vis_slot", (C.c_int32 * MAX_VIS) * MAX_ENTRIES)]


class ToyWeights(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("w_in", "w_cond", "w_level", "w_q", "w_k",
                                          "w_v", "w_o", "w_head")] + \
               [(n, C.c_int32) for n in ("layers", "heads", "dim", "cond_dim")]


class WanDims(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "layers", "heads", "head_dim", "ffn_dim", "text_len", "text_dim", "freq_dim",
        "latent_h", "latent_w", "block_size", "n_slots", "max_entries")]


WAN_PARAM_FIELDS = (
    "patch_w", "patch_b", "text_w1", "text_b1", "text_w2", "text_b2",
    "time_w1", "time_b1", "time_w2", "time_b2", "tproj_w", "tproj_b",
    "head_w", "head_b", "head_mod",
    "qkv_w", "qkv_b", "o_w", "o_b", "cq_w", "cq_b", "ckv_w", "ckv_b", "co_w", "co_b",
    "ffn1_w", "ffn1_b", "ffn2_w", "ffn2_b", "norm_q", "norm_k", "cnorm_q", "cnorm_k",
    "norm3_w", "norm3_b", "modulation")


class WanParams(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in WAN_PARAM_FIELDS]


class WanUpdate(C.Structure):
    _fields_ = [("post", C.c_int32 * MAX_ENTRIES),
                ("next_level", C.c_double * MAX_ENTRIES),
                ("latents", C.c_void_p * MAX_ENTRIES),
                ("eps", C.c_void_p * MAX_ENTRIES),
                ("out", C.c_void_p * MAX_ENTRIES)]


MAX_PEERS = 8


class WanPeers(C.Structure):
    _fields_ = [("n_peers", C.c_int32), ("my_rank", C.c_int32), ("n_ranks", C.c_int32),
                ("peer_arena", C.c_void_p * MAX_PEERS), ("peer_flags", C.c_void_p * MAX_PEERS),
                ("peer_done", C.c_void_p * MAX_PEERS), ("my_flags", C.c_void_p),
                ("my_done", C.c_void_p), ("counters", C.c_void_p),
                ("my_y", C.c_void_p), ("peer_y", C.c_void_p * MAX_PEERS),
                ("my_yready", C.c_void_p), ("peer_yready", C.c_void_p * MAX_PEERS)]


class WanDist(C.Structure):
    _fields_ = [("epoch", C.c_uint32), ("need", (C.c_uint32 * MAX_VIS) * MAX_ENTRIES),
                ("pmask", (C.c_uint8 * MAX_VIS) * MAX_ENTRIES),
                ("stage", C.c_int32), ("layer", C.c_int32), ("row0", C.c_int32), ("row1", C.c_int32)]


class VaeConvArgs(C.Structure):
    _fields_ = [("in_", C.c_void_p), ("w", C.c_void_p), ("bias", C.c_void_p)] + \
               [(n, C.c_int32) for n in ("H", "W", "n_frames", "frame0", "n_out_frames", "cin", "cout",
                                         "kt", "kh", "kw")] + \
               [(n, C.c_void_p) for n in ("res", "out32", "out16", "act", "gamma")] + \
               [("act_silu", C.c_int32), ("video", C.c_void_p), ("video_channels", C.c_int32),
                ("video_frame0", C.c_int32)]


VAE_MAX_FRAMES = 16


class VaeFrameMap(C.Structure):
    _fields_ = [("src", C.c_int32 * VAE_MAX_FRAMES), ("frame", C.c_int32 * VAE_MAX_FRAMES),
                ("chan", C.c_int32 * VAE_MAX_FRAMES)]


_SIGS = {
    "bc_last_error": (C.c_char_p, []),
    "bc_version": (C.c_char_p, []),
    "bc_noise_run": (C.c_int, [C.POINTER(NoiseTask), C.c_int, C.c_int, C.c_int]),
    "bc_philox4x64": (C.c_int, [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                C.POINTER(C.c_uint64)]),
    "bc_renoise_f64": (C.c_int, [C.c_void_p, C.c_void_p, C.c_double, C.c_void_p,
                                 C.c_int64, C.c_void_p, C.c_void_p]),
    "bc_renoise_f32": (C.c_int, [C.c_void_p, C.c_void_p, C.c_double, C.c_void_p,
                                 C.c_int64, C.c_void_p, C.c_void_p]),
    "bc_toy_forward": (C.c_int, [C.POINTER(ToyWeights), C.POINTER(Batch),
                                 C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                 C.c_void_p, C.c_int32, C.POINTER(C.c_void_p),
                                 C.c_void_p, C.c_void_p, C.c_void_p]),
    "bc_wan_workspace_bytes": (C.c_int64, [C.POINTER(WanDims)]),
    "bc_wan_create": (C.c_int, [C.POINTER(WanDims), C.POINTER(WanParams), C.c_void_p,
                                C.c_void_p, C.c_int64, C.POINTER(C.c_void_p)]),
    "bc_wan_destroy": (C.c_int, [C.c_void_p]),
    "bc_wan_set_graphs": (C.c_int, [C.c_int]),
    "bc_attention_set_balance": (C.c_int, [C.c_int]),
    "bc_attention_plan": (C.c_int, [C.POINTER(Batch), C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_int32,
                                    C.c_void_p, C.POINTER(C.c_int32)]),
    "bc_wan_set_text": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "bc_wan_step": (C.c_int, [C.c_void_p, C.POINTER(Batch), C.POINTER(WanUpdate),
                              C.c_void_p, C.c_void_p]),
    "bc_gemm_plan": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                               C.POINTER(C.c_int32)]),
    "bc_gemm_bf16": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                               C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_int32,
                               C.c_int32, C.c_void_p]),
    "bc_attention_paged": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                     C.c_int32, C.POINTER(Batch), C.c_int32, C.c_int32,
                                     C.c_void_p, C.c_void_p]),
    "bc_launch_count": (C.c_longlong, []),
    "bc_wan_set_peers": (C.c_int, [C.c_void_p, C.POINTER(WanPeers)]),
    "bc_wan_step_dist": (C.c_int, [C.c_void_p, C.POINTER(Batch), C.POINTER(WanUpdate),
                                   C.POINTER(WanDist), C.c_void_p, C.c_void_p]),
    "bc_wan_signal_done": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p]),
    "bc_ipc_malloc": (C.c_int, [C.c_int64, C.POINTER(C.c_void_p), C.c_char_p]),
    "bc_ipc_open": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "bc_ipc_close": (C.c_int, [C.c_void_p]),
    "bc_free": (C.c_int, [C.c_void_p]),
    "bc_memset_async": (C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_void_p]),
    "bc_copy_async": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "bc_stream_write_u32": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p]),
    "bc_stream_wait_geq_u32": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p]),
    "bc_vae_conv": (C.c_int, [C.POINTER(VaeConvArgs), C.c_void_p]),
    "bc_vae_prep": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
                    + [C.c_int32] * 6 + [C.c_void_p]),
    "bc_vae_upsample": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(VaeFrameMap), C.c_int32, C.c_int32,
                                  C.c_int32, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    "bc_vae_attn_gather": (C.c_int, [C.c_void_p] + [C.c_int32] * 5 + [C.c_void_p] * 4),
    "bc_vae_softmax": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_float,
                                 C.c_void_p]),
    "bc_vae_norm_act": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p] + [C.c_int32] * 6 + [C.c_void_p]),
    "bc_vae_attn_out": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p] + [C.c_int32] * 4
                        + [C.c_void_p]),
    "bc_profile_enable": (C.c_int, [C.c_int]),
    "bc_profile_collect": (C.c_int, [C.POINTER(C.c_double), C.POINTER(C.c_double),
                                     C.POINTER(C.c_double), C.POINTER(C.c_int64), C.c_int]),
}

PROFILE_CLASSES = ("self_attention", "cross_attention", "gemm", "bandwidth")


def profile_enable(on: bool) -> None:
    check(lib().bc_profile_enable(1 if on else 0), "bc_profile_enable")


def profile_collect() -> dict:
    """{class: (ms, flops, bytes, launches)} accumulated since the last call."""
    n = len(PROFILE_CLASSES)
    ms, fl, by = (C.c_double * n)(), (C.c_double * n)(), (C.c_double * n)()
    cnt = (C.c_int64 * n)()
    check(lib().bc_profile_collect(ms, fl, by, cnt, n), "bc_profile_collect")
    return {name: (ms[i], fl[i], by[i], cnt[i]) for i, name in enumerate(PROFILE_CLASSES)}


def launch_count() -> int:
    return int(lib().bc_launch_count())


def exported_symbols() -> list:
    """Every entry point declared in include/bcb200.h."""
    return sorted(_SIGS)


def lib():
    """Load (once) and return the native library."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise DeviceError(
                    f"{LIB_PATH} is missing: build it with "
                    f"`make -C paper_2511_20426_b200/csrc` (there is no CPU fallback)")
            handle = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def check(code: int, what: str) -> None:
    if code:
        raise_for_status(code, what, lib().bc_last_error().decode(errors="replace"))


# ---------------------------------------------------------------------------
# Noise
# ---------------------------------------------------------------------------

def run_noise_tasks(tasks, dtype: int, threads: int = 0) -> None:
    """tasks: iterable of (key0, key1, (c0, c1, c2, c3), out ndarray)."""
    tasks = list(tasks)
    if not tasks:
        return
    arr = (NoiseTask * len(tasks))()
    keep = []
    want = np.float64 if dtype == 0 else np.float32
    for t, (k0, k1, ctr, out) in zip(arr, tasks):
        if out.dtype != want or not out.flags.c_contiguous:
            raise ContractViolation("noise output must be a C-contiguous array of the dtype")
        t.key[0], t.key[1] = k0 & 0xFFFFFFFFFFFFFFFF, k1 & 0xFFFFFFFFFFFFFFFF
        for i in range(4):
            t.counter[i] = ctr[i] & 0xFFFFFFFFFFFFFFFF
        t.n = out.size
        t.out = out.ctypes.data
        keep.append(out)
    check(lib().bc_noise_run(arr, len(tasks), dtype, threads), "bc_noise_run")


def _block_tasks(seed, block, pass_index, frame0, size, out):
    return [(seed, 0, (block, pass_index, frame0 + i, 0), out[i]) for i in range(size)]


def noise_block_f64(seed, block, pass_index, frame0, size, dim, out) -> None:
    run_noise_tasks(_block_tasks(seed, block, pass_index, frame0, size, out), 0)


def noise_block_f32(seed, block, pass_index, frame0, size, dim, out) -> None:
    run_noise_tasks(_block_tasks(seed, block, pass_index, frame0, size, out), 1)


def philox4x64(key, counter) -> list:
    k = (C.c_uint64 * 2)(*[int(v) & 0xFFFFFFFFFFFFFFFF for v in key])
    c = (C.c_uint64 * 4)(*[int(v) & 0xFFFFFFFFFFFFFFFF for v in counter])
    o = (C.c_uint64 * 4)()
    check(lib().bc_philox4x64(k, c, o), "bc_philox4x64")
    return list(o)


# ---------------------------------------------------------------------------
# torch plumbing
# ---------------------------------------------------------------------------

def torch_mod():
    import torch
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the B200 path has no CPU fallback")
    return torch


def stream_ptr(stream=None) -> int:
    torch = torch_mod()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t) -> int:
    return int(t.data_ptr()) if t is not None else 0


def renoise(x0, eps, level: float):
    """Device renoise; host arrays are uploaded, computed, and copied back."""
    torch = torch_mod()
    host = not hasattr(x0, "is_cuda")
    if host:
        x0_d = torch.from_numpy(np.ascontiguousarray(x0)).cuda()
        eps_d = torch.from_numpy(np.ascontiguousarray(eps, dtype=np.asarray(x0).dtype)).cuda()
    else:
        x0_d, eps_d = x0.contiguous(), eps.contiguous().to(x0.dtype)
    out = torch.empty_like(x0_d)
    fn = {torch.float64: lib().bc_renoise_f64, torch.float32: lib().bc_renoise_f32}.get(x0_d.dtype)
    if fn is None:
        raise ContractViolation(f"renoise supports float32/float64, got {x0_d.dtype}")
    check(fn(ptr(x0_d), ptr(eps_d), level, ptr(out), x0_d.numel(), None, stream_ptr()),
          "bc_renoise")
    if host:
        return out.cpu().numpy()
    return out


def make_batch(block_size: int, blocks, levels, slots, vis_slots) -> Batch:
    n = len(blocks)
    if not 1 <= n <= MAX_ENTRIES:
        raise ContractViolation(f"batch width {n} outside [1, {MAX_ENTRIES}]")
    b = Batch()
    b.n_entries = n
    b.block_size = block_size
    for e in range(n):
        b.block_index[e] = int(blocks[e])
        b.level[e] = float(levels[e])
        b.slot[e] = int(slots[e])
        vis = vis_slots[e]
        if len(vis) > MAX_VIS:
            raise ContractViolation(f"{len(vis)} visible blocks exceed {MAX_VIS}")
        b.n_vis[e] = len(vis)
        for j, s in enumerate(vis):
            b.vis_slot[e][j] = int(s)
    return b
