"""B200-native batched RNS-Montgomery RSA (arXiv:1305.3699, MR-MOD / MR-RSA hot path).

Thin ctypes binding of ``libmr_rns.so`` (C ABI: ``include/mr_rns.h``).  Same entry-point names as
the C header; argument marshalling only — every step of the path runs in the CUDA kernels of
``csrc/``.  There is no CPU fallback: if the shared library is missing or no CUDA device is usable,
calls raise.

Device buffers are ``torch`` CUDA tensors of dtype int32 whose bits are the uint32 limbs
(little-endian, row-major ``[count][limbs]``); the current torch stream of the tensor's device is
used unless ``stream`` is given.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

__all__ = [
    "lib", "MrError", "MR_OK", "MR_ERR_RANGE", "MR_COMPOSITE", "MR_PROBABLY_PRIME", "MR_FACTOR",
    "mr_rns_ctx_create", "mr_rns_ctx_destroy", "mr_rns_ctx_info", "mr_rns_supported_k",
    "mr_modexp_batch", "mr_rsa_encrypt_batch", "mr_rsa_priv_create", "mr_rsa_priv_destroy",
    "mr_rsa_decrypt_batch", "mr_miller_rabin_batch", "mr_rsa_keygen_batch", "mr_rsa_keygen_batch_drbg", "mr_strerror",
    "RnsContext", "RsaPrivateKey", "Drbg", "fips_health", "limbs_of", "ints_to_limbs", "limbs_to_ints",
]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MR_RNS_LIB") or os.path.join(HERE, "libmr_rns.so")   # override: A/B builds

MR_OK, MR_ERR_ARG, MR_ERR_EVEN_MODULUS, MR_ERR_NOT_COPRIME = 0, 1, 2, 3
MR_ERR_CAPACITY, MR_ERR_RANGE, MR_ERR_CUDA, MR_ERR_NOMEM = 4, 5, 6, 7
MR_COMPOSITE, MR_PROBABLY_PRIME, MR_FACTOR = 0, 1, 2

EXPORTS = (
    "mr_rns_ctx_create", "mr_rns_ctx_destroy", "mr_rns_ctx_info", "mr_rns_supported_k", "mr_modexp_batch",
    "mr_rsa_encrypt_batch", "mr_rsa_priv_create", "mr_rsa_priv_destroy", "mr_rsa_decrypt_batch",
    "mr_miller_rabin_batch", "mr_rsa_keygen_batch", "mr_strerror",
    "mr_drbg_create", "mr_drbg_generate", "mr_drbg_destroy", "mr_fips_health_batch", "mr_rsa_keygen_batch_drbg",
)


class MrError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        self.code = code
        super().__init__(f"{what}: {mr_strerror(code)} (code {code})" if what else mr_strerror(code))


_lib = None


def lib() -> ctypes.CDLL:
    """Load libmr_rns.so (raises if it has not been built — there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1305_3699_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        vp, sz, i32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
        ip = ctypes.POINTER(ctypes.c_int)
        up = ctypes.POINTER(ctypes.c_uint32)
        L.mr_rns_ctx_create.argtypes = [ctypes.POINTER(vp), up, sz, i32, i32]
        L.mr_rns_ctx_destroy.argtypes = [vp]
        L.mr_rns_ctx_destroy.restype = None
        L.mr_rns_ctx_info.argtypes = [vp, ip, ctypes.POINTER(sz), ip, ip, ip]
        L.mr_rns_supported_k.argtypes = [ip, i32]
        L.mr_modexp_batch.argtypes = [vp, vp, vp, sz, up, sz, vp, vp]
        L.mr_rsa_encrypt_batch.argtypes = [vp, up, sz, vp, vp, sz, vp, vp]
        L.mr_rsa_priv_create.argtypes = [ctypes.POINTER(vp), up, up, sz, up, up, up, i32, i32]
        L.mr_rsa_priv_destroy.argtypes = [vp]
        L.mr_rsa_priv_destroy.restype = None
        L.mr_rsa_decrypt_batch.argtypes = [vp, vp, vp, sz, vp, vp]
        L.mr_miller_rabin_batch.argtypes = [vp, sz, sz, vp, i32, i32, vp, vp, vp, i32, vp]
        L.mr_rsa_keygen_batch.argtypes = [sz, i32, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64, i32] + \
            [vp] * 7 + [i32, vp]
        L.mr_rsa_keygen_batch_drbg.argtypes = [vp, sz, i32, ctypes.c_uint32, i32] + [vp] * 7 + [i32, vp]
        L.mr_strerror.argtypes = [i32]
        L.mr_strerror.restype = ctypes.c_char_p
        cp = ctypes.c_char_p
        L.mr_drbg_create.argtypes = [ctypes.POINTER(vp), cp, sz, cp, sz, cp, sz, ctypes.c_uint32, i32]
        L.mr_drbg_generate.argtypes = [vp, vp, sz, vp]
        L.mr_drbg_destroy.argtypes = [vp]
        L.mr_drbg_destroy.restype = None
        L.mr_fips_health_batch.argtypes = [vp, sz, vp, vp]
        for name in EXPORTS:
            if name not in ("mr_rns_ctx_destroy", "mr_rsa_priv_destroy", "mr_strerror", "mr_drbg_destroy"):
                getattr(L, name).restype = i32
        _lib = L
    return _lib


# ------------------------------------------------------------------ marshalling helpers (I/O only)

def limbs_of(x: int, n: int) -> np.ndarray:
    """little-endian uint32 limbs of a non-negative int, fixed width n."""
    if x < 0 or x >> (32 * n):
        raise ValueError("value does not fit in %d limbs" % n)
    return np.frombuffer(x.to_bytes(4 * n, "little"), dtype=np.uint32).copy()


def ints_to_limbs(values: Sequence[int], n: int) -> np.ndarray:
    out = np.zeros((len(values), n), dtype=np.uint32)
    for i, v in enumerate(values):
        out[i] = limbs_of(int(v), n)
    return out


def limbs_to_ints(a) -> list[int]:
    a = np.ascontiguousarray(_to_numpy(a), dtype=np.uint32)
    return [int.from_bytes(row.tobytes(), "little") for row in a]


def _to_numpy(a):
    try:
        import torch
        if isinstance(a, torch.Tensor):
            return a.detach().cpu().numpy().view(np.uint32)
    except ImportError:
        pass
    return np.asarray(a)


def _hp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


def _dptr(t) -> Optional[int]:
    if t is None:
        return None
    if not t.is_cuda:
        raise MrError(MR_ERR_ARG, "device buffers must be CUDA tensors (no CPU fallback)")
    if not t.is_contiguous():
        raise MrError(MR_ERR_ARG, "device buffers must be contiguous")
    return t.data_ptr()


def _arg(t, what: str, itemsize: int, numel: int, width: Optional[int] = None, device: Optional[int] = None):
    """Validate a device buffer before its pointer crosses the C ABI (which cannot see sizes): a CUDA,
    contiguous tensor of `itemsize`-byte elements with at least `numel` of them; `width` given: 2-D with
    shape[1] == width; `device` given: on that CUDA ordinal.  Returns the pointer, or None for None."""
    if t is None:
        return None
    p = _dptr(t)
    if t.dtype.itemsize != itemsize:
        raise MrError(MR_ERR_ARG, f"{what}: expected {itemsize}-byte elements, got {t.dtype}")
    if width is not None and (t.dim() != 2 or t.shape[1] != width):
        raise MrError(MR_ERR_ARG, f"{what}: expected shape [count][{width}], got {tuple(t.shape)}")
    if t.numel() < numel:
        raise MrError(MR_ERR_ARG, f"{what}: {t.numel()} elements, the call needs {numel}")
    if device is not None and t.device.index != device:
        raise MrError(MR_ERR_ARG, f"{what}: tensor on cuda:{t.device.index}, context on cuda:{device}")
    return p


def _stream(t, stream) -> Optional[int]:
    if stream is not None:
        return getattr(stream, "cuda_stream", stream)
    import torch
    return torch.cuda.current_stream(t.device).cuda_stream


def _check(rc: int, what: str) -> None:
    if rc != MR_OK:
        raise MrError(rc, what)


# ------------------------------------------------------------------ C ABI, same names

def mr_strerror(code: int) -> str:
    return lib().mr_strerror(code).decode()


def mr_rns_supported_k() -> list[int]:
    buf = (ctypes.c_int * 64)()
    n = lib().mr_rns_supported_k(buf, 64)
    return list(buf[:n])


def mr_rns_ctx_create(modulus: int, limbs: int, k: int = 0, device: int = 0) -> ctypes.c_void_p:
    m = limbs_of(modulus, limbs)
    h = ctypes.c_void_p()
    _check(lib().mr_rns_ctx_create(ctypes.byref(h), _hp(m), limbs, k, device), "mr_rns_ctx_create")
    _devices[h.value] = (limbs, device)
    return h


def mr_rns_ctx_destroy(ctx) -> None:
    _devices.pop(getattr(ctx, "value", ctx), None)
    lib().mr_rns_ctx_destroy(ctx)


def mr_rns_ctx_info(ctx) -> dict:
    k, maxb, bits, cap = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    limbs = ctypes.c_size_t()
    _check(lib().mr_rns_ctx_info(ctx, ctypes.byref(k), ctypes.byref(limbs), ctypes.byref(maxb), ctypes.byref(bits),
                                 ctypes.byref(cap)), "mr_rns_ctx_info")
    return {"k": k.value, "limbs": limbs.value, "max_modulus_bits": maxb.value, "modulus_bits": bits.value,
            "paper_cap_bits": cap.value}


_devices: dict = {}   # handle value -> (limbs per row, device) of contexts and private keys made here


def _geom(handle, what: str):
    g = _devices.get(getattr(handle, "value", handle))
    if g is None:
        raise MrError(MR_ERR_ARG, f"{what}: unknown handle (create it with this module)")
    return g


def mr_modexp_batch(ctx, d_x, d_y, count: int, exp: int, d_status=None, stream=None) -> None:
    limbs, dev = _geom(ctx, "mr_modexp_batch")
    e = limbs_of(exp, max(1, (exp.bit_length() + 31) // 32))
    _check(lib().mr_modexp_batch(ctx, _arg(d_x, "d_x", 4, count * limbs, limbs, dev),
                                 _arg(d_y, "d_y", 4, count * limbs, limbs, dev), count, _hp(e), len(e) if exp else 0,
                                 _arg(d_status, "d_status", 4, count, None, dev), _stream(d_x, stream)),
           "mr_modexp_batch")


def mr_rsa_encrypt_batch(ctx, e: int, d_m, d_c, count: int, d_status=None, stream=None) -> None:
    limbs, dev = _geom(ctx, "mr_rsa_encrypt_batch")
    el = limbs_of(e, max(1, (e.bit_length() + 31) // 32))
    _check(lib().mr_rsa_encrypt_batch(ctx, _hp(el), len(el) if e else 0, _arg(d_m, "d_m", 4, count * limbs, limbs, dev),
                                      _arg(d_c, "d_c", 4, count * limbs, limbs, dev), count,
                                      _arg(d_status, "d_status", 4, count, None, dev), _stream(d_m, stream)),
           "mr_rsa_encrypt_batch")


def mr_rsa_priv_create(p: int, q: int, half_limbs: int, d_p: int, d_q: int, q_inv: int, k_half: int = 0,
                       device: int = 0) -> ctypes.c_void_p:
    arrs = [limbs_of(v, half_limbs) for v in (p, q, d_p, d_q, q_inv)]
    h = ctypes.c_void_p()
    _check(lib().mr_rsa_priv_create(ctypes.byref(h), *[_hp(a) for a in arrs[:2]], half_limbs,
                                    *[_hp(a) for a in arrs[2:]], k_half, device), "mr_rsa_priv_create")
    _devices[h.value] = (2 * half_limbs, device)
    return h


def mr_rsa_priv_destroy(priv) -> None:
    _devices.pop(getattr(priv, "value", priv), None)
    lib().mr_rsa_priv_destroy(priv)


def mr_rsa_decrypt_batch(priv, d_c, d_m, count: int, d_status=None, stream=None) -> None:
    limbs, dev = _geom(priv, "mr_rsa_decrypt_batch")
    _check(lib().mr_rsa_decrypt_batch(priv, _arg(d_c, "d_c", 4, count * limbs, limbs, dev),
                                      _arg(d_m, "d_m", 4, count * limbs, limbs, dev), count,
                                      _arg(d_status, "d_status", 4, count, None, dev), _stream(d_c, stream)),
           "mr_rsa_decrypt_batch")


def mr_miller_rabin_batch(d_n, limbs: int, count: int, d_bases, rounds: int, d_verdict, d_witness=None,
                          d_status=None, k: int = 0, device: int = 0, stream=None) -> None:
    if rounds < 1:
        raise MrError(MR_ERR_ARG, "mr_miller_rabin_batch: rounds >= 1")
    _check(lib().mr_miller_rabin_batch(_arg(d_n, "d_n", 4, count * limbs, limbs, device), limbs, count,
                                       _arg(d_bases, "d_bases", 4, count * rounds * limbs, None, device), rounds, k,
                                       _arg(d_verdict, "d_verdict", 1, count, None, device),
                                       _arg(d_witness, "d_witness", 2, count, None, device),
                                       _arg(d_status, "d_status", 4, count, None, device), device,
                                       _stream(d_n, stream)),
           "mr_miller_rabin_batch")


def mr_rsa_keygen_batch(count: int, bits: int, e: int, seed: int, rounds: int, d_n, d_p, d_q, d_d, d_dp, d_dq, d_qinv,
                        first_key: int = 0, device: int = 0, stream=None) -> None:
    """RSA key generation on the GPU (include/mr_rns.h).  Outputs are device uint32/int32 tensors of
    [count][bits/32] (n, d) and [count][bits/64] (p, q, dp, dq, qinv) limbs."""
    L, H = bits // 32, bits // 64
    outs = [_arg(t, nm, 4, count * w, w, device) for t, nm, w in
            ((d_n, "d_n", L), (d_p, "d_p", H), (d_q, "d_q", H), (d_d, "d_d", L), (d_dp, "d_dp", H), (d_dq, "d_dq", H),
             (d_qinv, "d_qinv", H))]
    _check(lib().mr_rsa_keygen_batch(count, bits, e, seed, first_key, rounds, *outs, device,
                                     _stream(d_n, stream)), "mr_rsa_keygen_batch")


def mr_rsa_keygen_batch_drbg(rng: "Drbg", count: int, bits: int, e: int, rounds: int, d_n, d_p, d_q, d_d, d_dp, d_dq,
                             d_qinv, device: int = 0, stream=None) -> None:
    """RSA key generation with every random choice (search starts, Miller-Rabin bases) drawn from the
    GPU Hash_DRBG `rng` (include/mr_rns.h).  Same outputs as mr_rsa_keygen_batch."""
    L, H = bits // 32, bits // 64
    outs = [_arg(t, nm, 4, count * w, w, device) for t, nm, w in
            ((d_n, "d_n", L), (d_p, "d_p", H), (d_q, "d_q", H), (d_d, "d_d", L), (d_dp, "d_dp", H), (d_dq, "d_dq", H),
             (d_qinv, "d_qinv", H))]
    _check(lib().mr_rsa_keygen_batch_drbg(rng.handle, count, bits, e, rounds, *outs, device, _stream(d_n, stream)),
           "mr_rsa_keygen_batch_drbg")


# ------------------------------------------------------------------ RAII conveniences

class RnsContext:
    """Modulus N with its device-resident RNS constants (mr_rns_ctx)."""

    def __init__(self, modulus: int, limbs: Optional[int] = None, k: int = 0, device: int = 0):
        self.modulus = modulus
        self.limbs = limbs or max(1, (modulus.bit_length() + 31) // 32)
        self.device = device
        self.handle = mr_rns_ctx_create(modulus, self.limbs, k, device)
        self.info = mr_rns_ctx_info(self.handle)
        self.k = self.info["k"]

    def modexp(self, d_x, d_y, exp: int, d_status=None, stream=None, count: Optional[int] = None) -> None:
        mr_modexp_batch(self.handle, d_x, d_y, d_x.shape[0] if count is None else count, exp, d_status, stream)

    def encrypt(self, d_m, d_c, e: int, d_status=None, stream=None) -> None:
        mr_rsa_encrypt_batch(self.handle, e, d_m, d_c, d_m.shape[0], d_status, stream)

    def close(self) -> None:
        if getattr(self, "handle", None):
            mr_rns_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class RsaPrivateKey:
    """RSA private key held for CRT decryption (mr_rsa_priv)."""

    def __init__(self, p: int, q: int, dp: int, dq: int, qinv: int, half_limbs: Optional[int] = None,
                 k_half: int = 0, device: int = 0):
        """(p, q, dp = d mod (p-1), dq = d mod (q-1), qinv = q^-1 mod p): the PKCS#1 CRT key fields."""
        self.half = half_limbs or max((p.bit_length() + 31) // 32, (q.bit_length() + 31) // 32)
        self.limbs = 2 * self.half
        self.device = device
        self.handle = mr_rsa_priv_create(p, q, self.half, dp, dq, qinv, k_half, device)

    def decrypt(self, d_c, d_m, d_status=None, stream=None) -> None:
        mr_rsa_decrypt_batch(self.handle, d_c, d_m, d_c.shape[0], d_status, stream)

    def close(self) -> None:
        if getattr(self, "handle", None):
            mr_rsa_priv_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------ DRBG + FIPS 140-2 health tests (§8(f) row 4)

class Drbg:
    """`streams` independent Hash_DRBG (SHA-256, SP 800-90A) instances on the GPU (mr_drbg)."""

    def __init__(self, entropy: bytes, nonce: bytes, pers: bytes = b"", streams: int = 1, device: int = 0):
        h = ctypes.c_void_p()
        _check(lib().mr_drbg_create(ctypes.byref(h), entropy, len(entropy), nonce, len(nonce), pers, len(pers),
                                    streams, device), "mr_drbg_create")
        self.handle, self.streams, self.device = h, streams, device

    def generate(self, d_out, nbytes: int, stream=None) -> None:
        """one generate request of every stream into d_out (CUDA uint8 tensor [streams][nbytes])."""
        if d_out is not None and (d_out.dtype.itemsize != 1 or d_out.numel() != self.streams * nbytes):
            raise MrError(MR_ERR_ARG, "d_out must be a uint8 tensor of streams * nbytes bytes")
        ptr = _dptr(d_out) if nbytes else None
        st = _stream(d_out, stream) if d_out is not None else stream
        _check(lib().mr_drbg_generate(self.handle, ptr, nbytes, st), "mr_drbg_generate")

    def close(self) -> None:
        if getattr(self, "handle", None):
            lib().mr_drbg_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def fips_health(d_blocks, d_stats, stream=None) -> None:
    """FIPS 140-2 tests of d_blocks (CUDA uint8 [n][2500]) into d_stats (CUDA int32 [n][16])."""
    n = d_blocks.shape[0]
    _check(lib().mr_fips_health_batch(_arg(d_blocks, "d_blocks", 1, n * 2500, 2500),
                                      n, _arg(d_stats, "d_stats", 4, n * 16), _stream(d_blocks, stream)),
           "mr_fips_health_batch")
