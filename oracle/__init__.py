"""ctypes binding of the CPU oracle (``oracle/oracle.c``).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product path
(``paper_1305_3699_b200``) never imports it, and the two share no code.

The oracle computes the plain definitions of what the paper's RNS/Montgomery path (PAPER.md:38-56,
§3.1-§3.3) reaches exactly: ``x^E mod N`` (square-and-multiply), Garner CRT decryption,
Miller-Rabin with explicit bases, all on positional radix-2^32 bignums.  See the header of
``oracle.c`` for the step list and the citations; DESIGN.md "Oracle" for the pins.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Iterable, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

COMPOSITE, PROBABLY_PRIME, FACTOR, BAD_INPUT = 0, 1, 2, -1


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (plain gcc -O2, pthreads)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread", "-Wall", "-Wno-unused-variable",
             "-o", _LIB, _SRC])
    return _LIB


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB)
        P = ctypes.POINTER(ctypes.c_uint32)
        I = ctypes.c_int
        IP = ctypes.POINTER(ctypes.c_int)
        sig = {
            "orc_cmp": (I, [P, I, P, I]),
            "orc_add": (I, [P, P, I, P, I]),
            "orc_sub": (I, [P, P, I, P, I]),
            "orc_mul": (I, [P, P, I, P, I]),
            "orc_divmod": (I, [P, IP, P, IP, P, I, P, I]),
            "orc_divmod_bitwise": (I, [P, IP, P, IP, P, I, P, I]),
            "orc_modexp": (I, [P, P, I, P, I, P, I]),
            "orc_modinv": (I, [P, P, I, P, I]),
            "orc_crt_decrypt": (I, [P, P, P, P, P, P, P, I]),
            "orc_small_primes": (I, [P, I]),
            "orc_base_primes": (I, [P, I]),
            "orc_miller_rabin": (I, [P, I, P, I, P, I, IP]),
            "orc_next_prime": (I, [P, P, I, I, I]),
            "orc_modexp_batch": (I, [P, I, I, P, I, P, I, P, I]),
            "orc_crt_decrypt_batch": (I, [P, I, P, P, P, P, P, I, P, I]),
            "orc_miller_rabin_batch": (I, [P, I, I, P, I, P, I, IP, IP, I]),
        }
        for name, (res, args) in sig.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


# ---------------------------------------------------------------- conversions (I/O only)

def limbs_of(x: int, n: int | None = None) -> np.ndarray:
    """little-endian uint32 limbs of a non-negative int (O1); n = fixed width or minimal."""
    if x < 0:
        raise ValueError("negative")
    if n is None:
        n = max(1, (x.bit_length() + 31) // 32)
    if x >> (32 * n):
        raise ValueError("does not fit")
    return np.frombuffer(x.to_bytes(4 * n, "little"), dtype=np.uint32).copy()


def int_of(a: np.ndarray) -> int:
    return int.from_bytes(np.ascontiguousarray(a, dtype=np.uint32).tobytes(), "little")


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


def _buf(n: int) -> np.ndarray:
    return np.zeros(max(n, 1), dtype=np.uint32)


# ---------------------------------------------------------------- scalar API on Python ints

def cmp(a: int, b: int) -> int:
    A, B = limbs_of(a), limbs_of(b)
    return lib().orc_cmp(_p(A), len(A), _p(B), len(B))


def add(a: int, b: int) -> int:
    A, B = limbs_of(a), limbs_of(b)
    R = _buf(max(len(A), len(B)) + 1)
    n = lib().orc_add(_p(R), _p(A), len(A), _p(B), len(B))
    return int_of(R[:n])


def sub(a: int, b: int) -> int:
    A, B = limbs_of(a), limbs_of(b)
    R = _buf(len(A))
    n = lib().orc_sub(_p(R), _p(A), len(A), _p(B), len(B))
    if n < 0:
        raise ValueError("underflow: a < b")
    return int_of(R[:n])


def mul(a: int, b: int) -> int:
    A, B = limbs_of(a), limbs_of(b)
    R = _buf(len(A) + len(B))
    n = lib().orc_mul(_p(R), _p(A), len(A), _p(B), len(B))
    return int_of(R[:n])


def _divmod(fn, a: int, m: int):
    A, M = limbs_of(a), limbs_of(m)
    Q = _buf(len(A) + 1)
    R = _buf(len(M))
    nq, nr = ctypes.c_int(0), ctypes.c_int(0)
    rc = fn(_p(Q), ctypes.byref(nq), _p(R), ctypes.byref(nr), _p(A), len(A), _p(M), len(M))
    if rc != 0:
        raise ZeroDivisionError("division by zero")
    return int_of(Q[: nq.value]), int_of(R[: nr.value])


def divmod_knuth(a: int, m: int):
    """Knuth Algorithm D (O4)."""
    return _divmod(lib().orc_divmod, a, m)


def divmod_bitwise(a: int, m: int):
    """Independent shift-subtract long division (pin for O4)."""
    return _divmod(lib().orc_divmod_bitwise, a, m)


def modexp(x: int, e: int, n: int) -> int:
    """x^e mod n by left-to-right binary square-and-multiply (O5)."""
    X, E, N = limbs_of(x), limbs_of(e), limbs_of(n)
    Y = _buf(len(N))
    r = lib().orc_modexp(_p(Y), _p(X), len(X), _p(E), len(E), _p(N), len(N))
    if r < 0:
        raise ZeroDivisionError("modulus 0")
    return int_of(Y[:r])


def modinv(a: int, m: int) -> int:
    """a^-1 mod m by extended Euclid (O6); raises if gcd(a, m) != 1."""
    A, M = limbs_of(a), limbs_of(m)
    R = _buf(len(M))
    n = lib().orc_modinv(_p(R), _p(A), len(A), _p(M), len(M))
    if n < 0:
        raise ValueError("not invertible")
    return int_of(R[:n])


def crt_decrypt(c: int, p: int, q: int, dp: int, dq: int, qinv: int, nh: int) -> int:
    """Garner CRT decryption (O7); nh = limbs per prime, c and the result have 2 nh limbs."""
    C = limbs_of(c, 2 * nh)
    args = [limbs_of(v, nh) for v in (p, q, dp, dq, qinv)]
    M = _buf(2 * nh)
    lib().orc_crt_decrypt(_p(M), _p(C), *[_p(a) for a in args], nh)
    return int_of(M)


def small_primes(count: int) -> list[int]:
    """the first `count` primes by the sieve of Eratosthenes (O9)."""
    out = _buf(count)
    n = lib().orc_small_primes(_p(out), count)
    return [int(v) for v in out[:n]]


def base_primes(two_k: int) -> list[int]:
    """the 2k largest primes below 2^32 (only those = 3 mod 4 when 2k <= 130), descending (reading R1),
    derived by the oracle itself."""
    out = _buf(two_k)
    n = lib().orc_base_primes(_p(out), two_k)
    return [int(v) for v in out[:n]]


def miller_rabin(n: int, bases: Sequence[int], factor_primes: Sequence[int] = ()) -> tuple[int, int]:
    """(verdict, witness round) per HAC 4.24 with explicit bases (O8)."""
    nn = max(1, (n.bit_length() + 31) // 32)
    N = limbs_of(n, nn)
    B = np.concatenate([limbs_of(b, nn) for b in bases]) if len(bases) else _buf(nn)
    FP = np.array(list(factor_primes) or [0], dtype=np.uint32)
    w = ctypes.c_int(-1)
    v = lib().orc_miller_rabin(_p(N), nn, _p(B), len(bases), _p(FP), len(factor_primes), ctypes.byref(w))
    return v, w.value


def next_prime(start: int, nlimbs: int, rounds: int = 64, max_steps: int = 1 << 20) -> int:
    """first probable prime >= start (odd), trial division + MR with bases 2,3,5,... (O10)."""
    S = limbs_of(start, nlimbs)
    P = _buf(nlimbs)
    r = lib().orc_next_prime(_p(P), _p(S), nlimbs, rounds, max_steps)
    if r < 0:
        raise RuntimeError("no prime found")
    return int_of(P)


# ---------------------------------------------------------------- threaded batch API on limb arrays

def modexp_batch(x: np.ndarray, e: int, n: int, threads: int = 1) -> np.ndarray:
    """x: [count][L] uint32; returns [count][nn] of x_i^e mod n (O5 + O12)."""
    x = np.ascontiguousarray(x, dtype=np.uint32)
    count, lx = x.shape
    E, N = limbs_of(e), limbs_of(n)
    y = np.zeros((count, len(N)), dtype=np.uint32)
    lib().orc_modexp_batch(_p(x), lx, count, _p(E), len(E), _p(N), len(N), _p(y), threads)
    return y


def crt_decrypt_batch(c: np.ndarray, p: int, q: int, dp: int, dq: int, qinv: int, nh: int,
                      threads: int = 1) -> np.ndarray:
    """c: [count][2 nh] uint32; returns [count][2 nh] (O7 + O12)."""
    c = np.ascontiguousarray(c, dtype=np.uint32)
    count = c.shape[0]
    args = [limbs_of(v, nh) for v in (p, q, dp, dq, qinv)]
    m = np.zeros((count, 2 * nh), dtype=np.uint32)
    lib().orc_crt_decrypt_batch(_p(c), count, *[_p(a) for a in args], nh, _p(m), threads)
    return m


def miller_rabin_batch(n: np.ndarray, bases: np.ndarray, factor_primes: Iterable[int] = (),
                       threads: int = 1) -> tuple[np.ndarray, np.ndarray]:
    """n: [count][nn], bases: [count][rounds][nn]; returns (verdict int32[count], witness int32[count])."""
    n = np.ascontiguousarray(n, dtype=np.uint32)
    bases = np.ascontiguousarray(bases, dtype=np.uint32)
    count, nn = n.shape
    rounds = bases.shape[1]
    fp = np.array(list(factor_primes) or [0], dtype=np.uint32)
    nfp = 0 if (len(fp) == 1 and fp[0] == 0) else len(fp)
    verdict = np.zeros(count, dtype=np.int32)
    witness = np.zeros(count, dtype=np.int32)
    IP = ctypes.POINTER(ctypes.c_int)
    lib().orc_miller_rabin_batch(_p(n), nn, count, _p(bases), rounds, _p(fp), nfp,
                                 verdict.ctypes.data_as(IP), witness.ctypes.data_as(IP), threads)
    return verdict, witness
