"""Pauli strings and their packed 3-bit encoding — host side of the build's input.

Same encoding and API as palettecolor.pauli (/root/reference/pkg/src/palettecolor/pauli.py):
codes X=110, Y=101, Z=011, I=000, position p at stream bits [3p, 3p+3), stream split
little-endian into uint64 words (pauli.py:7-14, 54, 104-123).  Two strings anticommute iff
popcount(a & b) is odd (pauli.py:138-155, 258-268).

Differences that matter only for speed: ``PauliSet.from_strings`` packs all strings at once
with numpy instead of one Python loop per character (the reference spends ~24 s on 1M
strings), and the per-string ``encoded`` objects are created lazily.  The device side never
sees strings: it receives ``PauliSet.words`` and repacks them into x/z bit planes.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from functools import cached_property
from typing import Iterable, Sequence

import numpy as np

from .errors import (
    BadSymbolError,
    EmptyInputError,
    LengthMismatchError,
    MixedLengthError,
    OracleTooLargeError,
    SameVertexError,
)

PAULI_CODES = {"I": 0b000, "X": 0b110, "Y": 0b101, "Z": 0b011}
ORACLE_MAX_QUBITS = 12
_CODE_CHAR = {v: k for k, v in PAULI_CODES.items()}

_LUT = np.full(256, 255, dtype=np.uint8)
for _ch, _code in PAULI_CODES.items():
    _LUT[ord(_ch)] = _code


def words_per_string(num_qubits: int) -> int:
    return (3 * num_qubits + 63) // 64


@dataclass(frozen=True)
class EncodedPauli:
    """One packed string: little-endian uint64 words, ``nbits`` = 3 * qubits."""

    words: tuple
    nbits: int
    value: int = field(init=False, repr=False, compare=False)

    def __post_init__(self):
        total = 0
        for k, w in enumerate(self.words):
            if not 0 <= int(w) < (1 << 64):
                raise ValueError("encoded word out of 64-bit range")
            total |= int(w) << (64 * k)
        if total >> self.nbits:
            raise ValueError("trailing bits beyond nbits must be zero")
        object.__setattr__(self, "value", total)

    @property
    def num_qubits(self) -> int:
        return self.nbits // 3


def _codes(strings: Sequence[str]) -> np.ndarray:
    """(n, q) uint8 code matrix; raises on empty, ragged or bad symbols."""
    if not strings:
        raise EmptyInputError("no Pauli strings given")
    q = len(strings[0])
    if q == 0:
        raise EmptyInputError("empty Pauli string")
    for s in strings:
        if len(s) != q:
            raise MixedLengthError(f"string {s!r} has length {len(s)}, expected {q}")
    try:
        raw = "".join(strings).encode("ascii")
    except UnicodeEncodeError:
        bad = next(s for s in strings if not s.isascii())
        raise BadSymbolError(f"invalid Pauli symbol in {bad!r}") from None
    codes = _LUT[np.frombuffer(raw, dtype=np.uint8)].reshape(len(strings), q)
    if (codes == 255).any():
        r, c = map(int, np.argwhere(codes == 255)[0])
        raise BadSymbolError(f"invalid Pauli symbol {strings[r][c]!r} in {strings[r]!r}")
    return codes


def pack_codes(codes: np.ndarray) -> np.ndarray:
    """(n, q) codes -> (n, ceil(3q/64)) uint64 words, LSB-first 3-bit stream."""
    n, q = codes.shape
    nw = words_per_string(q)
    bits = np.zeros((n, nw * 64), dtype=np.uint8)
    stream = ((codes[:, :, None] >> np.arange(3, dtype=np.uint8)) & 1).reshape(n, 3 * q)
    bits[:, : 3 * q] = stream
    packed = np.packbits(bits, axis=1, bitorder="little")
    return np.ascontiguousarray(packed).view("<u8").astype(np.uint64).reshape(n, nw)


def encode(p: str) -> EncodedPauli:
    words = pack_codes(_codes([p]))[0]
    return EncodedPauli(words=tuple(int(w) for w in words), nbits=3 * len(p))


def decode(e: EncodedPauli) -> str:
    out = []
    for i in range(e.num_qubits):
        code = (e.value >> (3 * i)) & 7
        if code not in _CODE_CHAR:
            raise ValueError(f"invalid 3-bit code {code:03b} at position {i}")
        out.append(_CODE_CHAR[code])
    return "".join(out)


def anticommutes_fast(a: EncodedPauli, b: EncodedPauli) -> bool:
    if a.nbits != b.nbits:
        raise LengthMismatchError(f"encodings have {a.num_qubits} vs {b.num_qubits} qubits")
    return bool((a.value & b.value).bit_count() & 1)


def anticommutes_chars(a: str, b: str) -> bool:
    if len(a) != len(b):
        raise LengthMismatchError(f"strings have length {len(a)} vs {len(b)}")
    odd = 0
    for x, y in zip(a, b):
        odd ^= int(x != "I" and y != "I" and x != y)
    return bool(odd)


def anticommutes_oracle(a: str, b: str) -> bool:
    """Dense 2^N matrices: AB + BA == 0 (pauli.py:176-191)."""
    if len(a) != len(b):
        raise LengthMismatchError(f"strings have length {len(a)} vs {len(b)}")
    if len(a) > ORACLE_MAX_QUBITS:
        raise OracleTooLargeError(f"oracle capped at {ORACLE_MAX_QUBITS} qubits, got {len(a)}")
    _codes([a, b])
    mats = {
        "I": np.eye(2, dtype=np.complex128),
        "X": np.array([[0, 1], [1, 0]], dtype=np.complex128),
        "Y": np.array([[0, -1j], [1j, 0]], dtype=np.complex128),
        "Z": np.array([[1, 0], [0, -1]], dtype=np.complex128),
    }

    def dense(s):
        m = np.ones((1, 1), dtype=np.complex128)
        for ch in s:
            m = np.kron(m, mats[ch])
        return m

    ma, mb = dense(a), dense(b)
    return not np.any(ma @ mb + mb @ ma)


def complement_edge(a: EncodedPauli, b: EncodedPauli) -> bool:
    return not anticommutes_fast(a, b)


class PauliSet:
    """Indexed same-length Pauli strings with their packed words (pauli.py:206-255)."""

    def __init__(self, strings: list, words: np.ndarray, encoded: list | None = None):
        self.strings = strings
        self.words = words
        self.words.setflags(write=False)
        if encoded is not None:
            self.__dict__["encoded"] = encoded

    @property
    def n(self) -> int:
        return len(self.strings)

    @property
    def num_qubits(self) -> int:
        return len(self.strings[0])

    @cached_property
    def encoded(self) -> list:
        nb = 3 * self.num_qubits
        return [EncodedPauli(tuple(int(w) for w in row), nb) for row in self.words]

    @classmethod
    def from_strings(cls, strings: Iterable[str]) -> "PauliSet":
        strings = list(strings)
        return cls(strings, pack_codes(_codes(strings)))

    def anticommutes(self, i: int, j: int) -> bool:
        acc = np.bitwise_xor.reduce(self.words[i] & self.words[j]) if self.words.shape[1] else 0
        return bool(int(acc).bit_count() & 1)

    def complement_edge(self, i: int, j: int) -> bool:
        if i == j:
            raise SameVertexError(f"self-pair query on vertex {i}")
        return not self.anticommutes(i, j)


def anticommute_pairs(words: np.ndarray, i, j) -> np.ndarray:
    """Host reference of the predicate over index arrays (pauli.py:258-268)."""
    acc = np.zeros(np.shape(i), dtype=np.uint64)
    for w in range(words.shape[1]):
        acc ^= words[i, w] & words[j, w]
    return (np.bitwise_count(acc) & 1).astype(bool)


def parse_pauli_text(text) -> PauliSet:
    """'string' or 'coeff string' per line; '#' comments; blanks skipped (pauli.py:271-312)."""
    lines = text.splitlines() if isinstance(text, str) else list(text)
    strings = []
    for lineno, raw in enumerate(lines, start=1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        parts = line.split()
        if len(parts) == 2:
            try:
                float(parts[0])
            except ValueError:
                raise BadSymbolError(
                    f"line {lineno}: expected a real coefficient, got {parts[0]!r}"
                ) from None
            s = parts[1]
        elif len(parts) == 1:
            s = parts[0]
        else:
            raise BadSymbolError(f"line {lineno}: expected 'string' or 'coeff string', got {line!r}")
        s = s.upper()
        bad = [ch for ch in s if ch not in PAULI_CODES]
        if bad:
            raise BadSymbolError(f"line {lineno}: invalid Pauli symbol {bad[0]!r} in {s!r}")
        strings.append(s)
    if not strings:
        raise EmptyInputError("no Pauli strings in input")
    return PauliSet.from_strings(strings)


def random_pauli_strings(n: int, num_qubits: int, seed: int = 0, exclude_identity: bool = False) -> list:
    """The reference generator (generate.py:18-32): PCG64 seeded by [seed, n, q]."""
    from .errors import BadParamsError

    if n < 1 or num_qubits < 1:
        raise BadParamsError("need n >= 1 and num_qubits >= 1")
    gen = np.random.default_rng(np.random.SeedSequence([seed, n, num_qubits]))
    symbols = np.frombuffer(b"IXYZ", dtype=np.uint8)
    out: list = []
    while len(out) < n:
        draw = gen.integers(0, 4, size=(n - len(out), num_qubits))
        if exclude_identity:
            draw = draw[draw.any(axis=1)]
        rows = symbols[draw]
        blob = rows.tobytes().decode("ascii")
        out.extend(blob[k * num_qubits:(k + 1) * num_qubits] for k in range(rows.shape[0]))
    return out


def pauli_file_text(strings: list) -> str:
    return "\n".join(strings) + "\n"
