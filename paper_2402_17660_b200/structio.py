"""Structures and weights in and out: extended-XYZ text and the reference's
little-endian array container.

* ``load_structure(path) -> (positions, species)`` and ``load_extxyz(path) -> [Frame, ...]`` read
  what ``nnpkit.data`` reads (data.py:89-200): per frame an atom-count line, a comment line whose
  ``key=value`` tokens must include ``energy=`` (``load_structure`` does not need it), and one line
  per atom ``symbol-or-Z x y z [fx fy fz]``; errors name the offending line.
* ``write_extxyz(path, frames)`` writes the same dialect (data.py:203-225), ``repr`` floats, so a
  round trip is exact.
* ``save_weights / load_weights``: a TensorNet parameter set in the reference's array encoding
  (data.py ``_write_array``: u16 name length + UTF-8 name, u8 dtype code 0 = f64 / 1 = i64, u8 rank,
  u64 shape entries, raw little-endian data) behind a ``TNW1`` magic and a JSON header holding the
  ``TNConfig``.  The reference's own ``MDKC`` checkpoints hold the weights of its invariant
  ``GraphPotential``, not of a TensorNet, so they are refused with a clear error.
"""

from __future__ import annotations

import json
import shlex
import struct
from dataclasses import asdict, dataclass
from pathlib import Path
from typing import Dict, List, Optional, Tuple, Union

import numpy as np

from .errors import DataError, ParseError, ValidationError

_SYMBOLS = ("X H He Li Be B C N O F Ne Na Mg Al Si P S Cl Ar K Ca Sc Ti V Cr Mn Fe Co Ni Cu Zn Ga Ge As Se "
            "Br Kr Rb Sr Y Zr Nb Mo Tc Ru Rh Pd Ag Cd In Sn Sb Te I Xe").split()
_Z_OF = {sym: z for z, sym in enumerate(_SYMBOLS) if z}
WEIGHTS_MAGIC = b"TNW1"
_DTYPES = {0: "<f8", 1: "<i8"}


def symbol_to_z(symbol: str) -> int:
    if symbol not in _Z_OF:
        raise ValidationError(f"unknown element symbol {symbol!r}")
    return _Z_OF[symbol]


def z_to_symbol(z: int) -> str:
    if not 1 <= int(z) < len(_SYMBOLS):
        raise ValidationError(f"no symbol for atomic number {z}")
    return _SYMBOLS[int(z)]


@dataclass(frozen=True)
class Frame:
    """One sample: coordinates, species, reference energy, optional forces (data.py:30-41)."""

    positions: np.ndarray
    species: np.ndarray
    energy: float
    forces: Optional[np.ndarray] = None

    @property
    def n_atoms(self) -> int:
        return self.positions.shape[0]


def _atom_fields(text: str, lineno: int):
    """``symbol-or-Z x y z [fx fy fz]`` -> (z, [x, y, z], [fx, fy, fz] or None)."""
    fields = text.split()
    if len(fields) != 4 and len(fields) != 7:
        raise ParseError(f"line {lineno}: expected 'symbol x y z [fx fy fz]', got {len(fields)} fields")
    head = fields[0]
    if head.lstrip("-").isdigit():
        z = int(head)
        if z < 1:
            raise ParseError(f"line {lineno}: bad element symbol {head!r}")
    elif head in _Z_OF:
        z = _Z_OF[head]
    else:
        raise ParseError(f"line {lineno}: bad element symbol {head!r}")
    try:
        numbers = [float(f) for f in fields[1:]]
    except ValueError:
        raise ParseError(f"line {lineno}: malformed coordinate") from None
    return z, numbers[:3], (numbers[3:] if len(numbers) == 6 else None)


def _lines_of(path: Union[str, Path]) -> List[str]:
    path = Path(path)
    if not path.exists():
        raise DataError(f"no such file: {path}")
    return path.read_text().splitlines()


def _energy_of(comment: str, lineno: int) -> Optional[float]:
    try:
        tokens = shlex.split(comment)
    except ValueError:
        raise ParseError(f"line {lineno}: unbalanced quoting") from None
    energy = None
    for token in tokens:
        key, eq, value = token.partition("=")
        if not eq or key != "energy":
            continue
        try:
            energy = float(value)
        except ValueError:
            raise ParseError(f"line {lineno}: malformed energy value {value!r}") from None
        if not np.isfinite(energy):
            raise ParseError(f"line {lineno}: energy must be finite, got {value}")
    return energy


def load_extxyz(path: Union[str, Path]) -> List[Frame]:
    """Every frame of an extended-XYZ file (data.py:89-177)."""
    lines = _lines_of(path)
    frames: List[Frame] = []
    at = 0
    while at < len(lines):
        if not lines[at].strip():
            at += 1
            continue
        try:
            n = int(lines[at].strip())
        except ValueError:
            raise ParseError(f"line {at + 1}: malformed atom count {lines[at].strip()!r}") from None
        if n < 1:
            raise ParseError(f"line {at + 1}: atom count must be positive")
        comment_no = at + 2
        if comment_no > len(lines):
            raise ParseError(f"line {comment_no}: missing comment line")
        energy = _energy_of(lines[comment_no - 1], comment_no)
        if energy is None:
            raise ParseError(f"line {comment_no}: missing energy key")
        species = np.empty(n, dtype=np.int64)
        positions = np.empty((n, 3))
        forces = np.empty((n, 3))
        with_forces = 0
        for a in range(n):
            lineno = comment_no + 1 + a
            if lineno > len(lines):
                raise ParseError(f"line {lineno}: truncated frame")
            species[a], positions[a], f = _atom_fields(lines[lineno - 1], lineno)
            if f is not None:
                forces[a] = f
                with_forces += 1
        if with_forces not in (0, n):
            raise ParseError(f"line {comment_no}: frame mixes atom lines with and without forces")
        frames.append(Frame(positions, species, energy, forces if with_forces else None))
        at = comment_no + n
    if not frames:
        raise ParseError("file contains no frames")
    return frames


def load_structure(path: Union[str, Path]) -> Tuple[np.ndarray, np.ndarray]:
    """First frame of an XYZ file as (positions, species); no energy needed (data.py:180-200)."""
    lines = _lines_of(path)
    if not lines:
        raise ParseError("empty structure file")
    try:
        n = int(lines[0].strip())
    except ValueError:
        raise ParseError(f"line 1: malformed atom count {lines[0].strip()!r}") from None
    if len(lines) < 2 + n:
        raise ParseError("truncated structure file")
    species = np.empty(n, dtype=np.int64)
    positions = np.empty((n, 3))
    for a in range(n):
        species[a], positions[a], _ = _atom_fields(lines[2 + a], 3 + a)
    return positions, species


def write_extxyz(path: Union[str, Path], frames, extra_comment: str = "") -> None:
    """Frames as extended XYZ, floats by ``repr`` (data.py:203-225)."""
    with open(path, "w") as out:
        for frame in frames:
            columns = "species:S:1:pos:R:3" + (":forces:R:3" if frame.forces is not None else "")
            comment = f"energy={float(frame.energy)!r} Properties={columns}"
            if extra_comment:
                comment += " " + extra_comment
            out.write(f"{frame.n_atoms}\n{comment}\n")
            for a in range(frame.n_atoms):
                row = [z_to_symbol(int(frame.species[a]))] + [repr(float(v)) for v in frame.positions[a]]
                if frame.forces is not None:
                    row += [repr(float(v)) for v in frame.forces[a]]
                out.write(" ".join(row) + "\n")


# ----------------------------------------------------------------------------- weights container
def _put_array(out, name: str, array: np.ndarray) -> None:
    code = {"f": 0, "i": 1}.get(array.dtype.kind)
    if code is None:
        raise ValidationError(f"unsupported dtype {array.dtype} for array {name!r}")
    data = np.ascontiguousarray(array.astype(_DTYPES[code], copy=False))
    label = name.encode("utf-8")
    out.write(struct.pack("<H", len(label)) + label + struct.pack("<BB", code, data.ndim))
    out.write(struct.pack(f"<{data.ndim}Q", *data.shape))
    out.write(data.tobytes())


def _take(handle, n: int, what: str) -> bytes:
    data = handle.read(n)
    if len(data) != n:
        raise DataError(f"truncated weights file while reading {what}")
    return data


def save_weights(path: Union[str, Path], config, params: Dict[str, np.ndarray]) -> None:
    """``TNW1`` + u32 JSON length + JSON ``TNConfig`` + u32 array count + arrays (reference encoding)."""
    header = json.dumps({"format": "tensornet-weights", "config": asdict(config)}).encode("utf-8")
    with open(path, "wb") as out:
        out.write(WEIGHTS_MAGIC + struct.pack("<I", len(header)) + header + struct.pack("<I", len(params)))
        for name in sorted(params):
            _put_array(out, name, np.atleast_1d(np.asarray(params[name])))


def load_weights(path: Union[str, Path]):
    """-> (TNConfig, params) as written by ``save_weights``; every array of ``init_params`` must be there."""
    from .tensornet import TNConfig, init_params

    path = Path(path)
    if not path.exists():
        raise DataError(f"no such weights file: {path}")
    with open(path, "rb") as handle:
        magic = handle.read(4)
        if magic == b"MDKC":
            raise DataError(f"{path} is an nnpkit trainer checkpoint (weights of its GraphPotential), "
                            "not a TensorNet weights file")
        if magic != WEIGHTS_MAGIC:
            raise DataError(f"not a TensorNet weights file: {path}")
        (hlen,) = struct.unpack("<I", _take(handle, 4, "header length"))
        header = json.loads(_take(handle, hlen, "header"))
        (count,) = struct.unpack("<I", _take(handle, 4, "array count"))
        arrays = {}
        for _ in range(count):
            (nlen,) = struct.unpack("<H", _take(handle, 2, "name length"))
            name = _take(handle, nlen, "array name").decode("utf-8")
            code, rank = struct.unpack("<BB", _take(handle, 2, "array header"))
            if code not in _DTYPES:
                raise DataError(f"array {name!r}: unknown dtype code {code}")
            shape = struct.unpack(f"<{rank}Q", _take(handle, 8 * rank, "shape"))
            dtype = np.dtype(_DTYPES[code])
            raw = _take(handle, int(np.prod(shape, dtype=np.int64)) * dtype.itemsize, f"array {name!r}")
            arrays[name] = np.frombuffer(raw, dtype=dtype).reshape(shape).copy()
    config = TNConfig(**header["config"])
    params = init_params(config, seed=0)
    for name, template in params.items():
        if name not in arrays:
            raise DataError(f"weights file is missing array {name!r}")
        if arrays[name].size != np.asarray(template).size:
            raise DataError(f"array {name!r} has {arrays[name].size} entries, the config needs {np.asarray(template).size}")
        params[name] = arrays[name].reshape(np.asarray(template).shape)
    return config, params
