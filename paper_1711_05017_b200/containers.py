"""On-disk containers for density fields (GFLD) and spectra (GSPC).

The byte layouts are the reference's, so files move freely between the two
packages (writers at /root/reference/pkg/src/geofield/descriptor.py:383-416
and spectral.py:233-265).  Both are little-endian: a 4-byte magic, then
(version, d) as two u32, then the grid, then a complex64 payload.  They differ
only in the order of the grid fields and in what follows the grid:

    GFLD  dims[d] u32 | origin[d] f64 | spacing f64 | N values | u32 count + u32 flags
    GSPC  dims[d] u32 | spacing f64 | origin[d] f64 | u64 m'   | m' amplitudes

One table-driven codec serves both, and the payload writer casts device
tensors to complex64 on the GPU so only half the bytes cross PCIe.
"""

from __future__ import annotations

import struct

import numpy as np

VERSION = 1

# grid record order per container; "count" is GSPC's explicit payload length
_GRID_ORDER = {
    b"GFLD": ("dims", "origin", "spacing"),
    b"GSPC": ("dims", "spacing", "origin", "count"),
}


def _field_format(key, d):
    return {"dims": f"<{d}I", "origin": f"<{d}d", "spacing": "<d", "count": "<Q"}[key]


def pack_header(magic, d, dims, origin, spacing, count=None):
    """Bytes of one container header (magic through the grid record)."""
    vals = {"dims": dims, "origin": origin, "spacing": (spacing,), "count": (count,)}
    parts = [magic, struct.pack("<II", VERSION, d)]
    parts += [struct.pack(_field_format(k, d), *vals[k]) for k in _GRID_ORDER[magic]]
    return b"".join(parts)


def unpack_header(fh, magic):
    """Read a header written by pack_header; returns (d, dims, origin,
    spacing, count) with count None for GFLD.  Raises ValueError on a wrong
    magic or version, like the reference readers."""
    kind = magic.decode()
    if fh.read(4) != magic:
        raise ValueError(f"not a {kind} file")
    version, d = struct.unpack("<II", fh.read(8))
    if version != VERSION:
        raise ValueError(f"unsupported {kind} version {version}")
    rec = {"count": (None,)}
    for key in _GRID_ORDER[magic]:
        fmt = _field_format(key, d)
        rec[key] = struct.unpack(fmt, fh.read(struct.calcsize(fmt)))
    return d, tuple(rec["dims"]), tuple(rec["origin"]), rec["spacing"][0], rec["count"][0]


def complex64_payload(host=None, device=None):
    """complex64 bytes of a payload held on the host (numpy) or the device
    (torch); the device path casts before the copy."""
    if device is not None:
        import torch

        return device.to(torch.complex64).cpu().numpy().tobytes()
    return np.asarray(host).astype(np.complex64).tobytes()


def read_complex(fh, n):
    """n complex64 values from fh, widened to complex128 on the host."""
    return np.frombuffer(fh.read(8 * n), dtype=np.complex64).astype(np.complex128)


def pack_flags(flags):
    arr = np.asarray(flags, dtype=np.uint32)
    return struct.pack("<I", arr.size) + arr.tobytes()


def read_flags(fh):
    (n,) = struct.unpack("<I", fh.read(4))
    return np.frombuffer(fh.read(4 * n), dtype=np.uint32).tolist()
