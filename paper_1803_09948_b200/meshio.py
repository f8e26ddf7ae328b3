"""Mesh ingestion for the command line: the two formats of the
reference's mesh_io.cpp, host-side I/O with the same acceptance rules.

  GMSH MSH 2.2 ASCII   6-node curved triangles (element type 9); every other element is skipped and
                       counted (mesh_io.cpp:38-136); nodes are written de-duplicated by exact
                       coordinate bits with 17 significant digits (:138-170)
  binary blocks        32-byte big-endian header (magic "HFMMMESH", version 1, element count, 6 points
                       per element) and 144-byte records of 18 big-endian f64 (:186-239); rank r of R
                       reads the elements [floor(r E / R), floor((r + 1) E / R))

Both return / take an array (elements, 6, 3): 3 corners then 3 edge midsides, the node order of
CurvilinearPatch (geometry.hpp:13-20)."""
from __future__ import annotations

import numpy as np


class MeshError(ValueError):
    """parse_error / format_error / structural_error of the reference, by kind"""

    def __init__(self, kind: str, message: str):
        super().__init__(f"{kind}: {message}")
        self.kind = kind


def read_gmsh(path):
    """-> (patches (E, 6, 3) float64, skipped element count)"""
    with open(path, "r") as f:
        lines = [ln.rstrip("\r\n") for ln in f]
    pos, nodes, elements, skipped = 0, None, None, 0

    def need(i, what):
        if i >= len(lines):
            raise MeshError("parse_error", f"{what} (line {i + 1})")
        return lines[i]

    while pos < len(lines):
        line = lines[pos]
        pos += 1
        if not line or line[0] != "$":
            continue                               # stray tokens between sections are ignored
        if line == "$MeshFormat":
            parts = need(pos, "unterminated $MeshFormat").split()
            pos += 1
            try:
                version, file_type = float(parts[0]), int(parts[1])
                int(parts[2])
            except (IndexError, ValueError):
                raise MeshError("parse_error", f"malformed format line (line {pos})")
            if version < 2.0 or version >= 3.0 or file_type != 0:
                raise MeshError("format_error", "unsupported mesh format version " + lines[pos - 1])
            if need(pos, "missing $EndMeshFormat") != "$EndMeshFormat":
                raise MeshError("parse_error", f"missing $EndMeshFormat (line {pos + 1})")
            pos += 1
        elif line == "$Nodes":
            try:
                count = int(need(pos, "unterminated $Nodes"))
            except ValueError:
                raise MeshError("parse_error", f"bad node count (line {pos + 1})")
            pos += 1
            nodes = {}
            for _ in range(count):
                parts = need(pos, "truncated $Nodes section").split()
                pos += 1
                try:
                    nid, p = int(parts[0]), (float(parts[1]), float(parts[2]), float(parts[3]))
                except (IndexError, ValueError):
                    raise MeshError("parse_error", f"malformed node line (line {pos})")
                if not np.all(np.isfinite(p)):
                    raise MeshError("parse_error", f"non-finite node coordinate (line {pos})")
                nodes[nid] = p
            if need(pos, "missing $EndNodes") != "$EndNodes":
                raise MeshError("parse_error", f"missing $EndNodes (line {pos + 1})")
            pos += 1
        elif line == "$Elements":
            if nodes is None:
                raise MeshError("parse_error", f"$Elements before $Nodes (line {pos})")
            try:
                count = int(need(pos, "unterminated $Elements"))
            except ValueError:
                raise MeshError("parse_error", f"bad element count (line {pos + 1})")
            pos += 1
            elements = []
            for _ in range(count):
                parts = need(pos, "truncated $Elements section").split()
                pos += 1
                try:
                    eid, etype, ntags = int(parts[0]), int(parts[1]), int(parts[2])
                    [int(t) for t in parts[3:3 + ntags]]
                    if len(parts) < 3 + ntags:
                        raise ValueError
                except (IndexError, ValueError):
                    raise MeshError("parse_error", f"malformed element line (line {pos})")
                if etype != 9:                     # only 6-node second-order triangles become patches
                    skipped += 1
                    continue
                try:
                    ids = [int(t) for t in parts[3 + ntags:3 + ntags + 6]]
                    if len(ids) != 6:
                        raise ValueError
                except ValueError:
                    raise MeshError("parse_error", f"element needs 6 node ids (line {pos})")
                for nid in ids:
                    if nid not in nodes:
                        raise MeshError("structural_error", f"element {eid} references unknown node {nid}")
                elements.append([nodes[nid] for nid in ids])
            if need(pos, "missing $EndElements") != "$EndElements":
                raise MeshError("parse_error", f"missing $EndElements (line {pos + 1})")
            pos += 1
        else:                                      # unknown section: skip to its terminator
            end = "$End" + line[1:]
            while pos < len(lines) and lines[pos] != end:
                pos += 1
            if pos >= len(lines):
                raise MeshError("parse_error", "unterminated section " + end)
            pos += 1
    if nodes is None or elements is None:
        raise MeshError("parse_error", "missing $Nodes or $Elements section")
    if not elements:
        raise MeshError("format_error", "mesh contains no usable curved triangles")
    return np.asarray(elements, dtype=np.float64).reshape(-1, 6, 3), skipped


def write_gmsh(patches, path):
    patches = np.asarray(patches, dtype=np.float64).reshape(-1, 6, 3)
    ids, unique, conn = {}, [], np.zeros((len(patches), 6), dtype=np.int64)
    for e, el in enumerate(patches):
        for n, p in enumerate(el):
            key = p.tobytes()                      # exact coordinate bits
            if key not in ids:
                ids[key] = len(unique)
                unique.append(p)
            conn[e, n] = ids[key] + 1
    with open(path, "w") as f:
        f.write(f"$MeshFormat\n2.2 0 8\n$EndMeshFormat\n$Nodes\n{len(unique)}\n")
        for i, p in enumerate(unique):
            f.write(f"{i + 1} {p[0]:.17g} {p[1]:.17g} {p[2]:.17g}\n")
        f.write(f"$EndNodes\n$Elements\n{len(patches)}\n")
        for e in range(len(patches)):
            f.write(f"{e + 1} 9 2 0 0 " + " ".join(str(v) for v in conn[e]) + "\n")
        f.write("$EndElements\n")


MAGIC = b"HFMMMESH"


def write_binary(patches, path) -> int:
    patches = np.asarray(patches, dtype=np.float64).reshape(-1, 6, 3)
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(np.array([1, len(patches), 6], dtype=">u8").tobytes())
        f.write(patches.astype(">f8").tobytes())
    return 32 + 144 * len(patches)


def read_binary(path, rank: int = 0, nranks: int = 1):
    """the block of `rank`: elements [floor(rank E / nranks), floor((rank + 1) E / nranks))"""
    if nranks <= 0 or rank < 0 or rank >= nranks:
        raise MeshError("config_error", f"read_block: rank {rank} of {nranks} out of range")
    with open(path, "rb") as f:
        head = f.read(32)
        if len(head) < 8 or head[:8] != MAGIC:
            raise MeshError("format_error", "read_block: bad magic")
        if len(head) < 32:
            raise MeshError("io_error", "truncated mesh file")
        version, count, ppe = (int(v) for v in np.frombuffer(head[8:], dtype=">u8"))
        if version != 1:
            raise MeshError("format_error", f"read_block: unsupported version {version}")
        if ppe != 6:
            raise MeshError("format_error", "read_block: expected 6 points per element")
        begin, end = rank * count // nranks, (rank + 1) * count // nranks
        f.seek(32 + 144 * begin)
        raw = f.read(144 * (end - begin))
        if len(raw) != 144 * (end - begin):
            raise MeshError("io_error", "truncated mesh file")
    return np.frombuffer(raw, dtype=">f8").astype(np.float64).reshape(-1, 6, 3)


def read_mesh(path):
    """by content: binary blocks start with the magic, anything else is parsed as MSH 2.2 ASCII"""
    with open(path, "rb") as f:
        if f.read(8) == MAGIC:
            return read_binary(path)
    return read_gmsh(path)[0]
