"""MDLB lookup-bundle files (reference tables.py:20-77), read into HBM.

Format (little endian): header struct "<4sHQIIII" = magic b"MDLB", version 1,
vocab, clusters E, n-gram depth n, layers, experts (30 bytes — the reference
docstring's "8+20" is wrong), then the sections
labels <i2[vocab], confidence <f4[vocab], provenance u1[vocab],
n-gram probs <f4[E^n * E], n-gram counts <u4[E^n * E], expert labels <i2[N].

`read_bundle` returns a `LookupBundle` exactly like the reference's (probs
are widened to float64, counts to int64, tables.py:69-70), so `best` /
`confidence` — and therefore the device lookup — are bit-identical.
`load_device_tables` goes one step further and leaves the tables resident on
the GPU for `lookup_devices` / `SpecMoELayer`.
"""

from __future__ import annotations

import struct

import numpy as np

from .predictor import DeviceNGramTable, TokenDeviceTable
from .scheduler import LookupBundle

BUNDLE_MAGIC = b"MDLB"
BUNDLE_VERSION = 1
_HEADER = struct.Struct("<4sHQIIII")


class TableError(ValueError):
    pass


def write_bundle(path, bundle) -> None:
    tok, ng = bundle.token_table, bundle.ngram_table
    head = _HEADER.pack(BUNDLE_MAGIC, BUNDLE_VERSION, len(tok.labels), int(tok.n_clusters),
                        int(ng.n), int(bundle.layers), len(bundle.expert_labels))
    parts = [head,
             np.asarray(tok.labels).astype("<i2").tobytes(),
             np.asarray(tok.confidence).astype("<f4").tobytes(),
             np.asarray(tok.provenance).astype("u1").tobytes(),
             np.asarray(ng.probs).astype("<f4").tobytes(),
             np.asarray(ng.counts).astype("<u4").tobytes(),
             np.asarray(bundle.expert_labels).astype("<i2").tobytes()]
    with open(path, "wb") as fh:
        fh.write(b"".join(parts))


def read_bundle(path) -> LookupBundle:
    with open(path, "rb") as fh:
        blob = fh.read()
    if len(blob) < _HEADER.size:
        raise TableError("truncated bundle header")
    magic, version, vocab, E, n, layers, n_experts = _HEADER.unpack_from(blob, 0)
    if magic != BUNDLE_MAGIC:
        raise TableError("not a lookup bundle (bad magic)")
    if version != BUNDLE_VERSION:
        raise TableError(f"unsupported bundle version {version}")
    rows = E ** n
    layout = [("labels", "<i2", vocab), ("confidence", "<f4", vocab), ("provenance", "u1", vocab),
              ("probs", "<f4", rows * E), ("counts", "<u4", rows * E),
              ("expert_labels", "<i2", n_experts)]
    off = _HEADER.size
    sec = {}
    for name, dt, count in layout:
        nbytes = np.dtype(dt).itemsize * count
        if off + nbytes > len(blob):
            raise TableError("truncated bundle payload")
        sec[name] = np.frombuffer(blob, dtype=dt, count=count, offset=off).copy()
        off += nbytes
    tok = TokenDeviceTable(labels=sec["labels"], confidence=sec["confidence"],
                           provenance=sec["provenance"], n_clusters=E)
    ng = DeviceNGramTable(n=n, n_clusters=E,
                          probs=sec["probs"].astype(np.float64).reshape(rows, E),
                          counts=sec["counts"].astype(np.int64).reshape(rows, E))
    return LookupBundle(token_table=tok, ngram_table=ng, expert_labels=sec["expert_labels"],
                        layers=layers)


def load_device_tables(path):
    """read_bundle + upload: (bundle, DeviceTables resident in HBM)."""
    from .scheduler import device_tables
    b = read_bundle(path)
    return b, device_tables(b)


def export_token_csv(path, bundle) -> None:
    tok = bundle.token_table
    with open(path, "w", newline="") as fh:
        fh.write("token,label,confidence,provenance\r\n")
        for j in range(len(tok.labels)):
            fh.write(f"{j},{int(tok.labels[j])},{float(tok.confidence[j]):.6f},"
                     f"{int(tok.provenance[j])}\r\n")
