"""CSV ingestion of labelled data and make_instance (data_io.hpp), the step
before the hot path, with the reference's API, file format and errors.

* read_csv / load_csv (data_io.hpp:199-352): the two-file format -- source
  ``label[,weight],f0,f1,...``, target ``[weight,]f0,f1,...`` -- parsed like
  the reference (strtod / strtol token rules, header checks, field counts),
  source rows stably sorted by label;
* partition_from_labels (data_io.hpp:127-152);
* make_instance (data_io.hpp:157-181): the cost matrix is computed ON THE
  GPU from the features (gsot_cost_matrix_device, k-sequential without FMA:
  bitwise the reference's cost_matrix) and normalised by its maximum;
  make_device_instance builds the solver context directly from the features
  (gsot_create_features) without the cost ever visiting the host;
* save_source_csv / save_target_csv / save_matrix_csv (data_io.hpp:352-400),
  numbers written with "%.17g" (data_io.hpp:185-189).

Errors: ParseError(line, column), MissingLabelColumn, InconsistentDimension
(line) and PartitionMismatch with the reference's messages
(errors.hpp:58-83).
"""
from __future__ import annotations

import ctypes as C
import math
import re
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .groupot import (Context, Error, GroupPartition, PartitionMismatch, ProblemInstance,
                      RegParams, _f64, _ptr, _raise)


class ParseError(Error):
    """errors.hpp:58-67."""

    def __init__(self, line: int, column: int, what: str):
        super().__init__(f"parse error at line {line}, column {column}: {what}")
        self.line, self.column = line, column


class MissingLabelColumn(Error):
    """errors.hpp:69-73."""

    def __init__(self, path: str):
        super().__init__(f"source file {path} must start with a 'label' column")


class InconsistentDimension(Error):
    """errors.hpp:75-81."""

    def __init__(self, line: int, what: str):
        super().__init__(f"inconsistent dimension at line {line}: {what}")
        self.line = line


@dataclass
class LabeledSamples:
    """data_io.hpp:17-22: rows sorted by label, labels dense in 1..L."""

    features: np.ndarray  # m x d
    labels: list
    weights: np.ndarray = field(default_factory=lambda: np.empty(0))


@dataclass
class UnlabeledSamples:
    """data_io.hpp:24-27."""

    features: np.ndarray  # n x d
    weights: np.ndarray = field(default_factory=lambda: np.empty(0))


# strtod accepts C99 floating literals (decimal, hex, inf / nan spellings)
# after optional leading whitespace; the reference requires the whole token.
_FLOAT = re.compile(
    r"[ \t\n\v\f\r]*[+-]?(?:(?:\d+\.?\d*(?:[eE][+-]?\d+)?|\.\d+(?:[eE][+-]?\d+)?)"
    r"|0[xX](?:[0-9a-fA-F]+\.?[0-9a-fA-F]*|\.[0-9a-fA-F]+)(?:[pP][+-]?\d+)?"
    r"|(?i:inf(?:inity)?|nan(?:\([0-9A-Za-z_]*\))?))\Z")
_LONG = re.compile(r"[ \t\n\v\f\r]*[+-]?\d+\Z")


def _strtod(tok: str) -> float | None:
    if not _FLOAT.match(tok):
        return None
    t = tok.strip(" \t\n\v\f\r")
    if t.lower().lstrip("+-").startswith("0x"):
        sign = -1.0 if t.startswith("-") else 1.0
        return sign * float.fromhex(t.lstrip("+-"))
    tl = t.lower()
    if "nan" in tl:
        return float("nan")
    if "inf" in tl:
        return float("-inf") if tl.startswith("-") else float("inf")
    return float(t)


def _parse_double(tok: str, line: int, column: int) -> float:
    """data_io.hpp:205-212."""
    v = _strtod(tok)
    if v is None:
        raise ParseError(line, column, f"'{tok}' is not a number")
    return v


def _parse_label(tok: str, line: int) -> int:
    """data_io.hpp:214-221."""
    if not _LONG.match(tok) or int(tok) < 1:
        raise ParseError(line, 0, f"'{tok}' is not a positive label")
    return int(tok)


def read_csv(path: str):
    """data_io.hpp:228-252: (header, rows); blank lines skipped, CR stripped,
    every row as wide as the header."""
    try:
        f = open(path, "rb")
    except OSError:
        raise Error(f"cannot open {path}") from None
    header, rows = [], []
    with f:
        for line_no, raw in enumerate(f.read().decode("latin-1").split("\n"), start=1):
            line = raw[:-1] if raw.endswith("\r") else raw
            if line == "":
                continue
            toks = line.split(",")
            if line_no == 1:
                header = toks
                continue
            if len(toks) != len(header):
                raise InconsistentDimension(
                    line_no, f"row has {len(toks)} fields, header has {len(header)}")
            rows.append(toks)
    if not header:
        raise ParseError(1, 0, f"empty file {path}")
    return header, rows


def _expect_feature_names(header, first: int, path: str) -> None:
    """data_io.hpp:254-263."""
    for i in range(first, len(header)):
        want = f"f{i - first}"
        if header[i] != want:
            raise ParseError(1, i, f"{path}: expected column '{want}', got '{header[i]}'")


def load_csv(source_path: str, target_path: str):
    """data_io.hpp:270-352: (LabeledSamples, UnlabeledSamples)."""
    sh, sr = read_csv(source_path)
    if not sh or sh[0] != "label":
        raise MissingLabelColumn(source_path)
    src_weighted = len(sh) > 1 and sh[1] == "weight"
    first = 2 if src_weighted else 1
    if len(sh) <= first:
        raise ParseError(1, len(sh), f"{source_path}: no feature columns")
    _expect_feature_names(sh, first, source_path)
    d = len(sh) - first
    recs = []
    for r, toks in enumerate(sr):
        line = r + 2
        lab = _parse_label(toks[0], line)
        w = _parse_double(toks[1], line, 1) if src_weighted else 1.0
        feat = [_parse_double(toks[first + k], line, first + k) for k in range(d)]
        recs.append((lab, w, feat))
    if not recs:
        raise ParseError(2, 0, f"{source_path}: no data rows")
    recs.sort(key=lambda t: t[0])  # stable, as std::stable_sort
    src = LabeledSamples(np.array([t[2] for t in recs], dtype=np.float64).reshape(len(recs), d),
                         [t[0] for t in recs],
                         np.array([t[1] for t in recs]) if src_weighted else np.empty(0))
    th, tr = read_csv(target_path)
    tgt_weighted = bool(th) and th[0] == "weight"
    tfirst = 1 if tgt_weighted else 0
    _expect_feature_names(th, tfirst, target_path)
    td = len(th) - tfirst
    if td != d:
        raise InconsistentDimension(1, f"{target_path} has {td} features, source has {d}")
    if not tr:
        raise ParseError(2, 0, f"{target_path}: no data rows")
    feats, ws = [], []
    for r, toks in enumerate(tr):
        line = r + 2
        if tgt_weighted:
            ws.append(_parse_double(toks[0], line, 0))
        feats.append([_parse_double(toks[tfirst + k], line, tfirst + k) for k in range(d)])
    tgt = UnlabeledSamples(np.array(feats, dtype=np.float64).reshape(len(feats), d),
                           np.array(ws) if tgt_weighted else np.empty(0))
    return src, tgt


def partition_from_labels(labels) -> GroupPartition:
    """data_io.hpp:127-152: contiguous partition of sorted labels dense in 1..L."""
    labels = [int(v) for v in labels]
    if not labels:
        raise PartitionMismatch("group partition: no labels")
    current = labels[0]
    if current != 1:
        raise PartitionMismatch(f"group partition: labels must start at 1, got {current}")
    sizes, count = [], 0
    for i, lab in enumerate(labels):
        if lab == current:
            count += 1
        elif lab == current + 1:
            sizes.append(count)
            current, count = lab, 1
        else:
            raise PartitionMismatch(
                f"group partition: labels not sorted/dense near index {i} "
                f"(label {lab} after {current})")
    sizes.append(count)
    return GroupPartition(sizes)


def _seq_sum(v: np.ndarray) -> float:
    """Eigen's sum() as the oracle's sequential build accumulates it."""
    return float(np.cumsum(np.asarray(v, np.float64))[-1]) if len(v) else 0.0


def _marginals(src: LabeledSamples, tgt: UnlabeledSamples, use_weights: bool):
    """make_instance's marginals (data_io.hpp:167-176)."""
    m, n = src.features.shape[0], tgt.features.shape[0]
    if use_weights and src.weights.size == m:
        a = src.weights / _seq_sum(src.weights)
    else:
        a = np.full(m, 1.0 / float(m))
    if use_weights and tgt.weights.size == n:
        b = tgt.weights / _seq_sum(tgt.weights)
    else:
        b = np.full(n, 1.0 / float(n))
    return np.ascontiguousarray(a, np.float64), np.ascontiguousarray(b, np.float64)


def cost_matrix(src: LabeledSamples, tgt: UnlabeledSamples, normalize: bool = False) -> np.ndarray:
    """cost_matrix (data_io.hpp:101-123), on the GPU: m x n, bitwise the
    reference's k-sequential no-FMA sums; divided by its max when normalize."""
    import torch

    s = np.ascontiguousarray(src.features, np.float64)
    t = np.ascontiguousarray(tgt.features, np.float64)
    m, d = s.shape
    n = t.shape[0]
    if t.shape[1] != d:
        raise InconsistentDimension(1, f"target has {t.shape[1]} features, source has {d}")
    dev = torch.empty((n, m), dtype=torch.float64, device="cuda")
    _raise(_lib.lib().gsot_cost_matrix_device(_ptr(s), m, _ptr(t), n, d, 1 if normalize else 0,
                                              C.c_void_p(dev.data_ptr())))
    torch.cuda.synchronize()
    return dev.cpu().numpy().T  # column-major m x n, as Eigen::MatrixXd


def make_instance(src: LabeledSamples, tgt: UnlabeledSamples, normalize_cost: bool = False,
                  use_weights: bool = False) -> ProblemInstance:
    """data_io.hpp:157-181 (cost on the device, then validate_instance)."""
    from .groupot import validate_instance

    c = cost_matrix(src, tgt, normalize_cost)
    a, b = _marginals(src, tgt, use_weights)
    inst = ProblemInstance(c, a, b, partition_from_labels(src.labels))
    validate_instance(inst)
    return inst


def make_device_instance(src: LabeledSamples, tgt: UnlabeledSamples, p: RegParams,
                         normalize_cost: bool = False, use_weights: bool = False) -> Context:
    """make_instance straight into a solver context (gsot_create_features):
    the cost is built in HBM from the features and never visits the host."""
    s = np.ascontiguousarray(src.features, np.float64)
    t = np.ascontiguousarray(tgt.features, np.float64)
    m, d = s.shape
    n = t.shape[0]
    if t.shape[1] != d:
        raise InconsistentDimension(1, f"target has {t.shape[1]} features, source has {d}")
    sizes = np.asarray(partition_from_labels(src.labels).sizes(), np.int32)
    a, b = _marginals(src, tgt, use_weights)
    h = C.c_void_p()
    _raise(_lib.lib().gsot_create_features(_ptr(s), m, _ptr(t), n, d, _ptr(sizes), len(sizes),
                                           _ptr(a), _ptr(b), 1 if normalize_cost else 0,
                                           float(p.gamma()), float(p.mu()), C.byref(h)))
    return Context(h.value)


def _fmt(v: float) -> str:
    """detail::format_double (data_io.hpp:185-189): printf("%.17g")."""
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "inf" if v > 0 else "-inf"
    return "%.17g" % v


def save_source_csv(src: LabeledSamples, path: str) -> None:
    """data_io.hpp:352-364."""
    d = src.features.shape[1]
    with open(path, "w") as f:
        f.write("label" + "".join(f",f{k}" for k in range(d)) + "\n")
        for lab, row in zip(src.labels, src.features):
            f.write(str(int(lab)) + "".join("," + _fmt(float(v)) for v in row) + "\n")


def save_target_csv(tgt: UnlabeledSamples, path: str) -> None:
    """data_io.hpp:366-380."""
    d = tgt.features.shape[1]
    with open(path, "w") as f:
        f.write(",".join(f"f{k}" for k in range(d)) + "\n")
        for row in tgt.features:
            f.write(",".join(_fmt(float(v)) for v in row) + "\n")


def save_matrix_csv(mat, path: str) -> None:
    """data_io.hpp:383-395: plain numeric CSV without header."""
    mat = np.asarray(mat, np.float64)
    with open(path, "w") as f:
        for row in mat:
            f.write(",".join(_fmt(float(v)) for v in row) + "\n")
