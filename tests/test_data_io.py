"""CSV ingestion (data_io.hpp:127-400) in the Python mirror against the
reference's own load_csv / partition_from_labels / make_instance (oracle/_ref)
on valid files and on every error path: the parsed samples equal bitwise, the
errors have the reference's type, line / column and message. The device
make_instance (cost built on the GPU) is checked in test_gpu_data_io.py."""
import os

import numpy as np
import pytest

import paper_2303_07597_b200 as G
from oracle_bindings import ref_available, ref_load_csv, ref_partition_from_labels

pytestmark = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")

ERR = {11: G.ParseError, 12: G.MissingLabelColumn, 13: G.InconsistentDimension,
       4: G.PartitionMismatch, 5: G.Error}


def write(tmp_path, name, text):
    p = os.path.join(tmp_path, name)
    with open(p, "w", newline="") as f:
        f.write(text)
    return p


VALID_TGT = "f0,f1\n0.5,1\n2,3\n"
CASES = {
    # name: (source text, target text)
    "plain": ("label,f0,f1\n2,1.5,2\n1,0.25,-3\n1,1e-3,4\n3,7,8\n", VALID_TGT),
    "weighted": ("label,weight,f0,f1\n1,0.5,1,2\n2,2,3,4\n", "weight,f0,f1\n1,0.5,1\n3,2,3\n"),
    "crlf_blank": ("label,f0,f1\r\n1,1,2\r\n\r\n2,3,4\r\n", "f0,f1\r\n1,2\r\n"),
    "number_forms": ("label,f0,f1\n1,+1.5E+2, 3\n2,0x1.8p1,-.5\n2,inf,-INFINITY\n", VALID_TGT),
    "no_trailing_newline": ("label,f0,f1\n1,1,2\n2,3,4", "f0,f1\n1,2"),
    "missing_label": ("lab,f0,f1\n1,1,2\n", VALID_TGT),
    "bad_feature_name": ("label,f0,g1\n1,1,2\n", VALID_TGT),
    "no_features": ("label\n1\n", VALID_TGT),
    "weight_no_features": ("label,weight\n1,1\n", VALID_TGT),
    "bad_number": ("label,f0,f1\n1,1,2\n2,x,4\n", VALID_TGT),
    "trailing_space": ("label,f0,f1\n1,1 ,2\n", VALID_TGT),
    "bad_label": ("label,f0,f1\n0,1,2\n", VALID_TGT),
    "float_label": ("label,f0,f1\n1.0,1,2\n", VALID_TGT),
    "short_row": ("label,f0,f1\n1,1,2\n2,3\n", VALID_TGT),
    "no_rows": ("label,f0,f1\n", VALID_TGT),
    "empty_source": ("", VALID_TGT),
    "leading_blank": ("\nlabel,f0,f1\n1,1,2\n", VALID_TGT),
    "target_dim": ("label,f0,f1\n1,1,2\n", "f0\n1\n"),
    "target_bad": ("label,f0,f1\n1,1,2\n", "f0,f1\n1,y\n"),
    "target_no_rows": ("label,f0,f1\n1,1,2\n", "f0,f1\n"),
    "target_weight_bad": ("label,f0,f1\n1,1,2\n", "weight,f0,f1\nz,1,2\n"),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_load_csv_matches_reference(tmp_path, name):
    s_text, t_text = CASES[name]
    sp = write(tmp_path, "src.csv", s_text)
    tp = write(tmp_path, "tgt.csv", t_text)
    ref = ref_load_csv(sp, tp)
    if ref[0] == "error":
        _, status, line, col, msg = ref
        with pytest.raises(ERR[status]) as ei:
            G.load_csv(sp, tp)
        assert str(ei.value) == msg
        if status == 11:
            assert (ei.value.line, ei.value.column) == (line, col)
        if status == 13:
            assert ei.value.line == line
        return
    _, sf, lab, sw, tf, tw = ref
    src, tgt = G.load_csv(sp, tp)
    assert src.labels == lab
    assert np.array_equal(src.features, sf, equal_nan=True)
    assert np.array_equal(src.weights, sw) and np.array_equal(tgt.weights, tw)
    assert np.array_equal(tgt.features, tf, equal_nan=True)


@pytest.mark.parametrize("labels", [[1, 1, 2, 2, 2, 3], [1], [2, 3], [1, 3], [1, 2, 1], [],
                                    [1, 1, 1], [1, 2, 2, 3, 4, 4, 4]])
def test_partition_from_labels_matches_reference(labels):
    ref = ref_partition_from_labels(labels)
    if ref[0] == "error":
        with pytest.raises(ERR[ref[1]]) as ei:
            G.partition_from_labels(labels)
        assert str(ei.value) == ref[2]
    else:
        assert G.partition_from_labels(labels).sizes() == ref[1]


def test_save_csv_round_trip(tmp_path):
    # save_source_csv / save_target_csv write "%.17g": load_csv reads back
    # the same doubles (data_io.hpp:185-189, :352-380)
    rng = np.random.default_rng(0)
    src = G.LabeledSamples(rng.normal(size=(7, 3)) * 10.0 ** rng.integers(-8, 8, (7, 3)),
                           [1, 1, 2, 2, 2, 3, 3])
    tgt = G.UnlabeledSamples(rng.normal(size=(5, 3)))
    sp, tp = os.path.join(tmp_path, "s.csv"), os.path.join(tmp_path, "t.csv")
    G.save_source_csv(src, sp)
    G.save_target_csv(tgt, tp)
    s2, t2 = G.load_csv(sp, tp)
    assert np.array_equal(s2.features, src.features) and s2.labels == src.labels
    assert np.array_equal(t2.features, tgt.features)
    ref = ref_load_csv(sp, tp)
    assert ref[0] == "ok" and np.array_equal(ref[1], src.features)
