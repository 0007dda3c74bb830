"""FLTE container (reference flte.hpp:4-9,
flte.cpp:95-213): our writer reproduces the reference library's bytes exactly,
our strict parser accepts them and rejects corruptions with the same section
name and byte offset as the reference (golden verdicts from
tools/make_golden_flte.py)."""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "flte.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def test_writer_matches_reference_bytes(F, gold):
    for i, (bits, group, k, n) in enumerate(gold["meta"]):
        w = gold[f"w{i}"]
        idx, sc = F.quantize_matrix(w, int(bits), int(group))
        ours = F.flte_write(idx, sc, F.build_nf_table(int(bits)), int(bits), int(group))
        assert ours == gold[f"flte{i}"].tobytes()
        assert F.flte_info(ours) == (bits, group, k, n)


def test_known_offsets(F, gold):
    """test_flte.cpp:108-121: the table starts at byte 19."""
    b = gold["flte0"].tobytes()
    with pytest.raises(F.InputError, match="section 'table' at byte offset 19"):
        F.flte_info(b[:19])


def test_parse_errors_match_reference(F, gold):
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "mgf", os.path.join(os.path.dirname(GOLD), "..", "..", "tools", "make_golden_flte.py"))
    mgf = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mgf)
    verdicts = dict(zip(gold["names"], zip(gold["sections"], gold["offsets"])))
    checked = 0
    for i, (bits, group, k, n) in enumerate(gold["meta"]):
        for name, c in mgf.corruptions(gold[f"flte{i}"].tobytes()):
            sec, off = verdicts[f"w{bits}:{name}"]
            if off < 0:
                F.flte_info(c)
                continue
            with pytest.raises(F.InputError) as ei:
                F.flte_info(c)
            assert f"section '{sec}' at byte offset {off}]" in str(ei.value), (name, str(ei.value))
            checked += 1
    assert checked >= 40
