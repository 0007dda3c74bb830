"""The reference's OWN C++ hot-path test suites (test_half, test_pack,
test_vec_lut, test_streamk, test_nf_table, test_mma, test_engine,
test_quantize, test_refine from /root/reference/proj/tests) compiled
unmodified against flute-b200's drop-in headers and libflute_b200.so
(tests/refsuite: doctest-compatible shim + Makefile; binary in oracle/_ref/,
built by __graft_entry__.build() where the reference sources exist).  The
engine, mma and refine suites call execute() / mma_fragment() /
ste_evaluate() / refine_scales() on the GPU; on a host without one they are
skipped here and run under the gpu marker."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "flute_refsuite")
# the same suites linked against the reference library itself
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "flute_refsuite_reflib")


def _run(skip, binary=BIN):
    if not os.path.exists(binary):
        pytest.skip(f"{os.path.basename(binary)} not built (needs the reference test sources)")
    env = dict(os.environ)
    if skip:
        env["REFSUITE_SKIP"] = skip
    r = subprocess.run([binary], capture_output=True, text=True, env=env, timeout=900)
    return r


def _failed(out: str) -> set:
    return {ln.split("]", 1)[1].strip() for ln in out.splitlines() if ln.startswith("[case FAILED]")}


def _check_against_reference(skip):
    """Every case the reference passes against its own library passes against
    ours.  Cases the reference library itself fails in this environment are
    reported, not required (engine's randomized binary64 sweep: its f16
    Stream-K reduction exceeds the bound; refine's
    heavy-tailed descent case: 27/30 trials improve with libstdc++'s
    student_t stream, for the reference and, bit-identically, for us)."""
    ours = _run(skip)
    ref = _run(skip, REF_BIN)
    extra = _failed(ours.stdout + ours.stderr) - _failed(ref.stdout + ref.stderr)
    assert not extra, (sorted(extra), ours.stdout[-2000:] + ours.stderr[-4000:])
    return ours


def test_reference_suites_host_parts():
    _check_against_reference("engine:,mma:,refine:")


@pytest.mark.gpu
def test_reference_suites_all_on_gpu():
    r = _check_against_reference("")
    assert "| 0 skipped" in r.stdout
