"""The reference's OWN C++ hot-path test suites (test_half, test_pack,
test_vec_lut, test_streamk, test_nf_table, test_mma, test_engine from
/root/reference/proj/tests) compiled unmodified against flute-b200's drop-in
headers and libflute_b200.so (tests/refsuite: doctest-compatible shim +
Makefile; binary in oracle/_ref/, built by __graft_entry__.build() where the
reference sources exist).  The engine and mma suites call execute() /
mma_fragment() on the GPU; on a host without one they are skipped here and run
under the gpu marker."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "flute_refsuite")


def _run(skip):
    if not os.path.exists(BIN):
        pytest.skip("flute_refsuite not built (needs the reference test sources)")
    env = dict(os.environ)
    if skip:
        env["REFSUITE_SKIP"] = skip
    r = subprocess.run([BIN], capture_output=True, text=True, env=env, timeout=900)
    return r


def test_reference_suites_host_parts():
    r = _run("engine:,mma:")
    assert r.returncode == 0, r.stdout + r.stderr[-4000:]
    assert "0 failed" in r.stdout


@pytest.mark.gpu
def test_reference_suites_all_on_gpu():
    r = _run("")
    assert r.returncode == 0, r.stdout + r.stderr[-4000:]
    assert "| 0 failed | 0 skipped" in r.stdout
