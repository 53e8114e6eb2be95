"""The reference's OWN unit tests, run against the B200 drop-in.

oracle/Makefile (target `unit`) compiles /root/reference/proj/tests/test_{datamodel,
fitness,evolution,expansion,synthgen,metrics}.cpp where they lie -- no copy in
this repo -- against oracle/catch_shim (a minimal Catch2 stand-in; Catch2 is
not in this image) twice:
  oracle/_ref/unit_ref     with the reference headers (proves the shim);
  oracle/_ref/unit_dropin  with include/ (shadow fitness.hpp, expansion.hpp,
                           evolution.hpp) first on the include path, linked to
                           libebic_b200.so.
test_cli.cpp is left out: it drives the reference's CLI binary.
The drop-in cases that evaluate series need the GPU; the rest (mutation
operators, tabu list, top-rank list, generation building, data model,
synthetic generator, metrics) run here on CPU.
"""
import subprocess

import pytest

import oracle

UNIT_REF = oracle.HERE / "_ref" / "unit_ref"
UNIT_DROPIN = oracle.HERE / "_ref" / "unit_dropin"

# Test cases (name substrings) whose drop-in path launches the count kernel.
DEVICE_CASES = [
    "match counting is independent of the chunking",
    "population evaluation combines counts and the score formula",
    "full runs are deterministic at any worker count",
    "runs never evaluate the same series twice",
    "the best fitness never decreases between generations",
    "zero iterations returns the initialization-only list",
    "runs on narrow column spaces terminate through the tabu list",
    "row assignment lists exactly the increasing rows",
    "row assignment agrees with the chunked match counts",
    "resolving a series produces its exact support",
    "expansion adds reversed and near-miss rows with their flags",
    "a row matching the reversed series outranks its near-miss reading",
    "expansion with everything disabled is the identity",
    "negative rows are the support of the reversed series",
    "expansion keeps the input rows and their flags",
]


def _run(binary, *args):
    r = subprocess.run([str(binary), *args], capture_output=True, text=True, timeout=900)
    summary = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else ""
    return r.returncode, summary, r.stdout + r.stderr


@pytest.mark.skipif(not UNIT_REF.exists(), reason="oracle/_ref/unit_ref not built")
def test_reference_unit_tests_pass_on_reference_headers():
    rc, summary, out = _run(UNIT_REF)
    assert rc == 0, out
    assert "failed: 0" in summary and "test cases: 73" in summary, summary


@pytest.mark.skipif(not UNIT_DROPIN.exists(), reason="oracle/_ref/unit_dropin not built")
def test_reference_unit_tests_pass_on_dropin_host_cases():
    rc, summary, out = _run(UNIT_DROPIN, *["!" + c for c in DEVICE_CASES])
    assert rc == 0, out
    assert f"test cases: {73 - len(DEVICE_CASES)}" in summary and "failed: 0" in summary, summary


@pytest.mark.gpu
@pytest.mark.skipif(not UNIT_DROPIN.exists(), reason="oracle/_ref/unit_dropin not built")
def test_reference_unit_tests_pass_on_dropin_gpu():
    rc, summary, out = _run(UNIT_DROPIN)
    assert rc == 0, out
    assert "test cases: 73" in summary and "failed: 0" in summary, summary


DRAW_CHECK = oracle.HERE / "_ref" / "draw_check"


@pytest.mark.skipif(not DRAW_CHECK.exists(), reason="oracle/_ref/draw_check not built")
def test_shadow_bounded_draws_equal_reference_rng():
    """detail::draw_index (cached reciprocal) == Rng::index (rng.hpp:20-32),
    one million draws over a sweep of bounds, engine states equal after."""
    rc, summary, out = _run(DRAW_CHECK)
    assert rc == 0 and '"mismatches": 0' in summary, out


IO_REF = oracle.HERE / "_ref" / "io_check_ref"
IO_DROPIN = oracle.HERE / "_ref" / "io_check_dropin"


@pytest.mark.skipif(not (IO_REF.exists() and IO_DROPIN.exists()), reason="oracle/_ref/io_check_* not built")
def test_result_files_byte_identical(tmp_path):
    """include/ebic/io.hpp (result files written without a per-row JSON DOM)
    against the reference io.hpp: result files (empty, no run summary, up to
    ~200k rows per bicluster), truth and score files, read-back, plateau
    thresholds, config parsing and error texts -- byte for byte."""
    outs = {}
    for name, exe in (("ref", IO_REF), ("dropin", IO_DROPIN)):
        d = tmp_path / name
        d.mkdir()
        r = subprocess.run([str(exe), str(d)], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        files = {p.name: p.read_bytes() for p in sorted(d.iterdir())}
        outs[name] = (r.stdout.replace(str(d), "<dir>"), files)
    assert outs["ref"][0] == outs["dropin"][0]
    assert outs["ref"][1].keys() == outs["dropin"][1].keys() and len(outs["ref"][1]) == 8
    for k in outs["ref"][1]:
        assert outs["ref"][1][k] == outs["dropin"][1][k], k
