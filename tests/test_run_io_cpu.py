"""Run I/O around the path, host side: PRSPAR01
arrays, datasets, SHA-256 and number formatting through the C ABI, checked
against the reference's own array_io.cpp / sha256.cpp (oracle/_ref). No GPU
compute is involved, so these run in the CPU suite.
"""
import os

import numpy as np
import pytest


@pytest.fixture(scope="module")
def rio():
    from paper_1908_06843_b200 import run_io

    return run_io


def test_array_bytes_match_reference(rio, ref, tmp_path):
    a = np.random.default_rng(0).normal(size=(9, 4))
    rio.save_array(tmp_path / "ours.prsp", a)
    ref.save_array(tmp_path / "ref.prsp", a)
    assert (tmp_path / "ours.prsp").read_bytes() == (tmp_path / "ref.prsp").read_bytes()
    assert np.array_equal(rio.load_array(tmp_path / "ref.prsp"), a)
    assert np.array_equal(rio.load_dataset(tmp_path / "ours.prsp"), ref.load_dataset(tmp_path / "ours.prsp"))


def test_array_errors(rio, tmp_path):
    from paper_1908_06843_b200 import DataError

    (tmp_path / "bad.prsp").write_bytes(b"NOTMAGIC" + bytes(16))
    with pytest.raises(DataError):
        rio.load_array(tmp_path / "bad.prsp")
    rio.save_array(tmp_path / "t.prsp", np.ones((4, 4)))
    (tmp_path / "short.prsp").write_bytes((tmp_path / "t.prsp").read_bytes()[:40])
    with pytest.raises(DataError):  # payload shorter than header promises (array_io.cpp:82-83)
        rio.load_array(tmp_path / "short.prsp")
    (tmp_path / "near.bin").write_bytes(b"PRSPxx01" + bytes(16))
    with pytest.raises(DataError):  # near-magic prefix is not a CSV (array_io.cpp:149-151)
        rio.load_dataset(tmp_path / "near.bin")


def test_csv_matches_reference(rio, ref, tmp_path):
    (tmp_path / "x.csv").write_text("1, 2,3\n\n4,5 ,6e-3\r\n-7,8.5,9\n")
    assert np.array_equal(rio.load_dataset(tmp_path / "x.csv"), ref.load_dataset(tmp_path / "x.csv"))
    from paper_1908_06843_b200 import DataError

    (tmp_path / "r.csv").write_text("1,2\n3\n")
    with pytest.raises(DataError):
        rio.load_dataset(tmp_path / "r.csv")
    (tmp_path / "e.csv").write_text("\n\n")
    with pytest.raises(DataError):
        rio.load_dataset(tmp_path / "e.csv")


def test_sha256(rio, ref, tmp_path):
    # FIPS 180-4 example digests
    assert rio.sha256_hex(b"") == "e3b0c44298fc1c149afbf4c8996fb92427ae41e4649b934ca495991b7852b855"
    assert rio.sha256_hex(b"abc") == "ba7816bf8f01cfea414140de5dae2223b00361a396177a9cb410ff61f20015ad"
    for b in [b"a" * 55, b"a" * 56, b"a" * 64, bytes(range(256)) * 9]:
        assert rio.sha256_hex(b) == ref.sha256(b)
    p = tmp_path / "blob"
    p.write_bytes(os.urandom(3 * 1024 * 1024 + 17))
    assert rio.sha256_file(p) == ref.sha256_file(p)


def test_format_double(rio, ref):
    for v in [0.0, -0.0, 0.1, 1.0, 1e22, 5e-324, -2.5e-300, 123456.789, np.pi, 1 / 3]:
        assert rio.format_double(v) == ref.format_double(v)
