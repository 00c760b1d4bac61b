"""File formats (PGM, IHST), the CSV harness schema and the CLI surface.

CPU tests: byte compatibility with the reference's formats (golden crcs made
by the reference, tests/golden/formats.json), parser errors, and the CLI exit
codes for failures raised before any device work.  GPU tests: the CLI
end-to-end and the device -> file IHST writer."""

import json
import os
import zlib

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import oracle as O
from paper_1711_01919_b200 import FormatError, GrayImage, IntegralHistogram
from paper_1711_01919_b200 import formats, harness
from paper_1711_01919_b200.cli import main


@pytest.fixture(scope="module")
def fx():
    with open(os.path.join(GOLDEN, "formats.json")) as fh:
        return json.load(fh)


def _synth(w, h, seed=0):
    return GrayImage(O.synth_image(w, h, seed))


def test_pgm_bytes_match_reference(fx):
    data = formats.write_pgm(_synth(23, 17))
    assert len(data) == fx["pgm_len"] and f"{zlib.crc32(data):08x}" == fx["pgm_crc"]
    back = formats.read_pgm(data)
    assert back.pixels.tobytes() == _synth(23, 17).pixels.tobytes()


def test_ihst_bytes_match_reference(fx):
    img = _synth(23, 17)
    counts = O.compute_sequential(img.pixels, O.np_uniform_table(8), 8)
    data = formats.serialize_ih(IntegralHistogram(counts))
    assert len(data) == fx["ihst_len"] and f"{zlib.crc32(data):08x}" == fx["ihst_crc"]
    assert np.array_equal(formats.deserialize_ih(data).counts, counts)


def test_map_pgm_matches_reference(fx):
    data = formats.write_map_pgm(np.linspace(0, 1, 35).reshape(5, 7))
    assert f"{zlib.crc32(data):08x}" == fx["map_pgm_crc"]
    with pytest.raises(ValueError):
        formats.write_map_pgm(np.array([[1.5]]))


def test_minimal_tensor_is_20_bytes():
    assert len(formats.serialize_ih(IntegralHistogram(np.ones((1, 1, 1), np.uint32)))) == 20


@pytest.mark.parametrize("bad", [
    b"P6 1 1 255 \x00", b"P5", b"P51 1 255 \x00", b"P5 x 1 255 \x00", b"P5 1 1 65535 \x00\x00",
    b"P5 0 1 255 ", b"P5 2 2 255 \x00", b"P5 1 1 255",
])
def test_pgm_errors(bad):
    with pytest.raises(FormatError):
        formats.read_pgm(bad)


def test_pgm_comments_and_whitespace():
    img = formats.read_pgm(b"P5\n# a comment\n3 # w\n1\n255\n\x01\x02\x03")
    assert img.pixels.tolist() == [[1, 2, 3]]


def test_ihst_errors():
    good = formats.serialize_ih(IntegralHistogram(np.arange(6, dtype=np.uint32).reshape(1, 2, 3)))
    for bad in (good[:10], b"XXXX" + good[4:], good[:4] + b"\x02\x00" + good[6:], good[:-1],
                good[:6] + b"\x00\x00" + good[8:]):
        with pytest.raises(FormatError):
            formats.deserialize_ih(bad)


def test_tensor_file_sink_equals_serialize(tmp_path):
    counts = O.compute_sequential(O.synth_image(9, 7, 3), O.np_uniform_table(5), 5)
    path = tmp_path / "t.ihst"
    with formats.TensorFileSink(path, 9, 7, 5) as sink:
        sink.write(0, 2, 0, 7, counts[0:2])
        sink.write(2, 5, 0, 3, counts[2:5, 0:3])
        sink.write(2, 5, 3, 7, counts[2:5, 3:7])
    assert path.read_bytes() == formats.serialize_ih(IntegralHistogram(counts))
    # host tensors go straight through save_ihst
    p2 = tmp_path / "u.ihst"
    assert formats.save_ihst(p2, IntegralHistogram(counts)) == p2.stat().st_size
    assert p2.read_bytes() == path.read_bytes()


def test_harness_csv_schema():
    rec = harness.BenchRecord("crossweave", 4, 3, 2, 0, 0, 1, 1.5, 1.25, 666.666667, "deadbeef")
    text = harness.csv_text([rec])
    assert text.splitlines()[0] == harness.CSV_HEADER
    assert text.splitlines()[1] == "crossweave,4,3,2,0,0,1,1.500000,1.250000,666.666667,deadbeef"
    assert harness.synth_image(7, 5, 1).pixels.tobytes() == O.synth_image(7, 5, 1).tobytes()


# ------------------------------------------------------------------- CLI
def test_cli_usage_errors(tmp_path):
    assert main([]) == 2
    assert main(["compute", "--bins", "4"]) == 2
    bad = tmp_path / "bad.pgm"
    bad.write_bytes(b"P6 1 1 255 \x00\x00\x00")
    assert main(["compute", "--in", str(bad), "--bins", "2", "--out", str(tmp_path / "o")]) == 2
    assert main(["compute", "--in", str(tmp_path / "missing.pgm"), "--bins", "2",
                 "--out", str(tmp_path / "o")]) == 4
    src = tmp_path / "one.pgm"
    src.write_bytes(b"P5 1 1 255 \x07")
    assert main(["compute", "--in", str(src), "--bins", "300", "--out", str(tmp_path / "o")]) == 2
    assert main(["bench", "--sizes", "4by4", "--bins", "2", "--strategies", "sequential",
                 "--out", str(tmp_path / "b.csv")]) == 2
    assert main(["query", "--tensor", str(tmp_path / "missing.ihst"), "--region", "0,0,0,0"]) == 4


@pytest.mark.gpu
def test_cli_end_to_end(tmp_path, capsys):
    img = _synth(23, 17)
    src = tmp_path / "img.pgm"
    src.write_bytes(formats.write_pgm(img))
    expect = formats.serialize_ih(IntegralHistogram(
        O.compute_sequential(img.pixels, O.np_uniform_table(8), 8)))
    blobs = []
    for strat in ("sequential", "sts", "crossweave", "wavefront"):
        out = tmp_path / f"{strat}.ihst"
        assert main(["compute", "--in", str(src), "--bins", "8", "--strategy", strat,
                     "--out", str(out)]) == 0
        blobs.append(out.read_bytes())
    assert set(blobs) == {expect}
    out = tmp_path / "s.ihst"
    assert main(["compute", "--in", str(src), "--bins", "8", "--budget", "4000",
                 "--out", str(out)]) == 0
    assert out.read_bytes() == expect
    one = tmp_path / "one.pgm"
    one.write_bytes(b"P5 1 1 255 \x07")
    assert main(["compute", "--in", str(one), "--bins", "1", "--out", str(tmp_path / "m")]) == 0
    assert (tmp_path / "m").stat().st_size == 20
    assert main(["compute", "--in", str(src), "--bins", "4", "--strategy", "wavefront",
                 "--tile", "0", "--out", str(tmp_path / "w")]) == 2
    capsys.readouterr()
    assert main(["query", "--tensor", str(tmp_path / "sequential.ihst"),
                 "--region", "2,3,10,20"]) == 0
    lines = capsys.readouterr().out.split()
    got = [int(x) for x in lines]
    assert got == O.brute_region_counts(img.pixels, O.np_uniform_table(8), 8, 2, 3, 10, 20).tolist()
    assert main(["query", "--tensor", str(tmp_path / "sequential.ihst"),
                 "--region", "2,3,17,20"]) == 3
    assert main(["likelihood", "--in", str(src), "--bins", "8", "--template", "2,3,9,10",
                 "--out", str(tmp_path / "map.pgm")]) == 0
    r, c, score = capsys.readouterr().out.split()
    assert (int(r), int(c)) == (2, 3) and abs(float(score) - 1.0) < 1e-12
    csv = tmp_path / "b.csv"
    assert main(["bench", "--sizes", "64x64", "--bins", "16", "--strategies",
                 "sequential,crossweave,wavefront", "--reps", "1", "--out", str(csv)]) == 0
    rows = csv.read_text().splitlines()
    assert rows[0] == harness.CSV_HEADER and len(rows) == 4
    assert {r.split(",")[-1] for r in rows[1:]} == {"73c6c1fe"}


@pytest.mark.gpu
def test_save_ihst_streams_device_tensor(tmp_path):
    from paper_1711_01919_b200 import compute, BinSpec, CROSSWEAVE

    img = _synth(300, 200, 4)
    ih = compute(img, BinSpec.uniform(37), CROSSWEAVE)
    path = tmp_path / "d.ihst"
    formats.save_ihst(path, ih, group_bytes=3 * 300 * 200 * 4)  # several plane groups
    counts = O.compute_sequential(img.pixels, O.np_uniform_table(37), 37)
    assert path.read_bytes() == formats.serialize_ih(IntegralHistogram(counts))
