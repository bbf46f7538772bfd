"""The `bitedge` CLI: exit codes and I/O errors on CPU, the
golden fixtures of SPEC acceptance 7 through real PBM files on the GPU."""

import numpy as np
import pytest

from paper_1401_5245_b200.cli import generate, main, read_pgm


def test_usage_errors_exit_2(tmp_path, capsys):
    assert main(["detect", "--input", str(tmp_path / "missing.pbm"), "--output",
                 str(tmp_path / "o.pbm")]) == 2
    assert "missing.pbm" in capsys.readouterr().err
    assert main(["compare", "--input", str(tmp_path / "missing.pbm")]) == 2
    assert main(["bench", "--repeats", "2"]) == 2
    assert main(["bench", "--sizes", "4"]) == 2
    pgm = tmp_path / "g.pgm"
    pgm.write_bytes(b"P2\n2 1\n255\n0 255\n")
    assert main(["binarize", "--input", str(pgm), "--output", str(tmp_path / "b.pbm"),
                 "--threshold", "128", "--otsu"]) == 2
    with pytest.raises(SystemExit) as e:
        main(["nonsense"])
    assert e.value.code == 2


def test_read_pgm_examples():
    assert read_pgm(b"P2\n2 1\n255\n0 255\n").tolist() == [[0, 255]]
    assert read_pgm(b"P5\n2 1\n255\n\x00\xff").tolist() == [[0, 255]]
    with pytest.raises(ValueError, match="offset"):
        read_pgm(b"P5\n2 1\n255\n\x00")
    with pytest.raises(ValueError, match="255"):
        read_pgm(b"P2\n1 1\n65535\n7\n")


def test_generators_deterministic():
    for shape in ("glyph", "rect", "disk", "noise"):
        a = generate(shape, 64, 0.5, seed=3)
        assert a.shape == (64, 64) and (a == generate(shape, 64, 0.5, seed=3)).all()
    assert generate("noise", 32, 0.0).all()


def _pbm_p1(a):
    black = 1 - np.asarray(a)
    return (f"P1\n{a.shape[1]} {a.shape[0]}\n" + "\n".join(
        " ".join(str(int(v)) for v in row) for row in black) + "\n").encode()


@pytest.mark.gpu
def test_golden_fixtures_via_cli(tmp_path, cuda_dev, capsys):
    from paper_1401_5245_b200.pbm import read_pbm, write_pbm
    from paper_1401_5245_b200.bitimage import BitImage

    cases = []
    block = np.ones((5, 5), np.uint8)
    block[1:4, 1:4] = 0
    ring = np.ones((5, 5), np.uint8)
    ring[1:4, 1:4] = 0
    ring[2, 2] = 1
    cases.append((block, ring))                                    # 5x5 centred block -> ring
    rect = np.ones((9, 12), np.uint8)
    rect[2:7, 3:10] = 0
    rring = rect.copy()
    rring[3:6, 4:9] = 1
    cases.append((rect, rring))                                    # filled rectangle -> boundary
    stroke = np.ones((8, 10), np.uint8)
    stroke[2, 1:9] = 0
    stroke[3:7, 8] = 0
    cases.append((stroke, stroke))                                 # thin stroke -> fixed point
    for k, (inp, exp) in enumerate(cases):
        src = tmp_path / f"in{k}.pbm"
        src.write_bytes(write_pbm(BitImage.from_array(inp), raw=True))
        outs = []
        for method in ("mask", "scan"):
            dst = tmp_path / f"out{k}_{method}.pbm"
            assert main(["detect", "--input", str(src), "--output", str(dst),
                         "--method", method]) == 0
            outs.append(dst.read_bytes())
            assert (read_pbm(outs[-1]).to_array() == exp).all(), (k, method)
        assert outs[0] == outs[1]                                  # byte-identical
        assert outs[0] == write_pbm(BitImage.from_array(exp), raw=True)
        assert main(["compare", "--input", str(src)]) == 0
        assert "MATCH" in capsys.readouterr().out
        p1 = tmp_path / f"p1_{k}.pbm"
        p1.write_bytes(_pbm_p1(inp))
        d1 = tmp_path / f"p1_{k}_out.pbm"
        assert main(["detect", "--input", str(p1), "--output", str(d1), "--raw-output",
                     "false"]) == 0
        assert read_pbm(d1.read_bytes()).to_array().tolist() == exp.tolist()
    assert main(["info", "--input", str(tmp_path / "in0.pbm")]) == 0
    assert capsys.readouterr().out.strip() == "5x5 black=9"
    bad = tmp_path / "trunc.pbm"
    bad.write_bytes(b"P4\n16 4\n\x00")
    assert main(["detect", "--input", str(bad), "--output", str(tmp_path / "x.pbm")]) == 2
    assert "offset" in capsys.readouterr().err


@pytest.mark.gpu
def test_binarize_and_otsu(tmp_path, cuda_dev, capsys):
    from paper_1401_5245_b200.cli import otsu_threshold
    from paper_1401_5245_b200.pbm import read_pbm

    pgm = tmp_path / "g.pgm"
    pgm.write_bytes(b"P2\n2 1\n255\n0 255\n")
    out = tmp_path / "b.pbm"
    assert main(["binarize", "--input", str(pgm), "--output", str(out), "--threshold", "128"]) == 0
    assert read_pbm(out.read_bytes()).to_array().tolist() == [[0, 1]]
    assert otsu_threshold(np.full((4, 4), 77, np.uint8)) == 0
    assert otsu_threshold(np.array([[0, 255]], np.uint8)) == 1
    bim = np.array([[10] * 8 + [200] * 8], np.uint8)
    t = otsu_threshold(bim)
    assert 10 < t <= 200
    assert main(["binarize", "--input", str(pgm), "--output", str(out), "--otsu"]) == 0
    assert "threshold=" in capsys.readouterr().out


@pytest.mark.gpu
def test_bench_table(tmp_path, cuda_dev, capsys):
    csv = tmp_path / "t.csv"
    assert main(["bench", "--sizes", "50,100", "--shape", "rect", "--repeats", "3",
                 "--csv", str(csv)]) == 0
    lines = csv.read_text().splitlines()
    assert lines[0] == "label,width,height,scan_ms,mask_ms,speedup,repeats"
    assert [l.split(",")[1] for l in lines[1:]] == ["50", "100"]             # ascending
