"""tools/runlab_gpu (the reference CLI's subcommands over the drop-in) end to end on PBM
files: gen, fill (device P4 path and P1), euler, tree, label with features CSV."""
from __future__ import annotations

import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "tools", "runlab_gpu")


@pytest.fixture(scope="module")
def cli():
    if not os.path.exists(CLI):
        import __graft_entry__ as g
        g.build_cli()
    return CLI


def run(cli, *args):
    return subprocess.run([cli, *args], capture_output=True, text=False, check=True).stdout


def test_gen_fill_euler(cli, tmp_path):
    src, dst, dst1 = tmp_path / "in.pbm", tmp_path / "out.pbm", tmp_path / "out1.pbm"
    run(cli, "gen", str(src), "--width", "777", "--height", "333", "--density", "0.55", "--granularity", "2",
        "--seed", "9")
    img = O.generate(777, 333, 0.55, 2, 9)
    assert src.read_bytes() == O.ref_write_pbm(img)  # generator.hpp + write_pbm, bit for bit
    run(cli, "fill", str(src), str(dst))
    want = O.label_canonical(img, 0).filled_image
    assert dst.read_bytes() == O.ref_write_pbm(want)
    run(cli, "fill", str(src), str(dst1), "--format", "p1")
    assert dst1.read_bytes() == O.ref_write_pbm(want, p1=True)
    assert int(run(cli, "euler", str(src))) == O.bitquad_euler(img, 0)
    assert int(run(cli, "euler", str(src), "--connectivity", "fg4bg8")) == O.bitquad_euler(img, 1)


def test_label_features_and_tree(cli, tmp_path):
    img = O.generate(300, 200, 0.5, 4, 3)
    src = tmp_path / "in.pbm"
    src.write_bytes(O.ref_write_pbm(img))
    fcsv = tmp_path / "f.csv"
    out = run(cli, "label", str(src), "--features-csv", str(fcsv)).decode()
    can = O.label_canonical(img, 0)
    assert f"foreground components: {can.n_fg}" in out and f"euler: {can.euler}" in out
    rows = fcsv.read_text().strip().split("\n")
    assert rows[0] == "root,parity,parent,s,sx,sy,rmin,rmax,cmin,cmax"
    assert len(rows) == 1 + can.n_components
    for line, c, i in zip(rows[1:], can.comps, range(can.n_components)):
        f = line.split(",")
        assert int(f[0]) == i and f[1] == ("FG" if c["flags"] & 1 else "BG")
        assert (f[2] == "" if i == 0 else int(f[2]) == c["parent"])
        assert [int(v) for v in f[3:6]] == [c["s"], c["sx"], c["sy"]]
    dot = run(cli, "tree", str(src)).decode()
    assert dot.startswith("digraph components {\n") and dot.count(" -> ") == can.n_components - 1
    js = run(cli, "tree", str(src), "--format", "json").decode()
    assert js.startswith('{"label":0,') and js.count('"label":') == can.n_components


def test_parse_error_offset(cli, tmp_path):
    bad = tmp_path / "bad.pbm"
    bad.write_bytes(b"P4\n9 2\n\x80\xff")
    r = subprocess.run([cli, "euler", str(bad)], capture_output=True)
    assert r.returncode == 1 and b"truncated P4 raster (byte 9)" in r.stderr


def test_bench_sweep_csv(cli, tmp_path):
    """runlab bench (tools/runlab.cpp:245-275, bench.hpp:89-207): same sweep, variants, rows and
    CSV columns; step times are the device phases."""
    out = tmp_path / "b.csv"
    run(cli, "bench", "--size", "256", "--densities", "0.2:0.5:0.3", "--granularities", "1,4", "--seeds", "2",
        "--iters", "2", "--clock-ghz", "2.0", "-o", str(out))
    rows = out.read_text().strip().split("\n")
    assert rows[0] == "d,g,config,step,min_ns_px,med_ns_px,max_ns_px,min_cpp,med_cpp,max_cpp"
    body = [r.split(",") for r in rows[1:]]
    # per cell: base encode/unify/closure/total, then euler/fill/features (total, extra) and
    # relabel (relabel, total, extra)
    assert len(body) == 2 * 2 * 13
    assert [b[2] + ":" + b[3] for b in body[:13]] == [
        "base:encode", "base:unify", "base:closure", "base:total", "euler:total", "euler:extra", "fill:total",
        "fill:extra", "features:total", "features:extra", "relabel:relabel", "relabel:total", "relabel:extra"]
    assert {(b[0], b[1]) for b in body} == {("0.2", "1"), ("0.2", "4"), ("0.5", "1"), ("0.5", "4")}
    for b in body:
        mn, md, mx = float(b[4]), float(b[5]), float(b[6])
        assert mn <= md <= mx
        if b[3] != "extra":
            assert mn > 0 and abs(float(b[8]) - 2.0 * md) < 1e-3 * max(1.0, md)
    txt = run(cli, "bench", "--size", "64", "--densities", "0.5", "--granularities", "2", "--seeds", "1",
              "--iters", "1", "--no-euler", "--no-fill", "--no-features", "--no-relabel").decode()
    assert len(txt.strip().split("\n")) == 1 + 4 and txt.strip().endswith(",,,")
