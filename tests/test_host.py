"""CPU tests of the host side: the C-ABI library loads and exports every symbol the header
declares (no compute without a GPU), the Python mirror's argument checking and host-side
projections, the C++ drop-in compiles, and the multi-rank plumbing under gloo."""
from __future__ import annotations

import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols() -> list[str]:
    src = open(os.path.join(ROOT, "include", "runlab_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rl_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2006_09299_b200 import _native
    lib = _native.load()
    syms = header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_native.EXPORTED_SYMBOLS) <= set(syms)


def test_library_is_sm100a():
    lib = os.path.join(ROOT, "paper_2006_09299_b200", "librunlab_gpu.so")
    out = subprocess.run(["cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_tile_shape_query():
    import ctypes as C
    from paper_2006_09299_b200 import _native
    th, tw = C.c_int32(), C.c_int32()
    _native.load().rl_tile_shape(C.byref(th), C.byref(tw))
    assert (th.value, tw.value) == (32, 256)


def test_cfg4_params_host_side():
    from oracle import oracle as O
    from paper_2006_09299_b200.runlab import cfg2_cells, cfg4_params
    assert [cfg4_params(i) for i in range(32)] == [O.cfg4_params(i) for i in range(32)]
    cells = cfg2_cells()
    assert len(cells) == 105 and cells[0] == (0.0, 1) and cells[-1] == (1.0, 16)


def test_config_errors_raise_before_device():
    from paper_2006_09299_b200 import LabelingConfig, label_image
    with pytest.raises(ValueError):
        label_image(np.zeros((1, 1), np.uint8), LabelingConfig(densify_labels=True))
    with pytest.raises(ValueError):
        label_image(np.zeros((0, 3), np.uint8), LabelingConfig())


def _fig3_result(fill: bool):
    """A LabelingResult as the GPU returns it for Fig. 3 (canonical ids), built by hand."""
    from paper_2006_09299_b200 import runlab as R
    from paper_2006_09299_b200._native import FEATURE_DTYPE
    t = np.array([0, 1, 1] if fill else [0, 1, 2], dtype=np.uint32)
    feats = np.zeros(3, dtype=FEATURE_DTYPE)
    feats["s"] = [38, 67 if fill else 56, 11]
    return R.LabelingResult(width=15, height=7, config=R.LabelingConfig(fill_holes=fill, compute_euler=True),
                            equivalences=R.EquivalenceTable(t=t, parity=np.array([0, 1, 0], np.uint8)),
                            adjacency=np.array([R.NO_LABEL, 0, 1], np.uint32), features=feats,
                            fg_count=1, hole_count=1, euler=0)


def test_analysis_projections_host_side():
    from paper_2006_09299_b200 import runlab as R
    res = _fig3_result(False)
    comps = R.components(res)
    assert [c.root for c in comps] == [0, 1, 2] and [c.depth for c in comps] == [0, 1, 2]
    assert [h.root for h in R.holes(res)] == [2]
    tree = R.adjacency_tree(res)
    assert tree.children == [[1], [2], []]
    assert R.euler_number(res) == 0
    filled = _fig3_result(True)
    assert filled.roots() == [0, 1]
    with pytest.raises(R.LogicError):
        R.holes(filled)
    res.euler = None
    with pytest.raises(R.LogicError):
        R.euler_number(res)
    labels = np.array([[0, 1, 2, 1]], np.uint32)
    assert list(R.binarize_labels(labels, res.equivalences)[0]) == [0, 1, 0, 1]


def test_cpp_dropin_header_compiles():
    for src in (os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp"), os.path.join(ROOT, "tools", "runlab_gpu.cpp")):
        out = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I" + os.path.join(ROOT, "include"), src],
                             capture_output=True, text=True)
        assert out.returncode == 0, out.stderr


def test_shard_range():
    from paper_2006_09299_b200.distributed import shard_range
    for n in (0, 1, 7, 105, 4096):
        for world in (1, 2, 3, 8):
            parts = [shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [hi - lo for lo, hi in parts]
            assert max(sizes) - min(sizes) <= 1


def test_balanced_shards():
    from paper_2006_09299_b200.distributed import balanced_shards, image_cost
    from paper_2006_09299_b200.runlab import cfg2_cells
    costs = [image_cost(d, g) for d, g in cfg2_cells()]
    for world in (1, 2, 3, 4, 8):
        parts = balanced_shards(costs, world)
        assert sorted(i for p in parts for i in p) == list(range(105))
        loads = [sum(costs[i] for i in p) for p in parts]
        # LPT: the heaviest rank exceeds the lightest by at most the largest item
        assert max(loads) - min(loads) <= max(costs) + 1e-9
        assert parts == balanced_shards(costs, world)  # deterministic
    assert balanced_shards([1.0] * 5, 8)[5:] == [[], [], []]


def test_bench_relaunch_command(monkeypatch):
    """`bench.py --gpus N` outside torchrun re-runs itself under torch.distributed.run."""
    import sys
    sys.path.insert(0, ROOT)
    import bench
    seen = {}

    def fake_call(cmd, env=None):
        seen["cmd"], seen["env"] = cmd, env
        return 0

    monkeypatch.setattr(bench.subprocess, "call", fake_call)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "5"])
    assert bench.relaunch_distributed(4) == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert "127.0.0.1" in cmd and cmd[-4:] == ["--gpus", "4", "--steps", "5"]
    assert seen["env"]["NCCL_DEBUG"] == "INFO"


def _gloo_worker(rank, world, port, q):
    import sys
    import torch.distributed as dist
    from paper_2006_09299_b200.distributed import max_over_ranks, shard_range, sum_over_ranks
    sys.path.insert(0, ROOT)
    import bench
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    lo, hi = shard_range(105, rank, world)
    t = max_over_ranks(1.0 + rank)
    n = sum_over_ranks(hi - lo)
    mine = {c: [s[1:] for s in bench.Workload(c).local_specs(rank, world)] for c in ("cfg2", "cfg4")}
    counts = {c: sum_over_ranks(len(v)) for c, v in mine.items()}
    dist.destroy_process_group()
    q.put((rank, t, n, mine, counts))


def test_multirank_reductions_gloo():
    """world_size-2 gloo run of the bench's N>1 plumbing: shard, max-time, sum."""
    import multiprocessing as mp
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=120) for _ in procs), key=lambda r: r[0])  # before join: large items
    for p in procs:
        p.join(120)
    assert [r[1] for r in res] == [2.0, 2.0]
    assert [r[2] for r in res] == [105, 105]
    # the bench's batch sharding: every image on exactly one rank, both ranks agree on the split
    import bench
    for c, total in (("cfg2", 105), ("cfg4", 4096)):
        assert [r[4][c] for r in res] == [total, total]
        both = sorted(res[0][3][c] + res[1][3][c])
        assert both == sorted(s[1:] for s in bench.Workload(c).specs)


def test_strip_rows():
    from paper_2006_09299_b200.strips import strip_rows
    for H in (32, 33, 1000, 1024, 32768):
        for n in (1, 2, 3, 5, 8):
            if n > (H + 31) // 32:
                with pytest.raises(ValueError):
                    strip_rows(H, n)
                continue
            rows = strip_rows(H, n)
            assert len(rows) == n
            assert rows[0][0] == 0 and sum(h for _, h in rows) == H
            for (y0, h), (y1, _) in zip(rows, rows[1:]):
                assert y0 % 32 == 0 and h % 32 == 0 and y0 + h == y1


def _strip_coll_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2006_09299_b200.strips import TorchCollectives, _max_classes
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    coll = TorchCollectives()
    infos = coll.gather_infos(np.array([10 + rank, 3 * rank, rank, 4 * rank, 4 * rank + 4], dtype=np.int64), "cpu")
    rec = torch.full((16,), rank + 1, dtype=torch.uint8)
    gathered = coll.gather_records(rec)
    links = torch.zeros(6, dtype=torch.int64)
    links[2 * rank] = 7 + rank
    links[2 * rank + 1] = -(rank + 1)
    coll.reduce_links(links)
    psum = torch.tensor([rank + 1] * 3, dtype=torch.int64)
    pmin = torch.tensor([5 - rank, 7 + rank], dtype=torch.int32)
    pmax = torch.tensor([5 - rank, 7 + rank], dtype=torch.int32)
    pcnt = torch.tensor([2 * rank + 1], dtype=torch.int64)
    coll.reduce_partials(psum, pmin, pmax, pcnt)
    dist.destroy_process_group()
    q.put((rank, infos.tolist(), _max_classes(infos), gathered.tolist(), links.tolist(), psum.tolist(),
           pmin.tolist(), pmax.tolist(), pcnt.tolist()))


def test_strip_collectives_gloo():
    """world_size-2 gloo run of the strip exchange's four collectives (host side of §8(e))."""
    import multiprocessing as mp
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_strip_coll_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = sorted(q.get(timeout=10) for _ in procs)
    for _, infos, mx, gathered, links, psum, pmin, pmax, pcnt in res:
        assert infos == [[10, 0, 0, 0, 4], [11, 3, 1, 4, 8]]
        assert mx == 11
        assert gathered == [1] * 16 + [2] * 16
        assert links == [7, -1, 8, -2, 0, 0]
        assert psum == [3, 3, 3] and pmin == [4, 7] and pmax == [5, 8] and pcnt == [4]


def test_bench_reference_arm_json_contract():
    """`bench.py --impl reference` (the driver's reference arm): one JSON line with the contract's
    keys, the reference's own CPU path from oracle/_ref, same metric/config as our arm."""
    import json
    import sys
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "cfg1",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    if "unavailable" in line:
        pytest.skip(line["unavailable"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["unit"] == "Gpixel/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    import bench
    assert line["metric"] == bench.METRIC and line["config"]["workload"].startswith("cfg1")
