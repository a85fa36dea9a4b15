#!/usr/bin/env python
"""Executed warp instructions / stall samples of an `ncu --page source --csv` export, grouped by
phase of the tile kernels (line ranges located by marker strings in the current sources)."""
import collections
import csv
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_2006_09299_b200", "csrc")
MARKS = {
    "tile_ccl.cuh": [("helpers", "__device__ __forceinline__ int run_at("), ("tile_runs", "bool tile_runs("),
                     ("events", "__device__ bool ccl_tile("), ("first-contact", "---- first contact"),
                     ("prefix", "const int nev = __popc(ev)"), ("pre-flatten", "The first-contact forest links"),
                     ("union", "compact the warp's events into its queue"), ("roots", "---- roots (final now)"),
                     ("border-mark", "---- border components, marked"), ("scan/alloc", "---- tile components = root runs"),
                     ("map-pass", "---- every run: walk to its root"), ("rows/map-tail", "first component of each row"),
                     ("end", "}  // namespace rlg")],
    "kernels.cu": [("border_words", "__device__ __forceinline__ void border_words("),
                   ("a:load", "bool analyze_tile("), ("a:border-op", "The map pass of ccl_tile counts"),
                   ("a:hdr", "the two allocations are issued"), ("a:perimeter", "---- perimeter labels"),
                   ("a:nodes", "---- border-component nodes"), ("a:cnt/fg", "---- interior components per row"),
                   ("k_analyze", "class S: one CTA per tile"), ("merge", "M1: union across tile seams"),
                   ("e:prologue", "bool emit_tile("), ("e:runs", "runs again from the packed bits"),
                   ("e:features", "---- interior components, in chunks"), ("e:records", "pre-fill records, post-fill roots"),
                   ("e:dfold", "folds into interior survivors"), ("e:flush", "flush border-keyed folds"),
                   ("e:filled", "---- hole-filled image"), ("e:labels", "---- optional label image"),
                   ("end", "the sharded hole-fill accumulators")],
}


def ranges():
    out = []
    for f, marks in MARKS.items():
        lines = open(os.path.join(SRC, f)).read().splitlines()
        pos = []
        for name, m in marks:
            ln = next((i + 1 for i, s in enumerate(lines) if m in s), None)
            if ln is None:
                print(f"marker not found: {f}: {m}", file=sys.stderr)
                continue
            pos.append((ln, name))
        pos.sort()
        for (a, n), (b, _) in zip(pos, pos[1:]):
            out.append((f, a, b - 1, n))
    return out


def main():
    R = ranges()
    rows = list(csv.reader(open(sys.argv[1])))
    fname = None
    agg, aggs = collections.Counter(), collections.Counter()
    tot = tots = 0
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No"):
            continue
        if len(r) > 7 and r[2] == "-":
            try:
                s, ins, ln = int(r[4] or 0), int(r[7] or 0), int(r[0])
            except ValueError:
                continue
            tot += ins
            tots += s
            name = f"{fname}:other"
            for f, a, b, n in R:
                if f == fname and a <= ln <= b:
                    name = n
            agg[name] += ins
            aggs[name] += s
    print(f"total warp instructions {tot}")
    for k, v in agg.most_common():
        print(f"{k:34s} inst {100 * v / tot:5.1f}%  stall {100 * aggs[k] / max(tots, 1):5.1f}%")


if __name__ == "__main__":
    main()
