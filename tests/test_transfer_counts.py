"""Memcpy counts re-derived from the REFERENCE's emitted source (CPU).

The executor's expected `h2d_calls` / `d2h_calls` (and bytes) come from its
own action list.  Here they are derived independently, from the
`#pragma acc data` lines the reference emitter inserted for each golden
genome (tests/golden/reference_programs.json, recorded by
tests/golden/make_golden.py from `acctuner.emit_annotated`):

* a data line precedes its target loop's header; its clauses are the
  per-target unions of the planner's directives (`emitter.py:41-49`);
* the line executes once per entry of that loop (`directive_exec_counts`,
  `transfer.py:161-165`, entry counts from the golden profile): copyin and
  copy variables go host->device before the loop, copyout and copy
  variables device->host after it -- one memcpy per variable per entry.
"""

from __future__ import annotations

import re

import pytest

from conftest import golden_programs
from paper_1811_03882_b200.executor import PatternExecutor
from paper_1811_03882_b200.nets import build_net

CLAUSE = re.compile(r"(copyin|copyout|copy)\(([^)]*)\)")


def pragma_counts(program_record: dict, inserted, net) -> dict:
    from paper_1811_03882_b200 import build_loop_tree, parse
    tree = build_loop_tree(parse(program_record["source"]))
    header = {}
    for n in tree.nodes:
        assert n.header_pos.line not in header
        header[n.header_pos.line] = n.loop_id
    entries = {lp["id"]: lp["entry_count"] for lp in program_record["profile"]["loops"]}
    lines = sorted((int(ln), text) for ln, text in inserted)
    inserted_at = {ln for ln, _ in lines}
    out = {"h2d_calls": 0, "d2h_calls": 0, "h2d_bytes": 0, "d2h_bytes": 0}
    for ln, text in lines:
        if not text.lstrip().startswith("#pragma acc data"):
            continue
        nxt = ln + 1
        while nxt in inserted_at:
            nxt += 1
        loop = header[nxt - sum(1 for other, _ in lines if other < nxt)]
        clauses: dict[str, set] = {}
        for clause, names in CLAUSE.findall(text):
            clauses.setdefault(clause, set()).update(v for v in names.split(",") if v)
        ins = clauses.get("copy", set()) | clauses.get("copyin", set())
        outs = clauses.get("copy", set()) | clauses.get("copyout", set())
        for v in ins | outs:
            assert v in net.arrays, f"scalar {v} in a data clause"
        n = entries[loop]
        out["h2d_calls"] += n * len(ins)
        out["d2h_calls"] += n * len(outs)
        out["h2d_bytes"] += n * sum(net.arrays[v].nbytes for v in ins)
        out["d2h_bytes"] += n * sum(net.arrays[v].nbytes for v in outs)
    return out


@pytest.mark.parametrize("name", ["micro", "demo", "yolov2-tiny"])
def test_memcpy_counts_equal_emitted_pragmas_times_entries(name):
    rec = golden_programs()[name]
    net = build_net(name)
    assert net.source == rec["source"]
    ex = PatternExecutor(net, device=None)
    checked = 0
    for case in rec["cases"]:
        if not case["valid"]:
            continue
        want = pragma_counts(rec, case["inserted"], net)
        got = ex.compile(case["genome"]).expected
        for key, val in want.items():
            assert got[key] == val, (name, case["genome"], key, got[key], val)
        checked += 1
    assert checked >= 10
