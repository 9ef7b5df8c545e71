"""Differential parity against golden vectors produced by the REFERENCE
package (tests/golden/make_golden.py): loop trees, verdicts, genome maps,
transfer plans (directives and notes), emitted text, exec counts, simulated
times, GA histories and tune reports must match exactly -- floats included.
"""

from __future__ import annotations

import hashlib
import json
import tempfile
from pathlib import Path

import pytest

import paper_1811_03882_b200 as at
from paper_1811_03882_b200 import cli
from paper_1811_03882_b200.legality import profile_from_dict

from conftest import golden_programs, golden_reports

NAMES = sorted(golden_programs())


def sha(text: str) -> str:
    return hashlib.sha256(text.encode()).hexdigest()


def table_seconds(bits: str) -> float:
    h = int(hashlib.sha256(bits.encode()).hexdigest()[:8], 16)
    return 0.5 + (h % 100000) / 10000.0


def _load(entry):
    program = at.parse(entry["source"])
    tree = at.build_loop_tree(program)
    accesses = at.extract_accesses(program)
    return program, tree, accesses


def _model(entry):
    if entry["model"] is None:
        return None
    with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as fh:
        json.dump(entry["model"], fh)
    return at.load_cost_model(fh.name)


@pytest.mark.parametrize("name", NAMES)
def test_front_end_matches_reference(name):
    g = golden_programs()[name]
    program, tree, accesses = _load(g)
    loops = [[n.loop_id, n.kind, n.parent, n.function, n.header_pos.line, n.header_pos.col,
              n.canonical, n.counter] for n in tree.nodes]
    assert loops == g["loops"]
    assert len(accesses) == g["n_accesses"]
    digest = sha(json.dumps([[a.var, a.is_array, a.kind, a.pos.line, a.pos.col, a.pos.offset,
                              list(a.loop_path), a.function, a.header_of,
                              None if a.indices is None else [list(x) if x else None
                                                              for x in a.indices]]
                             for a in accesses]))
    assert digest == g["accesses_digest"]
    verdicts = at.check_all_parallelizable(tree, accesses)
    assert [[v.loop_id, v.eligible, v.reason] for v in verdicts] == g["verdicts"]


@pytest.mark.parametrize("name", NAMES)
def test_plans_emission_counts_match_reference(name):
    g = golden_programs()[name]
    program, tree, accesses = _load(g)
    gm = at.build_genome_map(at.check_all_parallelizable(tree, accesses))
    assert list(gm.loop_ids) == g["genome_map"]
    prof = profile_from_dict(g["profile"], name, tree) if g["profile"] else None
    if prof is not None:
        d = at.gate(tree, prof)
        assert [d.passed, d.max_total_iterations, d.threshold, d.loop_id] == g["gate"]
    model = _model(g)
    for case in g["cases"]:
        bits = case["genome"]
        assert at.check_genome_valid(bits, gm, tree) == case["valid"]
        if not case["valid"]:
            with pytest.raises(at.InvalidGenome):
                at.plan_transfers(program, tree, accesses, bits, gm)
            continue
        plan = at.plan_transfers(program, tree, accesses, bits, gm)
        got = {"directives": [[d.target_loop, d.clause, list(d.vars), d.origin_region]
                              for d in plan.directives], "notes": list(plan.notes)}
        assert got == case["plan"], bits
        ann = at.emit_annotated(program, tree, bits, gm, plan)
        assert sha(ann.text) == case["emitted_sha256"]
        assert [[i.line_no, i.content] for i in ann.inserted_lines] == case["inserted"]
        assert at.strip_annotations(ann) == g["source"]
        if prof is not None:
            counts = at.directive_exec_counts(plan, tree, prof)
            assert [counts[d] for d in plan.directives] == case["exec_counts"]
            assert sum(at.directive_exec_counts(at.unhoisted(plan), tree, prof).values()) \
                == case["unhoisted_exec_total"]
        if model is not None and prof is not None:
            assert at.simulate_time(model, bits, gm, tree, prof, plan).seconds == case["sim_seconds"]
    if "expected_emitted" in g:
        bits = "1" * len(gm)
        plan = at.plan_transfers(program, tree, accesses, bits, gm)
        assert at.emit_annotated(program, tree, bits, gm, plan).text == g["expected_emitted"]


def _result_json(res):
    return {
        "best": [res.best.genome, res.best.seconds, res.best.fitness, res.best.status],
        "history": [[s.generation, s.best_seconds, s.best_fitness, s.mean_fitness,
                     s.evaluations_performed, s.cache_hits] for s in res.history],
        "gene_length": res.gene_length, "effective_population": res.effective_population,
        "evaluations": res.evaluations_performed, "cache_hits": res.cache_hits,
    }


@pytest.mark.parametrize("name", NAMES)
def test_ga_histories_match_reference(name):
    g = golden_programs()[name]
    program, tree, accesses = _load(g)
    gm = at.build_genome_map(at.check_all_parallelizable(tree, accesses))
    prof = profile_from_dict(g["profile"], name, tree) if g["profile"] else None
    model = _model(g)
    for run in g["ga"]["runs"]:
        cfg = at.GAConfig(rng_seed=run["seed"], **g["ga"]["config"])
        if run["evaluator"] == "table":
            calls = []

            def ev(bits, _c=calls):
                _c.append(bits)
                return at.Measurement(table_seconds(bits), "measured")
            res = at.run_ga(cfg, gm, tree, ev, at.MeasurementCache())
            assert calls == run["calls"]
        else:
            ev = at.make_sim_evaluator(model, program, tree, accesses, gm, prof)
            res = at.run_ga(cfg, gm, tree, ev, at.MeasurementCache())
        assert _result_json(res) == run["result"], (name, run["seed"], run["evaluator"])


def test_ga_is_independent_of_worker_count():
    g = golden_programs()["yolov2-tiny"]
    program, tree, accesses = _load(g)
    gm = at.build_genome_map(at.check_all_parallelizable(tree, accesses))
    run = next(r for r in g["ga"]["runs"] if r["evaluator"] == "table")

    def ev(bits):
        return at.Measurement(table_seconds(bits), "measured")
    cfg = at.GAConfig(rng_seed=run["seed"], workers=8, **g["ga"]["config"])
    assert _result_json(at.run_ga(cfg, gm, tree, ev)) == run["result"]


@pytest.mark.parametrize("idx", range(len(golden_reports())))
def test_tune_reports_match_reference(idx, tmp_path):
    rep = golden_reports()[idx]
    g = golden_programs()[rep["name"]]
    (tmp_path / "p.c").write_text(g["source"])
    (tmp_path / "p_profile.json").write_text(json.dumps(g["profile"]))
    (tmp_path / "p_model.json").write_text(json.dumps(g["model"]))
    code = cli.main(["tune", "--source", str(tmp_path / "p.c"), "--profile",
                     str(tmp_path / "p_profile.json"), "--evaluator",
                     f"sim:{tmp_path}/p_model.json", "--seed", str(rep["seed"]),
                     "--out", str(tmp_path / "best.c"), "--report",
                     str(tmp_path / "report.json"), *rep["extra"]])
    assert code == rep["exit_code"]
    report = (tmp_path / "report.json").read_text().replace(str(tmp_path), "<tmp>")
    assert report == rep["report"]
    best = tmp_path / "best.c"
    assert (sha(best.read_text()) if best.exists() else None) == rep["best_sha256"]
