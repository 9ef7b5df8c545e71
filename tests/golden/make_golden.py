"""Generate golden vectors by running the REFERENCE package (acctuner) here.

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/make_golden.py            # rewrites tests/golden/*.json

For every program -- the reference's own fixtures (golden/, tune/, stress/)
and this repo's Darknet-style nets -- it records, as computed by the
reference code: loop tree, verdicts, genome map, plans (directives + notes)
and emitted-text digests for a seeded set of genomes, directive exec
counts, simulated times, GA histories (sim evaluator and a hash-table
evaluator) and tune reports.  Floats are stored through JSON's repr, so
equality checks are exact.  The fixture inputs are embedded in the output
so the tests need nothing from /root/reference at run time.
"""

from __future__ import annotations

import hashlib
import json
import random
import sys
import tempfile
from pathlib import Path

REF_SRC = Path("/root/reference/pkg/src")
REF_FIX = Path("/root/reference/pkg/tests/fixtures")
HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]

sys.dont_write_bytecode = True
sys.path.insert(0, str(REF_SRC))
sys.path.insert(1, str(REPO))

import acctuner as ref  # noqa: E402  (the reference implementation)
from acctuner import cli as ref_cli  # noqa: E402

from paper_1811_03882_b200.nets import build_net  # noqa: E402  (program text only)


def sha(text: str) -> str:
    return hashlib.sha256(text.encode()).hexdigest()


def table_seconds(bits: str) -> float:
    """Deterministic stand-in for measured seconds (used on both sides)."""
    h = int(hashlib.sha256(bits.encode()).hexdigest()[:8], 16)
    return 0.5 + (h % 100000) / 10000.0


def cnn_cost_model(net) -> dict:
    """Synthetic cost model for a CNN program so the sim evaluator (and
    hence the GA) can run over it."""
    loops = {}
    for lid in range(len(net.loop_trips)):
        loops[str(lid)] = {"cpu_us_per_iter": 0.001 * (1 + lid % 3), "gpu_speedup": 20.0 + lid % 7,
                           "kernel_launch_us": 5.0}
    vars_ = {a.name: {"size_bytes": a.nbytes} for a in net.arrays.values()}
    for scalar in ("b", "i", "j", "k", "c", "h", "w", "n", "m"):
        vars_[scalar] = {"size_bytes": 4}
    return {"loops": loops, "vars": vars_, "transfer_fixed_us": 10.0,
            "transfer_us_per_kib": 0.08}


def genomes_for(gm, tree, count: int, seed: int) -> list[str]:
    a = len(gm)
    rng = random.Random(seed)
    out = ["0" * a, "1" * a, "1" + "0" * (a - 1), "0" * (a - 1) + "1"]
    tries = 0
    while len(out) < count and tries < 50 * count:
        tries += 1
        bits = "".join("1" if rng.random() < rng.choice((0.2, 0.5, 0.8)) else "0" for _ in range(a))
        out.append(bits)
    seen, uniq = set(), []
    for b in out:
        if b not in seen:
            seen.add(b)
            uniq.append(b)
    return uniq


def plan_json(plan) -> dict:
    return {"directives": [[d.target_loop, d.clause, list(d.vars), d.origin_region]
                           for d in plan.directives], "notes": list(plan.notes)}


def result_json(res) -> dict:
    return {
        "best": [res.best.genome, res.best.seconds, res.best.fitness, res.best.status],
        "history": [[s.generation, s.best_seconds, s.best_fitness, s.mean_fitness,
                     s.evaluations_performed, s.cache_hits] for s in res.history],
        "gene_length": res.gene_length, "effective_population": res.effective_population,
        "evaluations": res.evaluations_performed, "cache_hits": res.cache_hits,
    }


def record_program(name: str, source: str, profile: dict | None, model: dict | None,
                   n_genomes: int, ga_seeds: tuple, ga_cfg: dict) -> dict:
    program = ref.parse(source)
    tree = ref.build_loop_tree(program)
    accesses = ref.extract_accesses(program)
    verdicts = ref.check_all_parallelizable(tree, accesses)
    entry = {
        "name": name, "source": source, "profile": profile, "model": model,
        "loops": [[n.loop_id, n.kind, n.parent, n.function, n.header_pos.line,
                   n.header_pos.col, n.canonical, n.counter] for n in tree.nodes],
        "accesses_digest": sha(json.dumps([[a.var, a.is_array, a.kind, a.pos.line, a.pos.col,
                                            a.pos.offset, list(a.loop_path), a.function,
                                            a.header_of,
                                            None if a.indices is None else [list(x) if x else None for x in a.indices]]
                                           for a in accesses])),
        "n_accesses": len(accesses),
        "verdicts": [[v.loop_id, v.eligible, v.reason] for v in verdicts],
    }
    try:
        gm = ref.build_genome_map(verdicts)
    except ref.EmptyGenome:
        entry["genome_map"] = None
        return entry
    entry["genome_map"] = list(gm.loop_ids)

    prof = None
    if profile is not None:
        with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as fh:
            json.dump(profile, fh)
        prof = ref.load_profile(fh.name, tree)
        g = ref.gate(tree, prof)
        entry["gate"] = [g.passed, g.max_total_iterations, g.threshold, g.loop_id]
    cm = None
    if model is not None:
        with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as fh:
            json.dump(model, fh)
        cm = ref.load_cost_model(fh.name)

    cases = []
    for bits in genomes_for(gm, tree, n_genomes, seed=len(source)):
        case = {"genome": bits, "valid": ref.check_genome_valid(bits, gm, tree)}
        if case["valid"]:
            plan = ref.plan_transfers(program, tree, accesses, bits, gm)
            case["plan"] = plan_json(plan)
            ann = ref.emit_annotated(program, tree, bits, gm, plan)
            case["emitted_sha256"] = sha(ann.text)
            case["inserted"] = [[i.line_no, i.content] for i in ann.inserted_lines]
            if prof is not None:
                counts = ref.directive_exec_counts(plan, tree, prof)
                case["exec_counts"] = [counts[d] for d in plan.directives]
                case["unhoisted_exec_total"] = sum(
                    ref.directive_exec_counts(ref.unhoisted(plan), tree, prof).values())
            if cm is not None and prof is not None:
                case["sim_seconds"] = ref.simulate_time(cm, bits, gm, tree, prof, plan).seconds
        cases.append(case)
    entry["cases"] = cases

    runs = []
    for seed in ga_seeds:
        cfg = ref.GAConfig(rng_seed=seed, **ga_cfg)
        calls = []

        def table_eval(bits, _calls=calls):
            _calls.append(bits)
            return ref.Measurement(table_seconds(bits), "measured")
        res = ref.run_ga(cfg, gm, tree, table_eval, ref.MeasurementCache())
        run = {"seed": seed, "evaluator": "table", "result": result_json(res), "calls": calls}
        runs.append(run)
        if cm is not None and prof is not None:
            ev = ref.make_sim_evaluator(cm, program, tree, accesses, gm, prof)
            res = ref.run_ga(cfg, gm, tree, ev, ref.MeasurementCache())
            runs.append({"seed": seed, "evaluator": "sim", "result": result_json(res)})
    entry["ga"] = {"config": ga_cfg, "runs": runs}
    return entry


def tune_report(name: str, source: str, profile: dict, model: dict, seed: int,
                extra: list[str]) -> dict:
    with tempfile.TemporaryDirectory() as tmp:
        t = Path(tmp)
        (t / "p.c").write_text(source)
        (t / "p_profile.json").write_text(json.dumps(profile))
        (t / "p_model.json").write_text(json.dumps(model))
        code = ref_cli.main(["tune", "--source", str(t / "p.c"), "--profile",
                             str(t / "p_profile.json"), "--evaluator", f"sim:{t}/p_model.json",
                             "--seed", str(seed), "--out", str(t / "best.c"), "--report",
                             str(t / "report.json"), *extra])
        report = (t / "report.json").read_text() if (t / "report.json").exists() else None
        best = (t / "best.c").read_text() if (t / "best.c").exists() else None
        # the paths inside the report differ per run; normalise them
        if report is not None:
            report = report.replace(str(t), "<tmp>")
    return {"name": name, "seed": seed, "extra": extra, "exit_code": code,
            "report": report, "best_sha256": None if best is None else sha(best)}


def main():
    programs = []
    reports = []
    for stem in ("copyinout", "hoist", "copymerge"):
        src = (REF_FIX / "golden" / f"{stem}.c").read_text()
        entry = record_program(stem, src, None, None, 4, (1,), {"population": 4, "generations": 3})
        entry["expected_emitted"] = (REF_FIX / "golden" / f"{stem}_expected.c").read_text()
        programs.append(entry)
    fixtures = [("tune", n) for n in ("siblings3", "nested3", "synergy5", "deep3", "mix10")]
    fixtures.append(("stress", "stress75"))
    for folder, stem in fixtures:
        base = REF_FIX / folder
        src = (base / f"{stem}.c").read_text()
        prof = json.loads((base / f"{stem}_profile.json").read_text())
        model = json.loads((base / f"{stem}_model.json").read_text())
        big = stem == "stress75"
        programs.append(record_program(stem, src, prof, model, 60 if big else 40,
                                       (1, 2) if big else (1, 2, 3),
                                       {"population": 30, "generations": 20}))
        reports.append(tune_report(stem, src, prof, model, 9, []))
        reports.append(tune_report(stem, src, prof, model, 3, ["--pop", "6", "--gens", "4"]))
    for net_name in ("demo", "micro", "yolov2-tiny"):
        net = build_net(net_name)
        model = cnn_cost_model(net)
        programs.append(record_program(net_name, net.source, net.profile_dict(), model,
                                       40, (1, 2), {"population": 30, "generations": 20}))
        reports.append(tune_report(net_name, net.source, net.profile_dict(), model, 5,
                                   ["--gate-threshold", "100000"]))
    (HERE / "reference_programs.json").write_text(json.dumps(programs, separators=(",", ":")) + "\n")
    (HERE / "reference_reports.json").write_text(json.dumps(reports, separators=(",", ":")) + "\n")
    print(f"wrote {len(programs)} programs, {len(reports)} reports")


if __name__ == "__main__":
    main()
