"""Data-transfer planning (paper section 3.2) with precomputed indexes.

Semantics are the reference planner's, output for output
(`pkg/src/acctuner/transfer.py:34-189`):

For each selected region G (ascending) and each variable v accessed inside
G, minus the counters written by loop headers of G's own subtree:

* need_in  = v is read inside G and some CPU-side access of v (same
  function) is a set or a define;
* need_out = v is written inside G and the CPU side accesses v at all;
* a CPU-side access is one whose loop chain contains no selected loop;
* each needed directive hoists from G up the ancestor chain and stops
  below the first ancestor whose subtree holds a blocking CPU-side access
  (copyin: set/define; copyout: ref/set/define);
* in+out merge into one `copy` at the deeper of the two targets (ties go to
  the copyin target);
* directives are grouped per (origin, clause, target), variables sorted,
  then stably sorted by (target, clause, first variable).

What differs is cost.  The reference re-filters the whole access list for
every region and every variable (about 11 ms per genome on the 75-gene
stress fixture, 92% of a GA search).  Here the per-loop / per-variable
access lists are built once per program and each genome only flips a
CPU-side mask over the accesses inside its selected loops.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import InvalidGenome
from .legality import GenomeMap, Profile
from .loopnest import DEFINE, REF, SET, LoopTree

COPY = "copy"
COPYIN = "copyin"
COPYOUT = "copyout"
CLAUSE_ORDER = (COPY, COPYIN, COPYOUT)

_IN_BLOCKERS = frozenset((SET, DEFINE))
_OUT_BLOCKERS = frozenset((REF, SET, DEFINE))


@dataclass(frozen=True)
class DataDirective:
    target_loop: int        # the directive line precedes this loop
    clause: str             # copy | copyin | copyout
    vars: tuple             # sorted, no duplicates
    origin_region: int      # the selected loop that needed it


@dataclass(frozen=True)
class TransferPlan:
    directives: tuple
    notes: tuple


def selected_loops(genome_bits: str, genome_map: GenomeMap) -> set:
    if len(genome_bits) != len(genome_map):
        raise InvalidGenome(
            f"genome length {len(genome_bits)} != gene length {len(genome_map)}")
    if not set(genome_bits) <= {"0", "1"}:
        raise InvalidGenome(f"genome {genome_bits!r} must be a 0/1 string")
    ids = genome_map.loop_ids
    return {ids[k] for k, bit in enumerate(genome_bits) if bit == "1"}


def _has_nested_pair(chosen: set, tree: LoopTree) -> bool:
    return any(not chosen.isdisjoint(tree.ancestors(lid)) for lid in chosen)


def check_genome_valid(genome_bits: str, genome_map: GenomeMap, tree: LoopTree) -> bool:
    """Valid iff no selected loop encloses another selected loop."""
    return not _has_nested_pair(selected_loops(genome_bits, genome_map), tree)


class TransferPlanner:
    """Per-program access index; `plan(bits, genome_map)` is the planner."""

    def __init__(self, tree: LoopTree, accesses: list):
        self.tree = tree
        self.accesses = accesses
        self.size = len(accesses)
        self.kind = [a.kind for a in accesses]
        self.var = [a.var for a in accesses]
        self.ancestors = [tree.ancestors(n.loop_id) for n in tree.nodes]
        self.subtree = [frozenset(tree.subtree(n.loop_id)) for n in tree.nodes]
        self.depth = [len(a) for a in self.ancestors]
        # accesses inside each loop, bucketed by variable
        self.inside: list[dict[str, list[int]]] = [{} for _ in tree.nodes]
        # every access of (function, var)
        self.of_var: dict[tuple[str, str], list[int]] = {}
        for i, acc in enumerate(accesses):
            self.of_var.setdefault((acc.function, acc.var), []).append(i)
            for lid in acc.loop_path:
                self.inside[lid].setdefault(acc.var, []).append(i)
        # header-written counters of each loop's subtree
        self.counters: list[frozenset] = []
        for n in tree.nodes:
            sub = self.subtree[n.loop_id]
            names = {v for v, idxs in self.inside[n.loop_id].items()
                     if any(self.kind[i] == SET and accesses[i].header_of in sub for i in idxs)}
            self.counters.append(frozenset(names))

    def _hoist(self, region: int, var: str, cpu: list, blockers: frozenset) -> int:
        target = region
        for anc in self.ancestors[region]:
            for i in self.inside[anc].get(var, ()):
                if cpu[i] and self.kind[i] in blockers:
                    return target
            target = anc
        return target

    def plan(self, genome_bits: str, genome_map: GenomeMap) -> TransferPlan:
        chosen = selected_loops(genome_bits, genome_map)
        if _has_nested_pair(chosen, self.tree):
            raise InvalidGenome(
                f"nested selected loops: {sorted(chosen)} contains an ancestor pair")

        cpu = [True] * self.size
        for lid in chosen:
            for idxs in self.inside[lid].values():
                for i in idxs:
                    cpu[i] = False

        groups: dict[tuple[int, str, int], set] = {}
        notes: list[str] = []
        kind = self.kind
        for region in sorted(chosen):
            fn = self.tree.nodes[region].function
            here = self.inside[region]
            for var in sorted(set(here) - self.counters[region]):
                mine = here[var]
                reads = any(kind[i] == REF for i in mine)
                writes = any(kind[i] == SET for i in mine)
                host = [i for i in self.of_var.get((fn, var), ()) if cpu[i]]
                need_in = reads and any(kind[i] in _IN_BLOCKERS for i in host)
                need_out = writes and bool(host)
                if need_in and need_out:
                    t_in = self._hoist(region, var, cpu, _IN_BLOCKERS)
                    t_out = self._hoist(region, var, cpu, _OUT_BLOCKERS)
                    deeper = t_out if self.depth[t_out] > self.depth[t_in] else t_in
                    groups.setdefault((region, COPY, deeper), set()).add(var)
                    notes.append(f"{var}@region{region}: copyin+copyout merged to "
                                 f"copy at loop {deeper}")
                elif need_in:
                    t_in = self._hoist(region, var, cpu, _IN_BLOCKERS)
                    groups.setdefault((region, COPYIN, t_in), set()).add(var)
                    notes.append(f"{var}@region{region}: cpu-written, gpu-read -> "
                                 f"copyin at loop {t_in}")
                elif need_out:
                    t_out = self._hoist(region, var, cpu, _OUT_BLOCKERS)
                    groups.setdefault((region, COPYOUT, t_out), set()).add(var)
                    notes.append(f"{var}@region{region}: gpu-written, cpu-visible -> "
                                 f"copyout at loop {t_out}")

        found = [DataDirective(target, clause, tuple(sorted(names)), origin)
                 for (origin, clause, target), names in groups.items()]
        found.sort(key=lambda d: (d.target_loop, d.clause, d.vars[0]))
        return TransferPlan(tuple(found), tuple(notes))


_PLANNERS: dict[int, TransferPlanner] = {}


def planner_for(tree: LoopTree, accesses: list) -> TransferPlanner:
    """Planner cached per (tree, accesses) object pair."""
    hit = _PLANNERS.get(id(accesses))
    if hit is not None and hit.tree is tree and hit.accesses is accesses \
            and hit.size == len(accesses):
        return hit
    fresh = TransferPlanner(tree, accesses)
    if len(_PLANNERS) > 64:
        _PLANNERS.clear()
    _PLANNERS[id(accesses)] = fresh
    return fresh


def plan_transfers(program, tree: LoopTree, accesses: list, genome_bits: str,
                   genome_map: GenomeMap) -> TransferPlan:
    """Directive plan for a valid genome (reference `transfer.py:82-158`)."""
    return planner_for(tree, accesses).plan(genome_bits, genome_map)


def directive_exec_counts(plan: TransferPlan, tree: LoopTree, profile: Profile) -> dict:
    """Executions per directive: one per arrival at its target loop
    (reference `transfer.py:161-165`) -- the transfer-count contract the
    GPU executor's counters reproduce."""
    return {d: profile.entry_count(d.target_loop) for d in plan.directives}


def unhoisted(plan: TransferPlan) -> TransferPlan:
    """The same directives pinned to their origin regions."""
    return TransferPlan(tuple(DataDirective(d.origin_region, d.clause, d.vars, d.origin_region)
                              for d in plan.directives), plan.notes)


def plan_to_dict(plan: TransferPlan) -> dict:
    return {"directives": [{"target_loop": d.target_loop, "clause": d.clause,
                            "vars": list(d.vars), "origin_region": d.origin_region}
                           for d in plan.directives]}
