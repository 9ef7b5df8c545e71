"""B200-native offload-pattern tuner (arXiv 1811.03882 hot path).

Drop-in for the reference package `acctuner` (its public API,
`pkg/src/acctuner/__init__.py:10-85`, is re-exported here under the same
names), plus the B200 execution path:

* `nets`          -- Darknet-style CNN programs written in the C subset
                     (demo, yolov2-tiny 416, yolov2 608) with their op manifest
                     and analytic loop profiles;
* `kernels`       -- ctypes binding of `libacct_sm100.so`, the C-ABI over the
                     hand-written sm_100a kernels (include/acct.h);
* `executor`      -- runs a genome's offload pattern: selected loops as
                     kernels, the rest as native host loops, transfers exactly
                     where the plan's directives sit, counted;
* `gpu_evaluator` -- the `gpu:<config.json>` evaluator the GA consumes,
                     spread over a pool of GPUs.

The reference's module paths are aliased too (`.transfer`, `.ga`,
`.evaluation`, ...), so `from <pkg>.transfer import plan_transfers` works
as it does with `acctuner`.
"""

import sys as _sys

from . import annotate, errors, legality, loopnest, measure, planner, search, syntax, tuner
from .annotate import (
    AnnotatedSource, InsertedLine, emit_annotated, kernels_only_annotation, strip_annotations,
)
from .errors import (
    AutotunerError, DeviceError, DomainError, EmptyGenome, ExternalOracleError, InvalidGenome,
    ModelError, ParityError, ParseError, PlanMismatch, ProfileError, SpawnError,
)
from .legality import (
    DEFAULT_GATE_THRESHOLD, ExternalOracle, GateDecision, GenomeMap, ParallelizabilityVerdict,
    Profile, ProfileEntry, build_genome_map, check_all_parallelizable, check_parallelizable,
    gate, load_profile,
)
from .loopnest import LoopNode, LoopTree, VarAccess, build_loop_tree, extract_accesses
from .measure import (
    CommandEvaluatorConfig, CostModel, LoopCost, Measurement, MeasurementCache,
    cached_evaluate, command_evaluate, load_command_config, load_cost_model, simulate_time,
)
from .planner import (
    DataDirective, TransferPlan, TransferPlanner, check_genome_valid, directive_exec_counts,
    plan_to_dict, plan_transfers, selected_loops, unhoisted,
)
from .search import (
    EvaluatedIndividual, GAConfig, GenerationStats, SearchResult, fitness_from_time,
    init_population, mutate, one_point_crossover, run_ga, select_next_parents,
)
from .syntax import parse
from .tuner import (
    EXIT_EVALUATOR_FAILURE, EXIT_GATE_REJECT, EXIT_NO_OFFLOADABLE_LOOPS, EXIT_OK,
    EXIT_PARSE_ERROR, EXIT_PROFILE_ERROR, PipelineConfig, build_evaluator,
    make_cmd_evaluator, make_sim_evaluator, run_pipeline,
)

# reference module names -> modules of this package
for _ref_name, _mod in (("nodes", syntax), ("parser", syntax), ("loops", loopnest),
                        ("analysis", legality), ("transfer", planner),
                        ("evaluation", measure), ("ga", search), ("emitter", annotate),
                        ("pipeline", tuner)):
    _sys.modules.setdefault(f"{__name__}.{_ref_name}", _mod)
    globals().setdefault(_ref_name, _mod)

__version__ = "0.1.0"
