"""B200-native plan-search engine for HetRL's scheduler hot path.

Drop-in for the reference planner's evaluation + nested-SHA search path
(proj/src/search.cpp, proj/src/cost_model.cpp, proj/src/balance.cpp,
proj/src/plan.cpp). The compute runs in hand-written sm_100a CUDA kernels
behind a C ABI (include/hpg.h, libhpg.so); this package only binds it.
"""
from .hetplan import (  # noqa: F401
    CostModelConfig, Engine, HpgError, InfeasibleError, InputError, InternalError,
    SearchKnobs, SearchResult, Topology, UsageError, Workflow, build_workflow,
    load_library, load_topology, load_workflow, parse_topology, parse_workflow,
)
