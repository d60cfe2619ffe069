"""Seeded synthetic CFG generators shared by the oracle tests, the GPU tests and bench.py.

This package holds NO arithmetic of the method (no path enumeration, no SCC
logic, no maximality test): it only draws graphs.  Every generator returns a
successor CSR ``(offsets int64[n+1], targets int32[m])`` with each row sorted
ascending and free of duplicate arcs, plus metadata (entry/exit vertex).
"""
from .generators import (  # noqa: F401
    Graph,
    fig1b,
    structured_cfg,
    config2,
    dense_scc,
    config3,
    loop_chain,
    config4,
    parallel_sccs,
    config5,
    random_digraph,
    disjoint_union,
    k_nested_if,
    k_seq_if,
    single_loop,
    k_seq_loops,
    random_dag_cfg,
    CONFIGS,
    make_config,
)
