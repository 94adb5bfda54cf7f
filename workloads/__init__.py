"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This package holds model DESCRIPTIONS only (species, rules, rate constants,
initial counts, compartment tree, sweep grids) and the seeded generators that
draw them.  It contains none of the method's arithmetic: no flattening, no
propensities, no RNG of the simulation, no statistics.  Both `oracle/` and
`paper_1010_2438_b200/` consume these descriptions independently.

Model description (a plain dict, see `models.py`):

    n_types, n_species           compartment types (0 = TOP) / species per compartment
    parent[C], type[C]           fixed compartment tree; parent[0] = -1, parent[c] < c
    rules[i] = {label, child_label, reactants, products, rate}
        reactants/products: list of (where, species, mult); where 0 = context
        compartment, 1 = the child compartment matched by the rule's pattern
    init[C * n_species]          initial counts (shared by all replicas)
    n_obs, obs_of_cell[C * n_species]   observable of each (compartment, species) cell or -1
    species_names                optional

A sweep is {"rules": [rule ids], "values": [[v, ...] per point]}.
"""
from .models import (  # noqa: F401
    CONFIGS,
    config,
    decay_model,
    dimerisation_model,
    immigration_death_model,
    isomerisation_model,
    lotka_volterra_chain,
    lotka_volterra_model,
    michaelis_menten_model,
    mm_sweep,
    paper_example_model,
    random_network_model,
    cwc_compartment_model,
    small_cwc_model,
)
