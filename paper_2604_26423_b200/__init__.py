"""B200-native LR-QAOA state-vector simulator (drop-in for lrqbench's hot path).

The public names mirror lrqbench/__init__.py for the noiseless path
(instance -> circuit -> run_circuit -> exact_expected_r / sample -> ratios).
Compute runs in liblrq.so (hand-written sm_100a CUDA, C ABI in include/lrq.h);
importing the package does not need a GPU, calling the engine does.
"""

__version__ = "0.1.0"

from .circuit import (
    CircuitIR,
    GateOp,
    LayerArrays,
    LrQaoaParams,
    Schedule,
    build_circuit,
    build_schedule,
    circuit_to_text,
    gate_counts,
    hqc_cost,
    lower_circuit,
)
from .engine import (
    CutDistribution,
    Precision,
    draw_indices,
    drain_state_pool,
    exact_cut_distribution,
    apply_gate,
    apply_h,
    apply_rx,
    apply_rzz,
    init_plus_state,
    load_statevector,
    zero_state,
    ShotSet,
    StateVector,
    check_memory,
    exact_expected_r,
    expected_r_from_probs,
    run_circuit,
    sample,
    save_statevector,
    state_bytes,
    uniform_amplitude,
)
from .errors import AbortedRunError, CapacityError, FitError, StateError, ValidationError
from .problem import (
    OptimalCut,
    WmcInstance,
    approximation_ratio,
    as_index,
    bitstring_to_index,
    complete_edge_list,
    cut_value,
    cut_values,
    cut_values_range,
    generate_instance,
    index_to_bitstring,
    load_instance,
    optimal_cut_bruteforce,
    random_baseline_expectation,
    save_instance,
    shot_ratios,
    solve_instance,
)
from .rng import derive_rng, derive_seed
from .sharded import (
    ExchangeStep,
    GateTiming,
    ShardedStateVector,
    ShardPlan,
    SweepConfig,
    TimingRecord,
    exchange_steps,
    exchange_volume,
    plan_for_shard_count,
    plan_shards,
    remap_volume,
    run_circuit_sharded,
    scaling_sweep,
    write_timing_csv,
)
from .noise import (
    DepolarizingConfig,
    NoiseFit,
    epsilon_accumulated,
    fit_k0,
    noisy_expected_probs,
    noisy_expected_r,
    predict_r_overlap,
    r_overlap,
    run_noisy_ensemble,
)
