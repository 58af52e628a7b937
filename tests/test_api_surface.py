"""The package exports every public name of the reference `offloader`
package (its __init__, pkg/src/offloader/__init__.py:4-65: the drop-in
surface of SURVEY §8b), so `import paper_2506_06472_b200 as offloader` works
for a reference user.  The name list was read from the reference once and is
kept here (the reference does not travel to the GPU box)."""

import paper_2506_06472_b200 as offloader

REFERENCE_NAMES = (
    'BandwidthChannel', 'Benefit', 'CandidateWindow', 'ChannelConfigError', 'ChannelRates',
    'CharacterizationReport', 'ConfigurationError', 'InactivePeriod', 'KernelRecord', 'MemoryTimeline',
    'MigrationPlan', 'PlanEntry', 'Reservation', 'RooflinePoint', 'SimReport', 'SimulationError', 'TensorKind',
    'TensorRecord', 'Trace', 'TraceParseError', 'TraceValidationError', 'TransformerGenConfig',
    'UnsatisfiableTraceError', 'ValidationReport', 'analysis', 'bandwidth', 'candidate_benefit',
    'candidate_window', 'channel_utilization', 'characterize', 'compute_inactive_periods',
    'compute_memory_timeline', 'gen_random_trace', 'gen_transformer_trace', 'load_trace', 'make_trace',
    'mark_urgent', 'parse_plan', 'parse_trace', 'per_kernel_active_bytes', 'plan_migrations', 'planner',
    'roofline', 'roofline_curve', 'saturation_bandwidth', 'save_trace', 'select_destination', 'simulate',
    'simulate_ideal', 'simulate_layer_granularity', 'simulate_on_demand', 'simulator', 'trace', 'tracegen',
    'transfer_duration', 'transformer_peak_bytes', 'validate_trace', 'write_plan', 'write_trace',
)


def test_every_reference_name_is_exported():
    missing = [n for n in REFERENCE_NAMES if not hasattr(offloader, n)]
    assert missing == []
