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


# parameter names of the reference functions (same source as REFERENCE_NAMES)
REFERENCE_SIGNATURES = {
    'candidate_benefit': ('window', 'period', 'residual', 'capacity', 'trace'),
    'candidate_window': ('period', 'trace', 'offload_channel', 'prefetch_channel', 'destination'),
    'channel_utilization': ('channel', 'window_start', 'window_end'),
    'characterize': ('trace', 'capacity', 'size_buckets', 'duration_buckets'),
    'compute_inactive_periods': ('trace',),
    'compute_memory_timeline': ('trace',),
    'gen_random_trace': ('seed', 'num_kernels', 'num_tensors', 'size_range', 'duration_range', 'global_fraction'),
    'gen_transformer_trace': ('cfg',),
    'load_trace': ('path',),
    'make_trace': ('kernels', 'tensors', 'meta'),
    'mark_urgent': ('plan', 'trace'),
    'parse_plan': ('data',),
    'parse_trace': ('data',),
    'per_kernel_active_bytes': ('trace',),
    'plan_migrations': ('trace', 'capacity', 'rates', 'host_cap'),
    'roofline_curve': ('trace', 'capacity', 'bandwidth_list'),
    'saturation_bandwidth': ('trace',),
    'save_trace': ('trace', 'path'),
    'select_destination': ('period', 'trace', 'ssd_channels', 'host_channels', 'host_cap', 'host_occupancy'),
    'simulate': ('trace', 'plan', 'capacity', 'rates'),
    'simulate_ideal': ('trace',),
    'simulate_layer_granularity': ('trace', 'capacity', 'rates', 'layer_map'),
    'simulate_on_demand': ('trace', 'capacity', 'rates'),
    'transfer_duration': ('channel', 'nbytes'),
    'transformer_peak_bytes': ('cfg',),
    'validate_trace': ('trace',),
    'write_plan': ('plan',),
    'write_trace': ('trace',),
}


def test_function_parameters_match_the_reference():
    import inspect
    bad = {n: tuple(inspect.signature(getattr(offloader, n)).parameters) for n, p in REFERENCE_SIGNATURES.items()
           if tuple(inspect.signature(getattr(offloader, n)).parameters) != p}
    assert bad == {}
