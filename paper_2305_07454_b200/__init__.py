"""B200-native (sm_100a) connected-vehicle ETL hot path of arXiv 2305.07454.

The product is the C-ABI library ``lib/libcvlg.so`` (CUDA kernels in ``csrc/``); this package
is the Python host mirror of the reference pipeline API on top of it (see cvlg.py).
"""
from .cvlg import (  # noqa: F401
    BatchFrame, Context, CvlError, FilterRules, GridSpec, Lattice, MultiGPU, PipelineStats,
    journey_features_device, journey_features_host, journey_ids, launch_count, pin_host, run_pipeline, run_pipeline_device,
    run_pipeline_host, run_pipeline_from_records, synth_day, unpin_host, write_container,
)
