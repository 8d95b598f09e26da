"""B200-native certified quantized decode attention (arXiv 2605.20868).

Drop-in for the reference ``certkv`` hot path: cache append / quantize, the
certified attention call, the bound report and the fallback ladder, backed by
hand-written sm_100a CUDA kernels behind the C ABI in include/certkv_b200.h.
"""

__version__ = "0.1.0"

from . import _lib, kernels
from .cache import (DeviceKVCache, PageInReport, ScratchCache, StorageReport, TieredCache,
                    storage_report, storage_table)
from .engine import (CertifiedDecoder, HeadStepResult, PendingStep, StepOutput, dense_attention,
                     run_decode_step, rung3_per_head, rung4_all_heads, rung4_staging_bytes)
from .errors import EmptyCacheError, PagingError, Tier2UnavailableError
from .harness import (RunResult, Workload, WorkloadConfig, aggregate_telemetry, dump_line,
                      generate_workload, gqa_union, resolve_manifest, run_manifest, run_workload,
                      write_telemetry)
from .policy import Certificate, FallbackEvent, PolicyConfig, RungFlags, e_key_bound
