"""CPU oracle for the certified quantized decode-attention path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2605_20868_b200`` imports this
package; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may use it, and only as the
checker (or as the timed CPU baseline), never as the thing measured.

What it is: a float64 NumPy restatement of the reference ``certkv`` package's
hot path (quantize-on-append, Phase-1 scoring, adaptive top-K with Rung 1/2,
LRU page-in accounting, Phase-2 mask-gated attend, the two-term certificate,
the ranking / boundary / canary monitors and the Rung 3/4 dense fallback).
Every function cites the reference ``file:line`` it restates
(paths relative to ``/root/reference/pkg/src/certkv``).

Pinning: ``tests/golden/make_golden.py`` imports the real reference from
``/root/reference`` (in the build container only) and freezes its outputs
into ``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks this
restatement against those fixtures (codes/metadata bit-exact, scores and
outputs to 1e-12, decisions identical).  Parity is therefore *pinned*.

``narrow=True`` applies the device storage widths the reference only charges
in accounting (cache.py:11-13, quantizer.py:13-18): FP32 key scale/offset and
FP16 value scale/offset are used for every reconstruction, and the value
annotations eta are measured on that narrowed reconstruction.  The CUDA path
is checked against ``narrow=True``; ``narrow=False`` is the reference itself.
"""

from .quant import (fit_key_block, fit_value_block, dequant_keys,
                    dequant_values, value_annotations, pairwise_sum128)
from .kv import OracleKV, OracleScratch, Tier2Lost, PagingFault
from .step import (OraclePolicy, phase1, select_blocks, phase2, dense_output,
                   decode_step, run_workload, make_workload, block_logmass,
                   fused_attend_f32, e_key_bound, storage_table)
