"""B200-native (sm_100a) attention templates — a drop-in for the attnforge / AttentionEngine hot path.

Construction API (same names as the reference's ``attnforge/__init__.py``)::

    from paper_2502_15349_b200 import builtin, with_causal_mask, run_tiled_parallel
    spec = with_causal_mask(builtin("softmax", batch=8, heads=32, heads_kv=8, seq=8192))
    o = run_tiled_parallel(spec, {"q": q, "k": k, "v": v})      # CUDA tensors in, CUDA out

Compute runs only in the sm_100a library ``_lib/libattn_b200.so`` (C ABI: ``include/attn_b200.h``).
"""

from .errors import (ForgeError, InputError, ParseError, LowerError, ShapeError, GraphError,
                     SchemaError, UnknownVariantError, SemanticError, UnsupportedError, NanError,
                     NoFeasiblePlanError, DeviceError)
from .spec import (AttentionSpec, Dims, ExtraInput, ModificationFn, DirectRowNorm, OnlineRowNorm,
                   Pattern, mod, online, builtin, causal_mask, with_causal_mask, diagonal_scale,
                   retention_gammas, spec_from_dict, spec_from_text, load_variant, spec_to_dict,
                   from_reference, BUILTIN_NAMES, BUILTIN_DIMS)
from .plan import plan_parallel, plan_linear, ParallelPlan, LinearPlan
from .api import (parallel_forward, parallel_backward, run_tiled_parallel, run_naive_parallel,
                  linear_forward, linear_backward, linear_step, run_chunk_recurrent, run_step_recurrent,
                  autodiff_grads, bind, AttentionEngine, mla_decode, use_deterministic_backward,
                  deterministic_backward)
from . import api, generic, hookvm, schedule
from .emit import code_generation
from .schedule import make_scheduling_task, measure_factory, tile_config_scheduling

__all__ = [n for n in dir() if not n.startswith("_")]
