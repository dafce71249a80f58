"""B200-native Star Attention two-phase hot path (drop-in for starsim's API).

Public names mirror the reference package surface (ss/__init__.py:3-64) for
the hot path: partition / AnchorSpec / augment / KVCache, run_phase1 /
run_phase2_step / start_session / decode / forward_star, causal_attention /
partial_attention / merge_partials.  Compute runs in libstar_attn.so
(sm_100a); there is no CPU fallback.
"""

from .attention import (AttnScale, PartialAttention, causal_attention, merge_partials,
                        partial_attention, streaming_causal_attention)
from .baselines import (DivergenceReport, FlopReport, divergence, global_pairs, ring_model,
                        star_model)
from .blocking import (CONTENT_MODES, POSITION_MODES, AnchorSpec, AugmentedBlock, BlockPlan,
                       KVCache, PagedKVPool, augment, encode_block, partition, sparsity_pattern)
from .errors import ConfigError, DeviceError, DomainError, ShapeError, StarSimError
from .model import (ModelConfig, ModelWeights, embed, forward_global, greedy_decode_global,
                    init_model, layer_step, logits_from)
from .numerics import (Prng, RopeConfig, default_dtype, precision, prng_fill, rope_apply,
                       set_default_dtype)
from .sim import (CommLedger, DecodeSession, Host, LedgerEntry, decode, forward_star,
                  run_phase1, run_phase2_step, set_query_host, start_session)

__version__ = "0.1.0"
