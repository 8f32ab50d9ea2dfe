"""B200-native batched SPHINCS+-{128f,192f,256f} signing (HERO-Sign capabilities).

Public API mirrors the reference package's sigcore (keygen / sign / verify,
byte-exact layouts) plus batch entry points; all hashing runs in the sm_100a
kernels of libherosign_b200.so through its C-ABI.
"""

from .engine import Engine, MultiEngine, PinnedBuffer, get_engine, get_multi_engine, shard_ranges
from .errors import (ConfigError, FormatError, GraphExecutionError, HeroSignError, TuningError,
                     UsageError)
from .params import PARAMETER_SETS, DerivedParams, ParameterSet, compressions_per_signature, derive
from .sigcore import (PublicKey, SecretKey, keygen, keygen_batch, message_to_indices, sign, sign_batch,
                      signature_regions, verify, verify_batch)

__all__ = [
    "Engine", "MultiEngine", "PinnedBuffer", "get_engine", "get_multi_engine", "shard_ranges", "ConfigError", "FormatError", "GraphExecutionError",
    "HeroSignError", "TuningError", "UsageError", "PARAMETER_SETS", "DerivedParams", "ParameterSet",
    "compressions_per_signature", "derive", "PublicKey", "SecretKey", "keygen", "keygen_batch",
    "message_to_indices", "sign", "sign_batch", "signature_regions", "verify", "verify_batch",
]
