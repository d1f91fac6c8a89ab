"""B200-native GTree (arXiv 2305.00645) MPC decision-tree hot path.

Three-party replicated-secret-share training and inference with the
reference package's entry points (``run_local``, ``train_tree``,
``infer_batch``, ``TrainConfig``) on top of hand-written sm_100a kernels
(``libgtree_b200.so``, C ABI in include/gtree_b200.h).
"""

from .engine import LocalRun, PartyEngine, TransportError, infer_batch, open_results, run_local, train_tree
from .ledger import Ledger, Metrics, Transcript, infer_metrics, train_metrics
from .seeds import SeedSetup, derive_seed, filler_values, make_keys
from .shares import RING8, RING32, RING64, AVec, BitVec, Ring, RingError, ShareError
from .train import DeviceTrainer, TrainConfig, TrainResult, counter_shift, levels_of, resolved_depth, train_3pc, train_components
from .infer import infer_3pc, infer_components, infer_device

__all__ = [
    "AVec", "BitVec", "DeviceTrainer", "Ledger", "LocalRun", "Metrics", "PartyEngine", "RING8", "RING32", "RING64",
    "Ring", "RingError", "SeedSetup", "ShareError", "TrainConfig", "TrainResult", "Transcript", "TransportError",
    "counter_shift", "derive_seed", "filler_values", "infer_3pc", "infer_batch", "infer_components", "infer_device",
    "infer_metrics", "levels_of", "make_keys", "open_results", "resolved_depth", "run_local", "train_3pc",
    "train_components", "train_metrics", "train_tree",
]
