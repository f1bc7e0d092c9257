"""paper_2511_10676_b200 — B200-native pre-attention MoE expert predictor.

Drop-in for the hot path of the reference `moepredict` package
(arXiv 2511.10676): predictor forward / selection, evaluation reductions,
ranking-aware training and expert prefetch, running on hand-written sm_100a
kernels (libmoep_b200.so, C ABI in include/moep_b200.h). Public names follow
pkg/src/moepredict/__init__.py for the hot path.
"""

__version__ = "0.1.0"

from .exceptions import (  # noqa: F401
    BadMagicError, ConfigurationError, DataError, MoePredictError, RecordValidationError,
    TraceFormatError, TruncatedFileError, UsageError, VersionError,
)
from .core import ExpertSelection, layer_norm, rank_order, softmax, top_k, top_k_batch  # noqa: F401
from .engine import DevicePredictor, EvalCounters  # noqa: F401
from .predictor import (  # noqa: F401
    PredictorModel, backward, forward, init_model, load_model, n_params, predict_logits, predict_topk,
    predict_topk_batch, save_model,
)
from .losses import (  # noqa: F401
    BatchLabels, LossSpec, focal_loss, loss_and_grad, mse_loss, ranking_aware_loss, ranking_hinge,
    weighted_bce_loss,
)
from .metrics import (  # noqa: F401
    EvalResult, affinity_tier_profile, default_m_list, evaluate, evaluate_predictions, exact_match,
    overprovision_hit, top1_hit,
)
from .data import TraceFile, make_dataset  # noqa: F401
from .trainer import EpochStats, TrainConfig, TrainingReport, compare_losses, train  # noqa: F401
from .train_engine import DeviceTrainer  # noqa: F401


def __getattr__(name):
    # sklearn is imported lazily so the kernels do not pay for it
    if name == "ExpertPredictor":
        from .estimator import ExpertPredictor
        return ExpertPredictor
    raise AttributeError(name)
