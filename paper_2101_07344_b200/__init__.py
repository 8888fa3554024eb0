"""latecache-b200: B200-native learned-cache (GATI, arXiv 2101.07344) serve path.

The hot path is hand-written sm_100a CUDA (tcgen05/TMEM/TMA contractions,
fused cache-lookup heads, warp-ballot compaction) behind the C-ABI in
include/latecache_b200.h; this package is its Python face.
"""
from ._lib import LIB_PATH, CudaError, InfeasiblePlanError, lib  # noqa: F401
from .api import (BaseModel, CacheVariant, Deployment, Request, RequestTrace, ServeResult,  # noqa: F401
                  SimSummary, build_variant, gen_workload, load_base_model, load_variant, make_base_model,
                  make_cnn_model, nearest_rank, plan_check, simulate_model, summarize, with_measured_lookup_ms,
                  load_base_model_binary, load_variant_binary, TrainConfig, train_predictor, train_selector,
                  AdaptationConfig, AdaptationResult, RetrainEvent, IntervalStat, run_adaptation)

__all__ = [
    "BaseModel", "CacheVariant", "Deployment", "Request", "RequestTrace", "ServeResult", "SimSummary",
    "build_variant", "gen_workload", "load_base_model", "load_variant", "make_base_model", "make_cnn_model",
    "nearest_rank", "plan_check", "simulate_model", "summarize", "with_measured_lookup_ms", "load_base_model_binary",
    "load_variant_binary", "CudaError", "TrainConfig", "train_predictor", "train_selector", "AdaptationConfig",
    "AdaptationResult", "RetrainEvent", "IntervalStat", "run_adaptation",
    "InfeasiblePlanError",
]
