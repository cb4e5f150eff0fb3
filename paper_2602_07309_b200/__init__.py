"""B200-native prefill relevance ranker (drop-in for the semrank scorer path).

The product is the C-ABI shared library lib/libsemrank_b200.so (hand-written
sm_100a kernels + C++ host runtime); this package is its Python binding with
the reference's API names. See DESIGN.md.
"""
from .semrank import (  # noqa: F401
    Batch, BatchEntry, CacheKey, CalibrationBlock, CalibrationHead, ErrorCode, FlopReport, HeadSpec, ItemScores, ModelConfig, ModelWeights,
    MultiItemMask, Comm, Plan, BatchPlan, PROF_CLASSES, ScoreItem, ScoreMode, ScoreRequest, ScoreResult, ScoringEngine, Scheduler, SemrankError,
    build_multi_item_mask, flops, init_model, parse_score_request_json, tokenize, kRelevanceTask, load_weights, plan_batches, request_report,
    save_weights, score_by_mode, score_mode_from_name, score_mode_name, topk_host, ScoreCache,
    canonical_query, fnv1a64, query_signature, PromptParts, build_prompt, kPromptSuffix,
    score_result_to_json)
from .retrieval import (  # noqa: F401
    Corpus, DeviceCorpus, DocumentRecord, QuerySpec, RARWeights, RankedDoc, exhaustive_topk,
    filter_candidates)
from ._capi import LIB_PATH  # noqa: F401
