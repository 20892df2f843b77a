"""B200-native hot path of the credo model-group pipeline (arXiv 2205.15757):
replica inference, per-request agreement and certificate digests behind a
C-ABI (include/credo_gpu.h). See DESIGN.md."""
from .credo import (AgreementOutcome, CHEBYSHEV, Context, CredoError,
                    CudaExecutor, DigestMismatch, EUCLIDEAN, GROUP_ACTIVE, GROUP_DEFINED,
                    GROUP_RETIRED, InferenceEngine, InvalidArgument, SUBMIT_INVALID,
                    SUBMIT_OK, SUBMIT_RETIRED, SUBMIT_UNKNOWN_GROUP,
                    MAX_MINUS_MIN, Model, ModelGroup, PerturbingExecutor,
                    RequestBatch, hash_ops_batches, host_sha256, lib)

__all__ = ["AgreementOutcome", "CHEBYSHEV", "Context", "CredoError",
           "CudaExecutor", "DigestMismatch", "EUCLIDEAN", "GROUP_ACTIVE", "GROUP_DEFINED",
           "GROUP_RETIRED", "InferenceEngine", "InvalidArgument", "SUBMIT_INVALID",
           "SUBMIT_OK", "SUBMIT_RETIRED", "SUBMIT_UNKNOWN_GROUP",
           "MAX_MINUS_MIN", "Model", "ModelGroup", "PerturbingExecutor",
           "RequestBatch", "hash_ops_batches", "host_sha256", "lib"]
