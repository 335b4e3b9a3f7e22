from oracle.step import *  # noqa: F401,F403
from oracle.step import SEQ_COMMIT, SNAPSHOT, apply_warm_gpu, apply_warm_oracle, oracle_step, warm_ops  # noqa: F401
