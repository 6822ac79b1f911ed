"""B200-native engine for the nested-Monte-Carlo Bermudan pricers of arXiv 0805.1827.

Drop-in for the reference package ``bermuda``'s pricer entry points
(``price``, ``build_iz_boundary``, ``build_cmc_rule``, ``fit_ensemble``,
``regress_boundary``) and config objects, computed by hand-written sm_100a
kernels in ``lib/libbermuda_b200.so`` (C ABI: include/bermuda_b200.h).
There is no CPU fallback: importing the package loads the library.
"""

from . import _native  # noqa: F401  (fails loudly without the CUDA library)
from .boosting import Stump, StumpEnsemble, TrainingSet, fit_ensemble, fit_stump, score
from .boundary_cmc import CmcBuildConfig, CmcBuildReport, CmcRule, build_cmc_rule, classifier_features
from .boundary_iz import (BoundaryPointJob, IzBoundary, IzBuildReport, PointResult, build_iz_boundary,
                          continuation_value, regress_boundary, solve_boundary_point)
from .engine import Engine, TaskPlan, TimingLog, partition
from .lowdisc import SeedGrid, default_box, generate_glp, uniform_log_grid
from .market import BermudanSpec, ConfigError, MarketParams, PayoffKind
from .pricer import (PATH_BLOCK, CmcScoreRule, EuropeanRule, ImmediateAtDate, IzRule, PriceEstimate, pool_moments,
                     price)

__version__ = "0.1.0"
