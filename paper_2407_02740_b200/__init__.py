"""B200-native Vecchia likelihood engine (arXiv 2407.02740) behind the reference
package's fitting API.  See DESIGN.md; the C ABI is include/vecchia_b200.h."""
from .errors import (DegenerateInformation, DeviceUnavailable, DimensionMismatch, EmptyData, LatitudeOutOfRange,
                     LengthMismatch, NonFiniteValue, NotPositiveDefinite, SingularDesign, UnknownFamily,
                     VecchiaError)
from .model import CovarianceParameters, Dataset, FitResult, ModelSpec, normalize_backend, validate_dataset
from .covariance import FAMILY_NAMES, covariance_registry, validate_parameters
from .preprocess import (NeighborArray, Ordering, embed_lonlat, find_ordered_neighbors, identity_ordering,
                         lonlat_to_xyz, maxmin_ordering, random_permutation, reorder_dataset, dependency_levels)
from . import engine, inference, io, predict, simulate
from .simulate import simulate_nn_gp
from .predict import PredictionSet, krige, rmse
from .engine import VecchiaParts, active_core_name, available_cores
from .inference import ProfiledEvaluation, assemble, default_start, evaluate, fisher_step, fit, to_log_scale

__version__ = "0.1.0"
