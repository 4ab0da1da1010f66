"""paper_2206_01298_b200 -- B200-native discrete-adjoint ODE-block gradients.

Drop-in for the gradient path of the reference ``odegrad`` package (PNODE,
arXiv 2206.01298): same names and argument meanings for the ODE-block API
(RHS field, time span, scheme, checkpoint policy, gradient call), batched over
samples and executed by hand-written sm_100a kernels behind a C ABI
(include/odeblock.h, libodeblock.so).  There is no CPU fallback.
"""

from .configs import ConfigInputs, make_config
from .controls import (AdaptiveController, ConvergenceError, DeviceError, FixedController, FixedGridController,
                       GradientExplosionError, IntegrationError, NfeCounters, SolverConfig,
                       StiffnessError, StoreCounters)
from .engine import (AdjointState, ForwardSolution, GradResult, adjoint_terminal, backward_sweep,
                     continuous_adjoint_solve, forward_pass, grad, loss_value)
from .autograd import ODEBlock
from .fields import (ACTIVATION_IDS, CnfField, ConvField, Field, MlpField, MlpModel, MlpSpec, StiffMlpField, init_model,
                     mlp_spec)
from .losses import LossSpec, terminal_loss
from .policies import CheckpointPolicy, ScheduleAction, revolve_count, revolve_schedule
from .schemes import SCHEME_NAMES, ButcherTableau, Scheme, tableau_catalog
from .formats import load_model, model_from_json, model_to_json, read_dataset_csv, save_model, write_dataset_csv
from .training import (AdamWConfig, Dataset, OptimizerState, TrainConfig, TrainingRecord, adamw_step,
                       geometric_grid, minmax_normalize, train)

__version__ = "0.1.0"

__all__ = [
    "ACTIVATION_IDS", "AdaptiveController", "ButcherTableau", "CnfField", "CheckpointPolicy", "ConvField", "ConfigInputs", "ConvergenceError",
    "DeviceError", "Field", "FixedController", "FixedGridController", "GradResult",
    "GradientExplosionError", "IntegrationError", "LossSpec", "MlpField", "MlpModel", "MlpSpec",
    "NfeCounters", "SCHEME_NAMES", "ScheduleAction", "Scheme", "SolverConfig", "StiffMlpField",
    "StiffnessError", "StoreCounters", "grad", "init_model", "make_config", "mlp_spec",
    "revolve_count", "revolve_schedule", "tableau_catalog", "terminal_loss",
    "AdamWConfig", "Dataset", "OptimizerState", "TrainConfig", "TrainingRecord", "adamw_step",
    "geometric_grid", "minmax_normalize", "train", "load_model", "model_from_json", "model_to_json",
    "read_dataset_csv", "save_model", "write_dataset_csv", "continuous_adjoint_solve",
    "AdjointState", "ForwardSolution", "adjoint_terminal", "backward_sweep", "forward_pass", "loss_value",
    "ODEBlock",
]
