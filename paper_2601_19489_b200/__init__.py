"""paper_2601_19489_b200: B200-native (sm_100a) differentiable tile rasterizer.

Drop-in for the hot path of the reference `tilesplat` package
(tilesplat/__init__.py:6-20): the same names, signatures and field layouts,
holding FP32 CUDA tensors, backed by hand-written CUDA kernels in
libtilesplat_b200.so (include/tilesplat_b200.h).  There is no CPU fallback.
"""

from .scene import TILE, Camera, GaussianSet, activate, inverse_sigmoid, sigmoid, validate
from .pose import PoseDelta, apply_delta
from .projection import (COV_DILATION, MIN_OPACITY, Grad3D, PoseGrad, SplatBatch, project,
                         project_vjp)
from .binning import (SnugBox, TileIndex, bin_aabb, bin_load_balanced, bin_sequential,
                      compute_snugboxes, lane_test_counts, snugbox)
from .forward import (ALPHA_CAP, CHECKPOINT_INTERVAL, MIN_ALPHA, T_TERMINATE, Contributions,
                      RenderBuffers, render)
from .backward import CheckpointsMissingError, Grad2D, backward_per_gaussian
from .losses import LossReport, depth_weight_schedule, disparity_loss, photometric, psnr
from .optim import Adam, position_lr
from .trainer import (TrainConfig, TrainingDiverged, TrainResult, TrainStep, ViewRender,
                      _full_grads, evaluate, init_gaussians, render_view, train,
                      view_loss_and_grads)
from .density import (DensifyDecision, ErrorMask, apply_decisions, error_mask, score_densify,
                      score_prune)
from .ingest import PlySchemaError, Scene, read_ply, write_ply
from .pose import bake, compose, identity_delta

__version__ = "0.1.0"
