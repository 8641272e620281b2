"""B200-native vMAP object-mapping step (drop-in for the reference `vobj` hot path).

Host API mirrors /root/reference/pkg/src/vobj (models, render, trainer,
objects); the compute runs in libvmap_b200.so (hand-written sm_100a CUDA).
"""

from .geometry import AABB, look_at
from .models import (ActivationCache, FieldOutput, Gradients, ModelArch, OptimState, StackedModelParams,
                     adam_step, append_model, backward, forward, init_stacked, positional_encode, set_frozen)
from .objects import AssociationConfig, Keyframe, ObjectInstance, ObjectMap, add_keyframe
from .render import (CameraIntrinsics, LossWeights, RenderResult, SamplingConfig, compute_losses,
                     loss_output_grads, render_backward, render_rays)
from .trainer import (BenchRow, RaySampleBatch, StepReport, TrainConfig, benchmark, train_on_batch,
                      train_on_batch_sequential)

__version__ = "0.1.0"
