"""paper_2411_12780_b200 — B200-native PPLL (pipeline parallelism based on
local learning, arXiv 2411.12780).

A drop-in for the reference ``locopipe`` training loop (its public names are
re-exported here with the same signatures, ``locopipe/__init__.py:10-85``),
running each stage's local step as hand-written sm_100a kernels behind a
C-ABI library (``include/ppll.h``) and the PPLL dataflow as device rings on
CUDA streams.  The analysis/UI/data parts of the reference (cost model,
config, CLI, figures, toy data) are outside this build's scope.
"""
from .blocks import (
    AuxHead,
    Hyperparams,
    LinearLayer,
    LocalModule,
    MemoryProxy,
    NetworkSpec,
    PartitionPlan,
    aux_depth,
    aux_forward,
    block_forward,
    build_modules,
    local_loss_and_update,
    memory_footprint,
    partition,
)
from .errors import (
    BadMagic,
    EmptyTape,
    NotScalar,
    ConfigMismatch,
    CountMismatch,
    DimensionMismatch,
    EmptyEvents,
    EmptyProfiles,
    InvalidArg,
    InvalidMode,
    InvalidValue,
    IoError,
    LabelOutOfRange,
    LocopipeError,
    MissingGradient,
    NonFiniteError,
    PushAfterClose,
    StepOutOfRange,
    TooManyStages,
    TruncatedFile,
    WorkerPanic,
    ZeroDuration,
)
from .optim import LrSchedule, OptimizerState, cosine_lr, sgd_nesterov_step
from .runtime import (
    END_OF_STREAM,
    BufferSlot,
    DevicePipeline,
    EpochMetrics,
    RunConfig,
    RunMode,
    StageBuffer,
    run_deterministic,
    run_epoch,
    throughput,
)
from .tensor import (GradTape, Tensor, active_tape, add, backward, backward_from, bias_add,
                     matmul, relu, scale, softmax_xent, sum_all)
from .data import (BatchIterator, Dataset, DeviceDataset, IdxDataset, ImageDataset, batches,
                   gen_blobs, gen_spirals, load_cifar10, load_idx, load_stl10, load_svhn,
                   spiral_reference)
from .costs import (
    CommModel,
    CostEstimate,
    ScheduleEvent,
    ScheduleResult,
    StageProfile,
    calibrate,
    ppll_beats_pp,
    ratio_ideal,
    render_gantt_csv,
    simulate_schedule,
    steady_throughput,
    t_e2e,
    t_pp,
    t_ppll,
)
from .harness import (CSV_HEADER, ComparisonReport, ExperimentConfig, MetricsRecord, ModeSummary,
                      build_pipeline, device_memory, estimate_k, evaluate, make_datasets,
                      report_table, run_experiment, validate_config, write_metrics_csv)
from .vit import (VitLocalModule, VitSpec, balanced_depths, balanced_vit_depths,
                  build_vit_modules, vit_stage_costs)
from .resnet import ResLocalModule, ResNetSpec, build_resnet_modules, resnet_split

__version__ = "0.1.0"
