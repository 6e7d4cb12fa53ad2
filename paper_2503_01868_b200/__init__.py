"""B200-native StripedHyena 2 convolution operators (arXiv 2503.01868), drop-in for the
reference `convhybrid` operator API (Hyena-SE / MR / LI forward, multi-hybrid layouts,
context-parallel conv schemes). Compute runs in hand-written sm_100a kernels behind the
C-ABI of include/hyena_b200.h; there is no CPU fallback.
"""

from . import cp, fft
from . import cp as cpsim  # the reference's module name; schemes take this rank's shard + a CPGroup
from .cp import (
    CPGroup,
    LayoutCP,
    ShardedSeq,
    a2a_conv,
    a2a_conv_backward,
    a2a_conv_pipelined,
    a2a_conv_saved,
    gather,
    layout_forward_cp,
    p2p_conv,
    p2p_conv_overlapped,
    p2p_fft_causal_wrapper,
    p2p_fft_conv,
    p2p_fft_forward,
    p2p_fft_inverse,
    shard,
)
from .fft import bit_reversal, circular_conv_oracle, dft_oracle, dif_split, dit_merge, idft_oracle
from .backward import (
    DeviceGrads,
    HyenaGrads,
    filter_param_grads,
    grad_for_path,
    hyena_backward,
    iter_params,
    layout_backward,
    operator_backward,
)
from .blockconv import (
    MultiplyCounter,
    ToeplitzFactors,
    TwoStageGrads,
    TwoStageIneligibleError,
    assemble_toeplitz,
    block_conv,
    build_factors,
    chunk_parallel_forward,
    spill_count,
    two_stage_backward,
    two_stage_flops,
    two_stage_forward,
    two_stage_forward_saved,
)
from .core import (
    ExplicitFilter,
    GroupSpec,
    ImplicitFilter,
    RegularizedFilter,
    SeqTensor,
    causal_conv_input_grad,
    causal_conv_taps_grad,
    direct_causal_conv,
    filter_length,
    full_toeplitz,
    materialize_filter,
    uniform_groups,
)
from .fft import fft_conv, next_pow2
from .hyena import (
    HyenaConfig,
    HyenaOperator,
    LayoutSpec,
    OperatorStack,
    build_layout,
    hyena_forward,
    hyena_forward_saved,
    identity_config,
    layout_forward,
    layout_forward_device,
    layout_forward_saved,
    make_hyena_config,
    make_inner_bank,
    make_layout,
    update_param,
)
from .rand import make_rng

__version__ = "0.1.0"
