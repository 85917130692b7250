"""gbopt_b200: B200-native (sm_100a) FP64 gray-box neural-network oracle.

Drop-in for the reference gbopt NN oracle (proj/include/gbopt/nn.hpp) --
y = NN(x), J = dy/dx and H = sum_i lambda_i Hess NN_i(x) -- computed by
hand-written CUDA kernels behind the C ABI in include/gbopt_b200.h.
"""
from .gbopt import (  # noqa: F401
    ACTIVATIONS, LINEAR, TANH, SIGMOID, SOFTMAX, SOFTPLUS,
    INIT_UNIFORM_FANIN, INIT_XAVIER_UNIFORM, INIT_XAVIER_NORMAL, INIT_NORMAL_FANIN,
    GboptError, StructuralError, NumericError, SingularError, IoError, FormatError, DimensionError,
    TruncatedError, RangeError, ArgumentError, DeviceError,
    NeuralNet, Prng, load_weights, save_weights, random_net, random_net_ex, LdltFactorization, ldlt_factor,
    KktPattern, KktSystem, assemble_kkt, IpmOptions, CorrectedFactorization, inertia_correct,
    device_count, last_error, version, LIB_PATH,
)
