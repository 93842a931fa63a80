"""B200-native Global Neighbor Sampling (arXiv 2106.06150) hot path.

Drop-in for the sampler / data-loader API of the reference package
``gnsbench`` (``/root/reference/pkg/src/gnsbench/__init__.py:5-22``): the cache
engine, the NS/GNS neighbour samplers, ``build_minibatch``, ``SamplerPool`` and
the GraphSAGE aggregation path, all running as hand-written sm_100a kernels in
``libgns.so`` behind the C ABI in ``include/gns.h``.
"""

from ._lib import GraphFormatError, InvariantError
from .cache import (CacheState, ProbVector, build_cache, degree_probs, inclusion_prob,
                    random_walk_probs, sample_cache)
from .formats import (build_csr, load_binary, load_edgelist, load_feature_csv, save_binary,
                      validate_graph)
from .graph import Graph, NodeSet, generate_powerlaw, generate_powerlaw_device
from .model import GraphSAGE, TrainConfig, init_params_numpy, micro_f1
from .pool import BatchItem, SamplerPool, epoch_targets
from .train import (AdamState, EpochStats, ModelParams, ParamGrads, TrainReport, adam_step, backward, evaluate,
                    forward, full_batch_forward, init_params, loss_and_grad, train)
from .sampling import (BatchRng, LayerBlock, MiniBatch, MiniBatchSampler, SamplerConfig,
                       build_minibatch, estimate_edge_inclusion, gns_weight_paper, isolated_fraction,
                       sample_neighbors_gns, sample_neighbors_uniform, validate_minibatch)

__version__ = "0.1.0"
