"""B200-native Barnes-Hut t-SNE hot path (Acc-t-SNE, arXiv 2212.11506).

A drop-in for the reference package ``bhtsne``'s optimisation path: the same
stage functions, config, run() and an estimator, executed by hand-written
sm_100a CUDA kernels in ``libbhtsne_b200.so`` behind a C ABI
(include/bhtsne_b200.h).  There is no CPU fallback: every compute call
raises when the library or a CUDA device is missing.  Importing the package
itself needs neither (so host logic and the ABI can be inspected on CPU).
"""

__version__ = "0.1.0"

from .affinity import (NeighborGraph, PerplexityResult, SparseAffinity,
                       calibrate_perplexity, from_csr, set_exaggeration,
                       symmetrize)
from .estimator import BarnesHutTSNE
from .io import InputMatrix, load_labels, load_matrix, save_matrix
from .forces import (GradientBuffers, attractive, repulsive_bh,
                     repulsive_counts, repulsive_exact)
from .knn import knn_exact
from .optimizer import (STAGES, Embedding, Engine, StepTimings, TsneConfig,
                        embedding_from, gradient_step, init_embedding,
                        kl_divergence, run)
from .quadtree import (MortonCodes, MortonQuadtree, build_tree,
                       compute_bounds, morton_codes, morton_interleave,
                       summarize)

__all__ = [
    "__version__", "InputMatrix", "load_matrix", "save_matrix",
    "load_labels", "NeighborGraph", "PerplexityResult", "SparseAffinity",
    "calibrate_perplexity", "symmetrize", "set_exaggeration", "from_csr",
    "MortonCodes", "MortonQuadtree", "compute_bounds", "morton_codes",
    "morton_interleave", "build_tree", "summarize", "GradientBuffers",
    "attractive", "repulsive_bh", "repulsive_exact", "repulsive_counts",
    "Embedding", "TsneConfig", "StepTimings", "init_embedding",
    "embedding_from", "gradient_step", "kl_divergence", "run", "Engine",
    "BarnesHutTSNE", "STAGES", "knn_exact",
]
