"""Write tests/golden/qkv1_small.bin with the UNMODIFIED reference's QKV1 writer
(qkv_io.py:25-35) so the package's reader/writer are pinned to its bytes.

    python tests/golden/make_qkv1.py      # in the build container (/root/reference present)

Inputs: VideoShape(2, 3, 4), d = 5, q/k/v ~ N(0, 1) from default_rng(7) in that order.
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from monarchbench.layout import VideoShape  # noqa: E402
from monarchbench.qkv_io import save_problem  # noqa: E402
from monarchbench.solver import AttentionProblem  # noqa: E402

rng = np.random.default_rng(7)
shape = VideoShape(2, 3, 4)
q, k, v = (rng.standard_normal((shape.n, 5)) for _ in range(3))
save_problem(AttentionProblem(q, k, v, shape), os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                             "qkv1_small.bin"))
