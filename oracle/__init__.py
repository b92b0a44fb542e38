"""CPU oracle for the Optimus 2D hot path — TEST INFRASTRUCTURE ONLY.

A float64 numpy restatement of the reference algorithm
(/root/reference/pkg/src/summagrid: dense.py, layers.py, model.py, oracle.py,
summa.py, mesh.py). Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it,
and only as the checker or the timed CPU baseline — never as part of the
product path, which has no CPU fallback.

Parity is pinned: ``oracle/gen_golden.py`` imports the real reference package
in the build container and writes golden vectors to ``tests/golden/``;
``tests/test_oracle_golden.py`` checks this restatement against them.
"""

from .bookkeeping import (  # noqa: F401
    act_block,
    bunched_tile,
    deinterleave_qkv,
    interleave_qkv,
    mesh_groups,
    node_map,
    token_block,
    v_padded,
    weight_block_owner,
)
from .model_ref import (  # noqa: F401
    RefConfig,
    init_params,
    sample_data,
    serial_backward,
    serial_forward,
)
