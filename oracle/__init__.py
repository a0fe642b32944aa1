"""CPU oracle for the DIP step — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline /
`--impl reference` legs may import this package, and only as the checker or
the timed CPU baseline. The product package (`paper_2507_14046_b200`) never
imports it; its hot path fails loudly without the sm_100a extension.

What it is: a restatement, in plain CPU PyTorch fp32 (the reference's own
arithmetic substrate, `pkg/pyproject.toml:13`), of the reference's DIP loop
`_FrameOptimizer.optimize` (`pkg/src/d2ip/pipeline.py:294-338`), its loss
(`pipeline.py:257-283`), drivers (`pipeline.py:394-560`), 4D-TV
(`pkg/src/d2ip/regularizers.py:86-140`) and `_kaiming_reset`
(`pkg/src/d2ip/priornet.py:267-282`), running the canonical config ResUNet of
SURVEY §7.1 built from `ChannelLayerNorm`/`ResConv3d`-shaped modules
(`priornet.py:96-148,183-232`), or the reference backbone FastResUNet3D
itself (`oracle/refnet.py`, `priornet.py:96-232`).

Parity pin: `tests/golden/make_golden.py` runs the REAL reference package
(imported from /root/reference in the build container, with the config net
injected exactly as SURVEY §8(c) verified) and commits the outputs under
`tests/golden/`; `tests/test_oracle_golden.py` checks this oracle against
them (`tests/golden/make_golden_refnet.py` does the same for FastResUNet3D,
unpatched). The reference is not present on the GPU box; the fixtures travel.
"""

from .refnet import OracleFastResUNet, build_oracle_refnet  # noqa: F401
from .resunet import ConfigResUNet, ChannelLayerNorm, kaiming_reset, build_oracle_net  # noqa: F401
from .frame import (  # noqa: F401
    OracleFrameOptimizer,
    oracle_loss_and_grads,
    oracle_reconstruct_sequence,
    oracle_tv4d,
)
