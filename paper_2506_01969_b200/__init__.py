# SPDX-License-Identifier: Apache-2.0
"""B200-native (sm_100a) ETAP MLA decode — the hot path of arxiv 2506.01969 behind the
reference's run_etap boundary (include/etap_mla.h)."""
from ._lib import EtapError, EtapShapeError, FLAG_EAGER_RESCALE, FLAG_NEGATE_RESCALE  # noqa: F401

__all__ = ["EtapError", "EtapShapeError", "FLAG_EAGER_RESCALE", "FLAG_NEGATE_RESCALE"]
