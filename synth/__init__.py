"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This package holds NO arithmetic of the paper's method: it only draws binary
voxel images (stand-ins for the paper's PD4/GLD4/Granular images, PAPER.md
§6, Table 1) and seeded test vectors.  Both sides
(``oracle/`` and ``paper_2510_22077_b200``) consume these inputs; neither
imports the other.
"""
from .geometry import make_image, load_config, config_path, CONFIG_NAMES  # noqa: F401
from .vectors import seeded_normal  # noqa: F401
