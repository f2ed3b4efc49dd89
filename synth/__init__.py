"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This package holds input generation only (scene and camera sampling, array
hashing). It contains none of the method's arithmetic (no projection, no
contraction, no visibility, no assignment): see DESIGN.md "Input recipe".
"""
from .scenes import CONFIGS, SceneConfig, Scene, make_scene, make_config, array_hashes  # noqa: F401
