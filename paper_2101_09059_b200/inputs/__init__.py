"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle's tests.

Holds no arithmetic of the method (mesh geometry, random fields and load vectors are
inputs to ens_create / ens_set_traction); see DESIGN.md "Inputs".
"""
from . import configs, fields, loads, mesh  # noqa: F401
