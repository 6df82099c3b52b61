"""Seeded synthetic input generators (no method arithmetic). See workloads.py."""
from .workloads import (CONFIGS, LayerConfig, bf16_bits_to_f32, local_experts, make_dy,  # noqa: F401
                        make_expert, make_experts, make_routing, make_x, popularity_rank,
                        to_bf16_bits)
