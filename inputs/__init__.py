"""Seeded synthetic inputs (networks, configs, dump-id choices); no method arithmetic."""
from .networks import (GATE_POSITIVE, GATE_ZERO, Config, Network, Reaction, config, configs, dimerization, dump_ids,  # noqa: F401
                       empty_network, hiv, hiv_delta_t_sweep, immigration_death, pure_death, rate_matrix,
                       synthetic, with_rates)
