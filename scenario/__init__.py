"""Seeded synthetic input generators shared by tests, bench and smoke.

Holds none of the filter's arithmetic ("Input recipe")."""
from . import configs
from .configs import CONFIGS, ORDER, get, scaled, POSITION, RANGE_BEARING, COUNT_FIXED, COUNT_ADAPTIVE
from .generate import (simulate_truth, measurements, initial_population, initial_count, init_args,
                       random_particles, clustered_particles, random_measurements)
