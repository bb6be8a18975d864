"""B200-native SPH hot path of arXiv 2103.07925 (fluid / rigid body / contact / heat / phase transitions).

Public API: `Simulation` (device context over the C ABI in include/sphg.h),
`ParticleStore` (host mirror of sphfsi::ParticleStore<3>), `scenarios`
(seeded BASELINE configs).  The CUDA library is loaded lazily by Simulation.
"""
from . import abi, scenarios
from .store import ParticleStore, BODY_DTYPE, empty_bodies
from .sim import Simulation, SPHError

__all__ = ["abi", "scenarios", "ParticleStore", "BODY_DTYPE", "empty_bodies", "Simulation", "SPHError"]
