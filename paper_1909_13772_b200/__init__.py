"""B200-native lattice Boltzmann stream-collide hot path (arXiv:1909.13772).

A drop-in for the reference's sweep API (blocksim: create_forest, PdfField,
ensure_flags, BoundaryHandling, fill_equilibrium, stream_collide,
exchange_ghosts, macroscopic_fields, gather_slice, mlups; forest snapshots
and VTK output) whose compute runs
in hand-written sm_100a kernels (csrc/, C-ABI include/lbm_b200.h) on
HBM-resident structure-of-arrays PDF fields, z-slab partitioned over GPUs.
The per-step halo of the crossing directions is fused into the boundary
planes' kernel, which stores them into the neighbour's ghost plane (peer
HBM over NVLink, CUDA IPC); NCCL send/recv of the contiguous runs is the
fallback transport (halo.py).
"""
from .errors import BackendError, BlocksimError, BufferUnderflowError, NumericsError, \
    SyncError, TopologyError, TypeTagError, UnrecoverableError, ValidationError
from .runtime import Context, ThreadContext, init_distributed, run
from .blockforest import BlockForest, BlockId, create_forest
from .field import Field, FieldDataHandler, FlagField, FlagFieldHandler, GhostPackInfo, \
    exchange_ghosts, gather_slice, sweep
from .lbm import *  # noqa: F401,F403
from . import lbm
from .vtk import write_block_vtk, write_vtk
from .wire import RecvBuffer, SendBuffer
from .bodies import BodyStorage, BodyStorageHandler, RigidBody, Sphere, add_sphere, find_body, \
    ghost_bodies, local_bodies, register_bodies, sync_bodies
from .checkpoint import BuddyCheckpoint
from .coupling import CoupledSystem, ParticleMapping, coupled_time_step, covered_cell_counts, \
    map_bodies, moving_boundary_sweep, reduce_hydrodynamic_forces, reinitialize_uncovered

__version__ = "0.1.0"
