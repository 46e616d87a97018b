"""splbm-b200: B200-native (sm_100a) T2C time-step path of the tiled sparse lattice Boltzmann
solver of arXiv 1703.08015, a drop-in for the reference `splbm` engine API.

Host API mirrors proj/include/splbm (geometry, tiling, fields, engine, overhead); the hot path is
the native library libsplbm_b200.so (CUDA kernels + C++ runtime behind include/splbm_b200.h).
"""
from .errors import (ConfigError, CudaError, DomainError, Error, IoError, NumericalError,
                     ParseError)
from .geometry import (BcParams, GenerateParams, Geometry, GeometryFormat, GeometryKind, NodeType,
                       Porosity, generate, is_solid, load_geometry_file, porosity,
                       save_geometry_file)
from .lattice import (Arrangement, CollisionKind, Compressibility, FluidModel, LatticeDescriptor,
                      lattice_descriptor, solver_lattice)
from .tiling import (Periodicity, TileGrid, TileStats, build_tile_grid, degenerate_bc_mask,
                     kEmptyTile, tile_stats)
from .fields import FieldData, linf_rel_diff
from .overhead import (CostParams, GeometryStats, NodeCosts, TileOverhead, bandwidth_utilization,
                       node_costs, overhead_t2c)
from .engine import (Method, SimConfig, SimulationResult, TileEngineT2C, make_engine,
                     run_simulation)

__all__ = [n for n in dir() if not n.startswith("_")]
