"""B200-native bidomain PCG hot path (arxiv 1711.08708, block-LU / monodomain).

Drop-in for the reference package's solver surface (`bidomain.system`,
`bidomain.precond`, `bidomain.krylov`, `bidomain.simulate.time_step`): the
same names and arguments, with the arithmetic in a hand-written sm_100a
library (`libbidomain_b200.so`, C ABI in include/bidomain_b200.h).
Assembly, meshes and conductivity tensors are host-side setup.
"""
from .conductivity import (ConductivityParams, TensorField, default_params, ReferenceFibers,
                           UniformFibers, CircumferentialFibers, TransmuralRotation,
                           EllipsoidHelical)
from .errors import (AssemblyError, BidomainError, ConfigError, NonConvergenceError,
                     NumericalBreakdownError, NumericalDegeneracyError, OracleError,
                     PreconditionerError)
from .ionic import (IonicParams, StimulusBox, StimulusProtocol, StimulusSite, default_protocol,
                    ionic_current, stimulus, stimulus_vector, update_gate)
from .mesh import (Mesh, Region, RestrictionMap, build_box_mesh, build_cube_mesh,
                   build_ellipse_torso_2d, build_ellipsoid_torso_3d, build_heart_torso_2d,
                   build_rect_mesh, build_square_mesh, restrict, transpose_restrict)
from .system import BidomainSystem, BlockVector, gamma
from .precond import (INNER_NAMES, BlockLUPreconditioner, ExactFactorization,
                      IncompleteCholesky0, Jacobi, build_monodomain_matrix, make_inner,
                      regularize_stiffness)
from .krylov import SolveStats, dump_residuals, pcg_solve
from .simulate import (ActivationMap, SimState, SimulationResult, SimulationSetup,
                       activation_times, run_simulation, time_step)

from .vtkio import read_mesh_vtk, write_activation_csv, write_fields_vtk, write_mesh_vtk
from . import study, vtkio  # bd/bench.py study harness, bd/vtkio.py formats
from .study import (BenchConfig, BenchRecord, ScalingStudy, calibrate_costs,  # noqa: E402
                    growth_rate, least_squares_slope, run_scaling_study, save_study)

__version__ = "0.1.0"
