"""B200-native DG right-hand-side path behind the array-context API of arxiv/paper_2512_17101.

Public surface:

* ``B200ArrayContext`` / ``DeviceArray``  -- drop-in for ``laze.ArrayContext`` (actx.py)
* ``DOFArray``, ``DGDiscretization``      -- element-major nodal data + per-mesh operators
* ``EulerOperator``, ``NavierStokesOperator``, ``rk4_step`` -- the operator program (operators.py)
* ``dg.mesh.box_mesh``                    -- conforming simplicial box meshes
* ``MultispeciesOperator``, ``Mixture``     -- multi-species reactive NS (configs[4]), generic device ops (multispecies.py)
* ``DeviceRK4``                           -- device-resident RK4 driver, one CUDA graph per step (timestepper.py)
"""
from .dofarray import DOFArray
from .discretization import BC_FARFIELD, BC_NONE, BC_WALL, DGDiscretization
from .operators import EulerOperator, NavierStokesOperator, rk4_step, rk4_step_fused
from .dg.mesh import box_mesh
from .multispecies import Mixture, MultispeciesOperator
from . import errors


def __getattr__(name):
    # the array context needs torch + the CUDA library; import lazily so that host-only code
    # (mesh generation, the operator program on a CPU context) does not pay for it
    if name in ("B200ArrayContext", "DeviceArray", "CompiledFunction"):
        from . import actx
        return getattr(actx, name)
    if name == "DeviceRK4":
        from .timestepper import DeviceRK4
        return DeviceRK4
    raise AttributeError(name)
