"""ctypes binding of the C ABI in include/dem_b200.h (the drop-in boundary).

The shared library is built in-tree (paper_1503_03553_b200/libdem_b200.so, see
__graft_entry__.build()). There is no fallback: if the library is missing the import fails.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdem_b200.so")

DEM_KERNEL_COUNT = 9
DEM_DEVICE_KERNEL_COUNT = 7

PHASE_INTEGRATE = 1
PHASE_GRAVITY = 2
PHASE_PP = 4
PHASE_RECT = 8
PHASE_LINE = 16
PHASE_STEP = 31

KERNEL_NAMES = ("Integrate", "CalcHash", "BitonicSort", "FindCellBoundsAndReorder",
                "ForceGravity", "InitializeContactIDs", "Collide", "CollideRectangle",
                "CollideLine")

D3 = C.c_double * 3


class dem_material(C.Structure):
    _fields_ = [("poisson_ratio", C.c_double), ("shear_modulus", C.c_double),
                ("youngs_modulus", C.c_double), ("restitution", C.c_double),
                ("sliding_friction", C.c_double)]


class dem_rect_wall(C.Structure):
    _fields_ = [("corner", D3), ("edge_u", D3), ("edge_v", D3), ("material_id", C.c_uint32)]


class dem_line_wall(C.Structure):
    _fields_ = [("a", D3), ("b", D3), ("material_id", C.c_uint32)]


class dem_config(C.Structure):
    _fields_ = [("dt", C.c_double), ("gravity", D3), ("domain_min", D3), ("domain_max", D3),
                ("material_count", C.c_uint32), ("materials", C.POINTER(dem_material)),
                ("pair_restitution", C.POINTER(C.c_double)),
                ("rect_wall_count", C.c_uint32), ("rect_walls", C.POINTER(dem_rect_wall)),
                ("line_wall_count", C.c_uint32), ("line_walls", C.POINTER(dem_line_wall)),
                ("grid_cell_size", C.c_double), ("contact_capacity", C.c_int32),
                ("collide_variant", C.c_int32), ("periodic", C.c_uint32), ("shear_rate", C.c_double),
                ("precision", C.c_int32)]


class dem_particles(C.Structure):
    _fields_ = [("count", C.c_uint64), ("ids", C.POINTER(C.c_uint32)),
                ("positions", C.POINTER(C.c_double)), ("velocities", C.POINTER(C.c_double)),
                ("angular_velocities", C.POINTER(C.c_double)), ("radii", C.POINTER(C.c_double)),
                ("masses", C.POINTER(C.c_double)), ("material_ids", C.POINTER(C.c_uint32))]


class dem_step_metrics(C.Structure):
    _fields_ = [("step", C.c_int64), ("contacts", C.c_int64), ("pp_contact_events", C.c_int64),
                ("max_contacts_per_particle", C.c_int32), ("reserved0", C.c_int32),
                ("clamps", C.c_int64), ("friction_max_ratio", C.c_double),
                ("capped_contacts", C.c_int64), ("cells", C.c_int64),
                ("device_kernel_ms", C.c_double * DEM_DEVICE_KERNEL_COUNT)]


class dem_grid(C.Structure):
    _fields_ = [("origin", D3), ("cell_size", C.c_double), ("nx", C.c_int32), ("ny", C.c_int32),
                ("nz", C.c_int32)]


class dem_error(C.Structure):
    _fields_ = [("code", C.c_int32), ("kernel", C.c_int32), ("particle_slot", C.c_uint32),
                ("particle_id", C.c_uint32), ("step", C.c_int64), ("message", C.c_char * 256)]


# Every symbol include/dem_b200.h and include/dem_b200_gen.h declare: (name, restype, argtypes)
_P = C.c_void_p
SIGNATURES = [
    ("dem_abi_version", C.c_int, []),
    ("dem_create", C.c_int, [C.POINTER(dem_config), C.POINTER(dem_particles), C.c_int, C.POINTER(_P)]),
    ("dem_clone", C.c_int, [_P, C.POINTER(_P)]),
    ("dem_destroy", None, [_P]),
    ("dem_step", C.c_int, [_P, C.c_int, C.POINTER(dem_step_metrics)]),
    ("dem_step_async", C.c_int, [_P, C.c_int]),
    ("dem_sync", C.c_int, [_P, C.POINTER(dem_step_metrics)]),
    ("dem_force_phase", C.c_int, [_P, C.c_uint32, C.POINTER(dem_step_metrics)]),
    ("dem_set_collide_variant", C.c_int, [_P, C.c_int]),
    ("dem_size", C.c_uint64, [_P]),
    ("dem_step_index", C.c_int64, [_P]),
    ("dem_get_particles", C.c_int, [_P, C.POINTER(dem_particles)]),
    ("dem_set_particles", C.c_int, [_P, C.POINTER(dem_particles)]),
    ("dem_get_forces", C.c_int, [_P, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    ("dem_set_forces", C.c_int, [_P, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    ("dem_get_grid", C.c_int, [_P, C.POINTER(dem_grid)]),
    ("dem_get_periodic_box", C.c_int, [_P, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    ("dem_get_order", C.c_int, [_P, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
    ("dem_get_contacts", C.c_int64, [_P, C.POINTER(C.c_uint32), C.POINTER(C.c_int32),
                                     C.POINTER(C.c_double), C.c_int64]),
    ("dem_get_traces", C.c_int64, [_P, C.POINTER(C.c_uint64), _P, C.c_int64]),
    ("dem_last_error", C.c_int, [_P, C.POINTER(dem_error)]),
    ("dem_time_steps", C.c_int, [_P, C.c_int, C.c_size_t, C.POINTER(C.c_float),
                                 C.POINTER(dem_step_metrics)]),
    ("dem_profile_step", C.c_int, [_P, C.c_size_t, C.POINTER(dem_step_metrics)]),
    ("dem_kernels_per_step", C.c_int, [_P]),
    ("dem_device_kernel_name", C.c_char_p, [C.c_int]),
    ("dem_device_bytes", C.c_uint64, [_P]),
    ("dem_gen_packing", C.c_int, [C.c_uint64, C.c_double, C.c_double, C.c_int, C.c_uint64,
                                  C.c_double, C.POINTER(dem_particles), C.POINTER(C.c_double)]),
    # slab decomposition
    ("dem_create_slab", C.c_int, [C.POINTER(dem_config), C.POINTER(dem_particles), C.c_int, C.c_int32,
                                  C.c_int32, C.c_uint64, C.POINTER(_P)]),
    ("dem_slab_record_bytes", C.c_int, [_P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    ("dem_slab_owned", C.c_uint64, [_P]),
    ("dem_slab_migrate", C.c_int, [_P, C.c_int, _P, _P, C.c_uint64, C.POINTER(C.c_uint64),
                                   C.POINTER(C.c_uint64)]),
    ("dem_slab_import", C.c_int, [_P, _P, C.c_uint64, _P, C.c_uint64]),
    ("dem_slab_halo", C.c_int, [_P, _P, _P, C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    ("dem_slab_ghosts", C.c_int, [_P, _P, C.c_uint64, _P, C.c_uint64]),
    ("dem_slab_force", C.c_int, [_P, C.c_uint32, C.POINTER(dem_step_metrics)]),
    ("dem_ipc_alloc", C.c_int, [C.c_int, C.c_uint64, C.POINTER(C.c_void_p)]),
    ("dem_ipc_free", C.c_int, [C.c_int, C.c_void_p]),
    ("dem_ipc_handle", C.c_int, [C.c_int, C.c_void_p, C.c_void_p]),
    ("dem_ipc_open", C.c_int, [C.c_int, C.c_void_p, C.POINTER(C.c_void_p)]),
    ("dem_ipc_close", C.c_int, [C.c_int, C.c_void_p]),
    # host-free sharded stepping
    ("dem_create_sharded", C.c_int, [C.POINTER(dem_config), C.POINTER(dem_particles), C.c_int, C.c_int, C.c_int,
                                     C.POINTER(_P)]),
    ("dem_shard_info", C.c_int, [_P, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_uint64)]),
    ("dem_shard_handle", C.c_int, [_P, C.c_void_p]),
    ("dem_shard_connect", C.c_int, [_P, C.c_void_p]),
    ("dem_shard_connect_local", C.c_int, [_P, _P, _P]),
    ("dem_shard_launch", C.c_int, [_P, C.c_int]),
    ("dem_shard_wait", C.c_int, [_P, C.POINTER(dem_step_metrics)]),
    ("dem_set_contacts", C.c_int, [_P, C.POINTER(C.c_uint32), C.POINTER(C.c_int32), C.POINTER(C.c_double), C.c_int64]),
    ("dem_selftest_division", C.c_int, [C.c_int, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64)]),
]


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build the CUDA library first (python -c 'import __graft_entry__ as g; g.build()')")
    lib = C.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        _lib = load()
    return _lib
