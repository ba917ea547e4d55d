"""B200-native CreateNewMapPoints + SearchAndFuse (arXiv 2511.02036 local-mapping hot path).

Drop-in for the reference ``localmap`` package's triangulation and fusion API, backed by
device-resident map state and hand-written sm_100a kernels behind a C ABI
(include/lm_b200.h, csrc/). See DESIGN.md.
"""

from .config import CullConfig, FuseConfig, GateConfig, MapConfig, MatchConfig, StoreConfig
from .errors import (DegenerateGeometryError, DeviceError, InvalidArgumentError, InvalidStateError,
                     LocalMapError, SlotConflictError, StoreCapacityError)
from .geometry import CameraIntrinsics, SE3Pose
from .mapmodel import UNBOUND, DeviceStore, KeyFrame, MapModel, MapPoint, MapSnapshot

__all__ = [
    "CullConfig", "FuseConfig", "GateConfig", "MapConfig", "MatchConfig", "StoreConfig",
    "DegenerateGeometryError", "DeviceError", "InvalidArgumentError", "InvalidStateError", "LocalMapError",
    "SlotConflictError", "StoreCapacityError", "CameraIntrinsics", "SE3Pose", "UNBOUND", "DeviceStore",
    "KeyFrame", "MapModel", "MapPoint", "MapSnapshot",
]
