"""B200-native generation stage of surface-based fixation density maps
(arXiv 2601.07571), a drop-in for the reference package's Python API.

The compute runs in hand-written sm_100a CUDA kernels (csrc/) reached through
a C ABI (include/gazemap_b200.h) loaded with ctypes; there is no CPU fallback.
"""

from .density import (DEFAULT_EPS_ABS, DEFAULT_EPS_REL, DEFAULT_K, DEFAULT_RESOLUTION, DensityMap, GenerationConfig,
                      ScenePlan, Timings, accumulate_fixation, generate, normalize)
from .errors import (ConfigError, GazemapError, GazeOutsideFrustumError, InvalidFrustumError, LayoutMismatchError,
                     ParseError)
from .estimator import FixationDensityMapper
from .fixlog import FixationLog, parse_fixation_log, parse_fixation_table
from .io_export import EXPORT_HEADER, ExportRecord, load_map, save_map, write_export
from .gaze import (DEFAULT_THETA, SQRT_TWO_PI, CropFrustum, EllipseParams, Fixation, GazeCone, build_crop_frustum,
                   crop_bounds, crop_projection_matrix, ellipse_intersection, fixation_setup, fixation_table,
                   frustum_from_matrix, gaussian_weight, perspective_matrix)
from .raster import DepthBuffer, cull_triangles, depth_to_image, is_visible, rasterize_depth
from .render import ColorMap, camera_view_matrix, default_colormap, render_heatmap
from .geometry import (Mesh, SampledMesh, Scene, SceneObject, Transform, TriangleSampling, adaptive_resolution,
                       build_sampled_mesh, build_sampled_meshes, quat_to_matrix, rowcol_to_barycentric,
                       sample_count, sample_index_to_rowcol, sample_positions_local, sample_world_position,
                       triangle_area)

__version__ = "0.1.0"
