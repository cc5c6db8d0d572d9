"""B200-native DET (density-equalizing transformation) engine with the cartomorph API.

Drop-in for the hot path of the reference package ``cartomorph``
(arxiv 2604.13880, "Fast Time-Varying Contiguous Cartograms Using Integral
Images"): the iteration loop rasterise -> integral images -> displacement ->
advect -> pixel-count error runs as hand-written sm_100a CUDA kernels behind a
C-ABI (``include/det_api.h``) bound with ctypes.  There is no CPU fallback:
importing works without a GPU, but every compute entry point needs the built
library and a CUDA device.
"""

from .engine import (BatchEngine, CartogramEngine, CartogramState, IterationRecord, RunResult, StoppingCriteria,
                     cartographic_error_arrays, run, target_weights)
from .errors import CartomorphError, IngestionError, NumericError, RasterizationError, RegionCollapsedError
from .geomodel import MapModel, Region, densify, ring_centroid, detect_adjacencies, shoelace_area, to_geojson, with_adjacency
from .integral import IntegralImageSet, integral_images, straight_inims, tilted_inims
from .displacement import (AnchorSet, DisplacementField, advect, anchors, base_mapping, mapping_grid,
                           mapping_point, residual_field)
from .raster import BACKGROUND, DensityTexture, LabelTexture, build_density, default_bdv, rasterize_labels
from .metrics import (QualityReport, cartographic_errors, full_report, hamming_distance, relative_position_error,
                      shape_distortion, topology_distortion)
from .sweep import sweep_bdv
from .temporal import (AreaFractionPolicy, Frame, FrameSequence, TimeSeriesDataset, background_mass_schedule,
                       interpolate_frames, interpolate_vertices, run_cumulative, run_direct)

__version__ = "0.1.0"
