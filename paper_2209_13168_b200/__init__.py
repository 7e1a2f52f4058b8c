"""B200-native bound evaluation for event-based divergence (arXiv 2209.13168).

Drop-in replacement for the hot path of the reference package ``eventdiv``
(``pkg/src/eventdiv/__init__.py:3-44``): the same public names for the motion
model, the contrast objective and its interval bound, and the branch-and-bound
solver, computed by hand-written sm_100a CUDA (libevd.so, include/evd.h).
"""

from .contrast import (ContrastBound, EventImage, accumulate_image, bound_terms,
                       image_contrast, image_contrast_expanded, rasterize_segment,
                       upper_bound_image)
from .events import (BIN_MAGIC, EventBatch, EventFormatError, EventStream, EventValidationError,
                     SensorGeometry, batch_stream, parse_event_bin, pixel_counts,
                     remove_hot_pixels, rescale_events, write_event_bin)
from .geometry import (CheiralityError, DivergenceSample, VelocityInterval,
                       continuous_divergence, divergence_from_velocity, radial_warp,
                       velocity_domain, warp_batch, warp_scale)
from .solver import (BnbResult, IterationLimitError, NoEventsError, SolverParams,
                     contrast_at, estimate_stream_divergence, grid_search_oracle,
                     maximise_contrast_bnb, stream_divergence, stream_divergence_bin)
from ._lib import EvdError, EvdUnavailable, set_device

__version__ = "0.1.0"
