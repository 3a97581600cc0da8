"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This package holds NONE of the method's arithmetic: no ramp/IIR filtering, no
dyadic pattern, no Hough transform, no family combine.  It draws random ellipse
phantoms (numpy PCG64, seed = 1000*config + slice) and integrates
them ANALYTICALLY along straight lines in the paper's (s,t) line
parameterisation (§4.1; Fig.1b), i.e. what a scanner's
linogram would hold, then applies the noise model of the BASELINE config.
Random numbers the method itself would draw: none (the method is deterministic).
"""
from .generator import (  # noqa: F401
    CONFIGS, EllipseSet, draw_ellipses, linogram_of_ellipses, add_noise,
    make_slice, make_batch, random_linogram, integer_linogram, integer_image, random_image,
    sinogram_of_ellipses, image_of_ellipses,
)
