"""B200-native per-frame bisector update (arXiv 2407.02215), drop-in for the
reference ``cbtmesh`` package's CBT / tessellation-update API."""

__version__ = "0.1.0"
