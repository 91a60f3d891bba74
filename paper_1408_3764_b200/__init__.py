"""paper_1408_3764_b200 — B200-native grand-canonical Monte Carlo per-move
energy path (arXiv 1408.3764), behind the reference's config / strategy /
simulation API. The compute lives in libgcmc_b200.so (hand-written sm_100a
CUDA, C ABI in include/gcmc_b200.h); this package is the host mirror.
"""
from .config import RunConfig, format_g17, parse_config_file, parse_config_text  # noqa: F401

__all__ = ["RunConfig", "parse_config_text", "parse_config_file", "format_g17", "engine",
           "checkpoint"]


def __getattr__(name):
    # The engine needs the CUDA library; import it lazily so config parsing
    # works on CPU-only hosts, and fail loudly (ImportError) when it is absent.
    if name in ("engine", "checkpoint"):
        import importlib

        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
