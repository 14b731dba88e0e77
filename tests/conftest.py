import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C-ABI)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_report_header(config):
    """Name the native library this session loads (CG_LIB selects e.g. the debug-bounds build), so a
    test log proves which build ran; nothing is loaded without a GPU."""
    lib = os.environ.get("CG_LIB") or os.path.join(ROOT, "paper_2601_17026_b200", "libcolgraph.so")
    try:
        import torch
        if not torch.cuda.is_available():
            return f"colgraph library: {lib} (not loaded: no CUDA device)"
        from paper_2601_17026_b200 import colgraph
        return f"colgraph library: {colgraph.LIB_PATH} -- {colgraph.version()}"
    except Exception as e:  # noqa: BLE001
        return f"colgraph library: {lib} (not loaded: {e})"


def pytest_sessionstart(session):
    # also written when -q hides the report header (the GPU logs are run with -q)
    if os.environ.get("CG_PRINT_LIB", "1") != "0":
        sys.stderr.write(pytest_report_header(session.config) + "\n")
