"""Force-rebuild libgsp.so (A/B experiments pass -D knobs through GSP_NVCC_EXTRA)."""
import importlib.util
import os
spec = importlib.util.spec_from_file_location(
    "_gsp_build", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2402_03548_b200", "_build.py"))
b = importlib.util.module_from_spec(spec)
spec.loader.exec_module(b)
b.build(force=True)
