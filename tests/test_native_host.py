"""Host-compiled checks of product device helpers that need no GPU."""
import os
import subprocess
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def test_rebuild_k_order_is_width_independent():
    """rebuild8<Q> maps the 32 elements of a plane word to the same byte slots for every Q and
    every byte is the element's offset digit — required for A and W of different widths to agree
    on the K order (a mismatch silently corrupts W_pA_q with p, q in different branches)."""
    src = os.path.join(ROOT, "tests", "native", "rebuild_check.cu")
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "rebuild_check")
        subprocess.check_call([NVCC, "-std=c++17", "-O1", "-o", exe, src])
        out = subprocess.run([exe], capture_output=True, text=True)
        assert out.returncode == 0 and out.stdout.startswith("OK"), out.stdout + out.stderr
