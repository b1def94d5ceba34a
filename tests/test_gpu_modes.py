"""Alternate kernel paths behind environment switches (read once per process, so each runs the
end-to-end parity subset in a subprocess): forced balanced attention on short contexts, one-Q-tile
passes, half-height replicated query tiles, the QKV GEMM with fp32 output + the separate RoPE kernel
(the fused RoPE epilogue is the default), the gate/up GEMM's last wave in K-parts with a last-arriver fixup.  Each must
stay parity-green against the oracle exactly like the default path (tests/test_gpu_verify.py)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env", [{"SPECEDGE_ATTN_BALANCED": "1"}, {"SPECEDGE_ATTN_NQ": "1"},
                                 {"SPECEDGE_ATTN_HALF_TILES": "1"}, {"SPECEDGE_QKV_FUSED": "0"},
                                 {"SPECEDGE_TAIL_SPLIT": "3"}],
                         ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_alternate_path_parity(env):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_verify.py", "-x", "-q", "-p", "no:cacheprovider",
                        "-k", "greedy_matches or long_ragged or sampled_matches or full_width"],
                       cwd=ROOT, env=e, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
