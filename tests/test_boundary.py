"""C-ABI boundary on CPU: the library loads, exports every symbol include/paragan.h
declares, validates configs, and its parameter layout agrees with the oracle's
independently written one (no GPU needed: these calls do not touch CUDA)."""
import os
import re

import pytest

from oracle import biggan as bg
from paper_2411_03999_b200 import api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    with open(os.path.join(ROOT, "include", "paragan.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"\b(paragan_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = api.lib()
    names = _declared()
    assert "paragan_d_step" in names and "paragan_layout_pack" in names
    for n in names:
        assert hasattr(L, n), n
    assert set(names) <= set(api.SYMBOLS), set(names) - set(api.SYMBOLS)


@pytest.mark.parametrize("res,ch,attn", [(128, 96, 64), (32, 8, 16), (16, 8, 8), (256, 96, 64), (512, 96, 64),
                                         (64, 16, 32)])
def test_param_layout_matches_oracle(res, ch, attn):
    ocfg = bg.Config(resolution=res, ch=ch, attn_res=attn)
    cfg = api.make_config(resolution=res, ch=ch, attn_res=attn, local_batch=2)
    for net, specs in ((api.NET_G, bg.g_param_specs(ocfg)), (api.NET_D, bg.d_param_specs(ocfg))):
        ns, nt = api.param_count(cfg, net)
        assert nt == bg.n_trainable(specs)
        assert ns == bg.n_state(specs)


@pytest.mark.parametrize("ch", [32, 4])
def test_sndcgan_param_layout_matches_oracle(ch):
    """Config 1 (R25): the library's SN-DCGAN state layout is the oracle's (written independently)."""
    ocfg = bg.Config(arch="sndcgan", resolution=32, ch=ch)
    cfg = api.make_sndcgan_config(ch=ch)
    for net, specs in ((api.NET_G, bg.g_param_specs(ocfg)), (api.NET_D, bg.d_param_specs(ocfg))):
        ns, nt = api.param_count(cfg, net)
        assert nt == bg.n_trainable(specs)
        assert ns == bg.n_state(specs)
    # bf16 and other resolutions are rejected for this architecture
    for kw in (dict(compute=api.BF16), dict(resolution=64)):
        bad = api.make_sndcgan_config(ch=ch)
        for k, v in kw.items():
            setattr(bad, k, v)
        with pytest.raises(api.ParaganError):
            api.workspace_size(bad)


def test_biggan128_total_is_paper_count():
    cfg = api.make_config()
    tot = api.param_count(cfg, api.NET_G)[1] + api.param_count(cfg, api.NET_D)[1]
    assert tot == 158_416_358   # "158.42M"


def test_config_validation():
    bad = [dict(resolution=100), dict(ch=3), dict(local_batch=0), dict(d_steps_per_g=0), dict(c_pad_image=4),
           dict(rank=2, world_size=2), dict(attn_res=48)]
    for kw in bad:
        cfg = api.make_config(**kw)
        with pytest.raises(api.ParaganError) as e:
            api.workspace_size(cfg)
        assert e.value.status == 2, kw
    cfg = api.make_config()
    cfg.abi_version = 99
    with pytest.raises(api.ParaganError):
        api.workspace_size(cfg)


def test_workspace_fits_b200_at_paper_config():
    n = api.workspace_size(api.make_config(local_batch=256))
    assert 1e9 < n < 170e9


def test_product_path_has_no_fallback():
    """The product package never reaches the oracle, and a missing library is an error, not a fallback."""
    import ast
    import subprocess
    import sys
    pkg = os.path.join(ROOT, "paper_2411_03999_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            tree = ast.parse(open(os.path.join(pkg, fn)).read())
            for node in ast.walk(tree):
                if isinstance(node, ast.Import):
                    assert not any(a.name.split(".")[0] == "oracle" for a in node.names), fn
                if isinstance(node, ast.ImportFrom):
                    assert (node.module or "").split(".")[0] != "oracle", fn
    code = ("import os, paper_2411_03999_b200.api as a\n"
            "try:\n    a.lib()\nexcept OSError as e:\n    print('LOUD', e)\nelse:\n    print('LOADED')\n")
    env = dict(os.environ, PARAGAN_LIB="/nonexistent/libparagan.so")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert "LOUD" in r.stdout, r.stdout + r.stderr
