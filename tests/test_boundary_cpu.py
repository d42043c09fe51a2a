"""The C-ABI boundary on CPU (no GPU calls): the library loads, exports every
symbol include/rbm.h declares, its config struct layout matches ctypes, and
eager validation returns the documented statuses (rbm_workspace_size runs the
same validation as rbm_init without touching the device)."""
import ctypes
import os
import re
import subprocess

import pytest

import rbm_inputs as RI

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "rbm.h")


@pytest.fixture(scope="module")
def R():
    from paper_1812_10575_b200 import build, rbm
    build.build()
    rbm.lib()
    return rbm


def declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rbm_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(R):
    names = declared()
    assert "rbm_init" in names and "rbm_step" in names and "rbm_run" in names and "rbm_gather" in names
    out = subprocess.run(["nm", "-D", "--defined-only", R.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (rbm_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    assert set(R.EXPORTS) == set(names)
    for n in names:
        assert hasattr(R.lib(), n)


def test_library_is_sm100a(R):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", R.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_config_layout_matches_header(tmp_path):
    from paper_1812_10575_b200 import rbm
    fields = [f for f, _ in rbm.RbmConfig._fields_]
    prog = tmp_path / "l.c"
    body = "".join(f'printf("{f} %zu\\n", offsetof(rbm_config, {f}));' for f in fields)
    prog.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "rbm.h"\nint main(void){'
                    + body + 'printf("sizeof %zu\\n", sizeof(rbm_config)); return 0;}\n')
    exe = tmp_path / "l"
    subprocess.check_call(["gcc", "-std=c11", f"-I{os.path.join(ROOT, 'include')}", str(prog), "-o", str(exe)])
    got = dict(l.split() for l in subprocess.check_output([str(exe)], text=True).splitlines())
    for f in fields:
        assert int(got[f]) == getattr(rbm.RbmConfig, f).offset, f
    assert int(got["sizeof"]) == ctypes.sizeof(rbm.RbmConfig)


def status_of(R, cfg):
    c = R.make_config(cfg)
    n = ctypes.c_size_t(0)
    return R.lib().rbm_workspace_size(ctypes.byref(c), ctypes.byref(n)), n.value


@pytest.mark.parametrize("bad,status", [
    (dict(p=1), 1), (dict(p=600), 1), (dict(d=4), 1), (dict(d=2), 1),  # dyson needs d=1
    (dict(sigma=-1.0), 1), (dict(dt=0.0), 1), (dict(kernel=99), 2), (dict(world_size=2), 1),
    (dict(world_size=3, n=100000), 1), (dict(world_size=2, rank=2, n=100000), 1),
    (dict(world_size=2, n=100000, scheme="rbmr"), 0), (dict(world_size=2, n=100000, scheme="rbmr_seq"), 3),
    (dict(world_size=2, n=100000, p=2), 0),
    (dict(integrator="split", p=4), 1), (dict(n=501, integrator="split"), 1),
    (dict(n=1), 1), (dict(replica=1 << 24), 1), (dict(p=65, n=100000), 1),
])
def test_validation_statuses(R, bad, status):
    cfg = RI.c1_dyson()
    cfg.update(bad)
    st, _ = status_of(R, cfg)
    assert st == status
    assert R.lib().rbm_last_error(None)


def test_valid_configs_and_workspace(R):
    for name, f in RI.ALL.items():
        st, nbytes = status_of(R, f())
        assert st == 0, (name, R.lib().rbm_last_error(None))
        assert nbytes > 0 and nbytes % 256 == 0
    # the workspace holds two SoA state buffers at least
    st, nbytes = status_of(R, RI.c4_aggregation())
    assert nbytes >= 2 * 10**8 * 12


def test_step_without_gpu_is_loud(R):
    """No silent CPU path: without a device rbm_init fails with RBM_ERR_CUDA / WORKSPACE."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    c = R.make_config(RI.c1_dyson())
    out = ctypes.c_void_p()
    st = R.lib().rbm_init(ctypes.byref(c), None, 0, None, None, ctypes.byref(out))
    assert st != 0 and not out.value


def test_part_info_layout_matches_header(tmp_path):
    from paper_1812_10575_b200 import partition as PT
    fields = [f for f, _ in PT.RbmPartInfo._fields_]
    prog = tmp_path / "p.c"
    body = "".join(f'printf("{f} %zu\\n", offsetof(rbm_part_info, {f}));' for f in fields)
    prog.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "rbm.h"\nint main(void){'
                    + body + 'printf("sizeof %zu\\n", sizeof(rbm_part_info)); return 0;}\n')
    exe = tmp_path / "p"
    subprocess.check_call(["gcc", "-std=c11", f"-I{os.path.join(ROOT, 'include')}", str(prog), "-o", str(exe)])
    got = dict(l.split() for l in subprocess.check_output([str(exe)], text=True).splitlines())
    for f in fields:
        assert int(got[f]) == getattr(PT.RbmPartInfo, f).offset, f
    assert int(got["sizeof"]) == ctypes.sizeof(PT.RbmPartInfo)


@pytest.mark.parametrize("G", [2, 4, 8])
def test_part_info_host_layout(R, G):
    """Exchange layout of the partitioned system (host computation only):
    regions inside the workspace, disjoint, equal chunks; the initial id
    ranges tile [0, N)."""
    from paper_1812_10575_b200 import partition as PT
    cfg = RI.c5_coulomb_reg(n=200003, p=8)
    ends = []
    for r in range(G):
        info = PT.rbm_part_info_get(R.make_config(dict(cfg, world_size=G, rank=r)))
        st, ws = status_of(R, dict(cfg, world_size=G, rank=r))
        assert st == 0 and info.ws_bytes == ws
        # one exchanged array: the state records (id + d fp32 coordinates = 16 B)
        assert info.narrays == 1 and info.elem_bytes[0] == 16 and info.nseg % G == 0
        regions = []
        for a in range(info.narrays):
            nb = G * info.chunk_elems * info.elem_bytes[a]
            regions += [(info.send_off[a], nb), (info.recv_off[a], nb)]
        regions += [(info.counts_send_off, 4 * info.nseg), (info.counts_all_off, 4 * G * info.nseg),
                    (info.halo_send_off, info.halo_bytes), (info.halo_recv_off, info.halo_bytes)]
        regions.sort()
        for (o1, n1), (o2, _) in zip(regions, regions[1:]):
            assert o1 + n1 <= o2
        assert regions[-1][0] + regions[-1][1] <= info.ws_bytes
        ends.append((info.id0, info.n0))
    assert ends[0][0] == 0 and sum(n for _, n in ends) == cfg["n"]
    for (a, na), (b, _) in zip(ends, ends[1:]):
        assert a + na == b
