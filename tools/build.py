"""Builds every native artefact in-tree (they travel to the GPU box with gpurun).

  paper_2510_10620_b200/libdcpx.so  : the product — sm_100a kernels + executor + C ABI
  planner/_build/libdcpplanner.so   : caller-side reference planner shim (needs /root/reference)
  oracle/_build/liboracle.so        : C restatement (test infrastructure)
  oracle/_ref/libdcpref.so          : the reference executor (test infrastructure; needs /root/reference)

Incremental: a target is rebuilt only when one of its sources is newer.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/proj"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# NCCL: the copy torch bundles (same soname as the one torch loads in-process)
NCCL_DIR = os.path.join(sys.prefix, "lib", f"python{sys.version_info.major}.{sys.version_info.minor}",
                        "site-packages", "nvidia", "nccl")


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd, cwd=REPO):
    print("+", " ".join(cmd), flush=True)
    subprocess.check_call(cmd, cwd=cwd)


def build_dcpx(force=False, jitter=False):
    csrc = os.path.join(REPO, "paper_2510_10620_b200", "csrc")
    srcs = sorted(glob.glob(os.path.join(csrc, "*.cu")))
    deps = srcs + glob.glob(os.path.join(csrc, "*.h")) + glob.glob(os.path.join(csrc, "*.cuh")) + \
        [os.path.join(REPO, "include", "dcpx.h")]
    # instrumented variants build into build/<variant>/ (never over the product library)
    variant = "debug" if os.environ.get("DCPX_DEBUG") else "prof" if os.environ.get("DCPX_PROFILE") else \
        os.environ.get("DCPX_VARIANT", "")  # DCPX_VARIANT=name DCPX_DEFS="-DX=1 ..." for experiments
    if jitter:
        variant = "jitter"
    out = os.path.join(REPO, "build", variant, "libdcpx.so") if variant else \
        os.path.join(REPO, "paper_2510_10620_b200", "libdcpx.so")
    if not force and not _stale(out, deps):
        return out
    os.makedirs(os.path.dirname(out), exist_ok=True)
    objdir = os.path.join(REPO, "build", "obj" + (f"_{variant}" if variant else ""))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for s in srcs:
        o = os.path.join(objdir, os.path.basename(s) + ".o")
        if force or _stale(o, [s] + [d for d in deps if not d.endswith(".cu")]):
            extra = ["-DDCPX_WATCHDOG_REPORT"] if os.environ.get("DCPX_DEBUG") else []
            if os.environ.get("DCPX_PROFILE"):  # per-role wait-cycle counters printed by CTA 0
                extra.append("-DDCPX_BWD_PROFILE")
            if os.environ.get("DCPX_VARIANT") and not jitter:
                extra += os.environ.get("DCPX_DEFS", "").split()
            if jitter:  # race-detection build (tests/test_gpu_jitter.py)
                extra.append("-DDCPX_JITTER")
            _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", f"-I{NCCL_DIR}/include",
                  "-Xptxas", "-warn-spills", *extra, "-c", s, "-o", o])
        objs.append(o)
    _run([NVCC, *ARCH, "-shared", "-o", out, *objs, "-lcudart", f"-L{NCCL_DIR}/lib", "-l:libnccl.so.2",
          "-Xlinker", "-rpath", "-Xlinker", f"{NCCL_DIR}/lib"])
    return out


# nlohmann json (the reference's io.hpp dependency, absent from the reference tree): the
# copy vendored by cudnn_frontend in this image, used only for the plan-file writer.
NLOHMANN = os.path.join(sys.prefix, "lib", f"python{sys.version_info.major}.{sys.version_info.minor}",
                        "site-packages", "include", "cudnn_frontend", "thirdparty", "nlohmann")


def build_planner(force=False):
    src = os.path.join(REPO, "planner", "dcp_planner_capi.cpp")
    out = os.path.join(REPO, "planner", "_build", "libdcpplanner.so")
    if not os.path.isdir(os.path.join(REF, "include", "dcp")):
        if not os.path.exists(out):
            print("planner shim: reference sources absent and no prebuilt library", file=sys.stderr)
        return out
    if force or _stale(out, [src, os.path.join(REPO, "include", "dcpx.h"),
                             os.path.join(REPO, "planner", "dcp_partition_parallel.hpp")]):
        os.makedirs(os.path.dirname(out), exist_ok=True)
        nl = [f"-I{NLOHMANN}"] if os.path.exists(os.path.join(NLOHMANN, "json.hpp")) else []
        _run(["g++", "-std=c++20", "-O3", "-fPIC", "-shared", f"-I{REF}/include", f"-I{REF}/tests",
              f"-I{os.path.join(REPO, 'planner')}", *nl,
              src, "-o", out, "-pthread"])
    return out


def build_oracle(force=False):
    args = ["make", "-s", "-f", os.path.join(REPO, "oracle", "Makefile")]
    if force:
        args.append("-B")
    _run(args)


def build_dropin_test(force=False):
    """tests/cpp/test_dcp_gpu_run: the reference's executor tests with dcp::gpu::run swapped in
    (include/dcp_gpu.hpp), and tests/cpp/test_gpu_pipeline: the look-ahead pipeline with the
    GPU executor as consumer (include/dcp_gpu_pipeline.hpp) against the reference's
    pipeline_run; both compiled against the unchanged reference headers."""
    lib = os.path.join(REPO, "paper_2510_10620_b200", "libdcpx.so")
    out = None
    for name, hdr in (("test_dcp_gpu_run", "dcp_gpu.hpp"), ("test_gpu_pipeline", "dcp_gpu_pipeline.hpp"),
                      ("test_dcp_gpu_cost", "dcp_gpu.hpp")):
        src = os.path.join(REPO, "tests", "cpp", name + ".cpp")
        out = os.path.join(REPO, "tests", "cpp", "_build", name)
        if not os.path.isdir(os.path.join(REF, "include", "dcp")):
            continue
        deps = [src, lib, os.path.join(REPO, "include", "dcp_gpu.hpp"), os.path.join(REPO, "include", hdr),
                os.path.join(REPO, "include", "dcpx.h")]
        if force or _stale(out, deps):
            os.makedirs(os.path.dirname(out), exist_ok=True)
            _run(["g++", "-std=c++20", "-O2", f"-I{REF}/include", f"-I{REF}/tests", f"-I{REPO}/include",
                  "-I/usr/local/cuda/include", src, "-o", out, lib, "-L/usr/local/cuda/lib64", "-lcudart",
                  "-Wl,-rpath,$ORIGIN/../../../paper_2510_10620_b200", "-pthread"])
    return out


def build_all(force=False):
    build_planner(force)
    build_oracle(force)
    out = build_dcpx(force)
    build_dcpx(force, jitter=True)
    build_dropin_test(force)
    return out


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
