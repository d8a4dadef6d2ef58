"""Build libgfq.so in-tree with nvcc for sm_100a (no JIT, no torch extension cache)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgfq.so")
SOURCES = ["gfq_code.cu", "gfq_kernels.cu", "gfq_bp.cu", "gfq_sus_dc.cu", "gfq_sus_dc64.cu", "gfq_bigq.cu", "gfq_decode.cu", "gfq_sim.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "--expt-relaxed-constexpr", "--extended-lambda",
         "-Xptxas", "-v"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh"))]
    deps.append(os.path.join(HERE, "..", "include", "gfq.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, defines=(), out: str = None) -> str:
    """Compile libgfq.so (or a tuning variant with extra -D defines into `out`)."""
    lib = out or LIB
    if not force and not defines and not _stale():
        return LIB
    tag = ("_" + os.path.basename(lib).replace(".so", "")) if out else ""
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    headers.append(os.path.join(HERE, "..", "include", "gfq.h"))
    hdr_t = max(os.path.getmtime(h) for h in headers)

    def compile_one(src):
        obj = os.path.join(CSRC, src.replace(".cu", tag + ".o"))
        path = os.path.join(CSRC, src)
        if (not force and not defines and os.path.exists(obj)
                and os.path.getmtime(obj) > max(os.path.getmtime(path), hdr_t)):
            return obj, ""      # object newer than its source and every header
        cmd = [NVCC, *FLAGS, *["-D" + d for d in defines], "-c", path, "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError("nvcc failed for %s:\n%s" % (src, res.stderr[-8000:]))
        return obj, res.stderr

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    objs = [o for o, _ in results]
    if verbose:
        for _, err in results:
            print(err)
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", lib, *objs,
           "-Xcompiler", "-fPIC"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("link failed:\n%s" % res.stderr[-8000:])
    return lib


SYNC_CHECK_LIB = os.path.join(HERE, "libgfq_synccheck.so")
KERNEL_SOURCES = ("gfq_bp.cu", "gfq_sus_dc.cu", "gfq_sus_dc64.cu")   # the ones GFQ_SYNC_CHECK changes


def build_sync_check(force: bool = False) -> str:
    """libgfq_synccheck.so: the hot kernels with a full group barrier at every
    elided one (GFQ_SYNC_CHECK=1, gfq_device.cuh), linked with the default
    objects of the other sources.  tests/test_gpu_sync_check.py requires its
    outputs to be bit-identical to libgfq.so's."""
    build()
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh"))]
    deps.append(os.path.join(HERE, "..", "include", "gfq.h"))
    if (not force and os.path.exists(SYNC_CHECK_LIB)
            and os.path.getmtime(SYNC_CHECK_LIB) > max(os.path.getmtime(d) for d in deps)):
        return SYNC_CHECK_LIB
    from concurrent.futures import ThreadPoolExecutor

    def one(src):
        obj = os.path.join(CSRC, src.replace(".cu", "_synccheck.o"))
        cmd = [NVCC, *FLAGS, "-DGFQ_SYNC_CHECK=1", "-c", os.path.join(CSRC, src), "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError("nvcc failed for %s (sync check):\n%s" % (src, res.stderr[-8000:]))
        return obj
    with ThreadPoolExecutor(max_workers=len(KERNEL_SOURCES)) as ex:
        objs = list(ex.map(one, KERNEL_SOURCES))
    objs += [os.path.join(CSRC, f.replace(".cu", ".o")) for f in SOURCES if f not in KERNEL_SOURCES]
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", SYNC_CHECK_LIB, *objs,
           "-Xcompiler", "-fPIC"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("link failed:\n%s" % res.stderr[-8000:])
    return SYNC_CHECK_LIB


def build_all(force: bool = False):
    """libgfq.so and libgfq_synccheck.so with their compiles running side by side
    (gfq_bp.cu alone takes minutes; the two variants of it are independent)."""
    from concurrent.futures import ThreadPoolExecutor
    srcs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh"))]
    srcs.append(os.path.join(HERE, "..", "include", "gfq.h"))
    newest = max(os.path.getmtime(d) for d in srcs)
    sync_fresh = os.path.exists(SYNC_CHECK_LIB) and os.path.getmtime(SYNC_CHECK_LIB) > newest
    if not force and sync_fresh:
        build()
        return SYNC_CHECK_LIB
    # compile the sync-check objects of the kernel sources while build() compiles the default ones
    def sync_objs():
        out = []
        for src in KERNEL_SOURCES:
            obj = os.path.join(CSRC, src.replace(".cu", "_synccheck.o"))
            cmd = [NVCC, *FLAGS, "-DGFQ_SYNC_CHECK=1", "-c", os.path.join(CSRC, src), "-o", obj]
            out.append(subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
        return out
    procs = sync_objs()
    with ThreadPoolExecutor(max_workers=1) as ex:
        fut = ex.submit(build, force)
        errs = []
        for src, pr in zip(KERNEL_SOURCES, procs):
            _, err = pr.communicate()
            if pr.returncode != 0:
                errs.append("nvcc failed for %s (sync check):\n%s" % (src, err[-8000:]))
        fut.result()
    if errs:
        raise RuntimeError(errs[0])
    objs = [os.path.join(CSRC, f.replace(".cu", "_synccheck.o")) for f in KERNEL_SOURCES]
    objs += [os.path.join(CSRC, f.replace(".cu", ".o")) for f in SOURCES if f not in KERNEL_SOURCES]
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", SYNC_CHECK_LIB, *objs,
           "-Xcompiler", "-fPIC"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("link failed:\n%s" % res.stderr[-8000:])
    return SYNC_CHECK_LIB


if __name__ == "__main__":
    import sys
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="-f" in sys.argv, verbose="-v" in sys.argv, defines=defs,
                out=os.path.join(HERE, outs[0]) if outs else None))
