"""Build libhelrm.so (sm_100a) in-tree: nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo."""
import concurrent.futures
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "lib")
SO = os.path.join(OUT, "libhelrm.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-fopenmp,-O3,-fext-numeric-literals", "-I", os.path.join(HERE, "..", "include")]


def _sources():
    return sorted(f for f in os.listdir(SRC) if f.endswith((".cu", ".cpp")))


def _headers_mtime():
    hs = [os.path.join(SRC, f) for f in os.listdir(SRC) if f.endswith((".h", ".cuh"))]
    hs.append(os.path.join(HERE, "..", "include", "helrm.h"))
    return max(os.path.getmtime(h) for h in hs)


def build(verbose: bool = False) -> str:
    os.makedirs(os.path.join(OUT, "obj"), exist_ok=True)
    hm = _headers_mtime()
    jobs = []
    objs = []
    for f in _sources():
        src = os.path.join(SRC, f)
        obj = os.path.join(OUT, "obj", f + ".o")
        objs.append(obj)
        if not os.path.exists(obj) or os.path.getmtime(obj) < max(os.path.getmtime(src), hm):
            cmd = [NVCC] + ARCH + FLAGS + ["-c", src, "-o", obj]
            if f.endswith(".cu"):
                cmd[1:1] = ["-Xptxas", "-v"] if verbose else []
            jobs.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("compile failed: " + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        return r.stdout + r.stderr

    with concurrent.futures.ThreadPoolExecutor(max(1, min(8, len(jobs)))) as ex:
        for out in ex.map(run, jobs):
            if verbose and out:
                print(out)
    if jobs or not os.path.exists(SO):
        cmd = [NVCC] + ARCH + ["-shared", "-Xcompiler", "-fopenmp", "-o", SO] + objs + ["-lquadmath", "-lgomp"]
        run(cmd)
    return SO


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
