"""Build an experimental variant of the library: the package sources with some files
replaced, into paper_1706_05586_b200/lib/variants/<name>.so (select with DOT_LIB_PATH).
  python tools/build_variant.py NAME [csrc_file=replacement_path ...]
(NVCC_EXTRA="flags" adds compiler flags, e.g. ptxas options.)"""
import os, shutil, subprocess, sys, tempfile
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1706_05586_b200 import build as b
name = sys.argv[1]
repl = dict(a.split("=", 1) for a in sys.argv[2:])
tmp = tempfile.mkdtemp()
src = os.path.join(tmp, "csrc")
shutil.copytree(b.CSRC, src)
for f, r in repl.items():
    shutil.copy(r, os.path.join(src, f))
out = os.path.join(b.LIBDIR, "variants")
os.makedirs(out, exist_ok=True)
objs, procs = [], []
for s in sorted(os.listdir(src)):
    if not s.endswith((".cu", ".cpp")):
        continue
    o = os.path.join(tmp, s + ".o")
    cmd = [b.NVCC, *b.ARCH, "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"),
           *os.environ.get("NVCC_EXTRA", "").split(), "-c", os.path.join(src, s), "-o", o]
    procs.append(subprocess.Popen(cmd))
    objs.append(o)
assert all(p.wait() == 0 for p in procs)
lib = os.path.join(out, name + ".so")
subprocess.check_call([b.NVCC, *b.ARCH, "-shared", "-o", lib, *objs])
print(lib)
