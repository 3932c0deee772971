"""Build an experiment variant of libgeer.so into _varlib/<name>.so (loaded with GEER_LIB=...):
the in-tree sources, optionally with some files taken from a git revision, and extra nvcc flags.

    python scripts/build_variant.py <name> [--rev REV --files a.cu,b.cu] [-- -DFOO=1 ...]
"""
import subprocess
import sys
import tempfile
import shutil
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "paper_2312_06123_b200"))
import build as B  # noqa: E402

args = sys.argv[1:]
extra = []
if "--" in args:
    extra = args[args.index("--") + 1:]
    args = args[:args.index("--")]
name = args[0]
rev = files = None
if "--rev" in args:
    rev = args[args.index("--rev") + 1]
    files = args[args.index("--files") + 1].split(",")
tmp = Path(tempfile.mkdtemp())
src = tmp / "pkg" / "csrc"
shutil.copytree(B.CSRC, src)
shutil.copytree(ROOT / "include", tmp / "include")
if rev:
    for f in files:
        (src / f).write_text(subprocess.run(["git", "show", f"{rev}:paper_2312_06123_b200/csrc/{f}"], cwd=ROOT,
                                            capture_output=True, text=True, check=True).stdout)
out = ROOT / "_varlib"   # git-ignored, travels to the GPU box
out.mkdir(exist_ok=True)


def one(s):
    o = tmp / (Path(s).stem + ".o")
    r = subprocess.run([B.nvcc(), *B.NVCC_FLAGS, *extra, "-I", str(tmp / "include"), "-c", "-o", str(o), str(src / s)],
                       capture_output=True, text=True)
    if r.returncode:
        sys.exit(r.stdout + r.stderr)
    return o


with ThreadPoolExecutor(len(B.SOURCES)) as ex:
    objs = list(ex.map(one, B.SOURCES))
subprocess.run([B.nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC", "-o",
                str(out / f"{name}.so"), *map(str, objs), "-lgomp"], check=True)
shutil.rmtree(tmp)
print(out / f"{name}.so")
