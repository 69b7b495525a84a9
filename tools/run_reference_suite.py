"""Run the REFERENCE's own pytest suite against the B200 build through the
`adasketch` drop-in shim (shim/adasketch).

    python tools/run_reference_suite.py --prepare   # build container: untracked copy of
                                                    # /root/reference/pkg/{src,tests} -> .refsuite/
    python tools/run_reference_suite.py [-- pytest args]   # GPU box: run it, summary -> stdout

.refsuite/ is git-ignored (the reference's sources are never committed); it
travels to the GPU box with the gpurun snapshot like the built .so files.
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(ROOT, ".refsuite")


def prepare():
    if os.path.exists(SUITE):
        shutil.rmtree(SUITE)
    shutil.copytree("/root/reference/pkg/src", os.path.join(SUITE, "src"))
    shutil.copytree("/root/reference/pkg/tests", os.path.join(SUITE, "tests"))
    print(f"prepared {SUITE}")


def run(extra):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "shim"), ROOT, env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", os.path.join(SUITE, "tests"), "-q", "-p", "no:cacheprovider",
           "--rootdir", SUITE, "-o", "addopts="] + extra
    return subprocess.call(cmd, env=env, cwd=SUITE)


if __name__ == "__main__":
    if "--prepare" in sys.argv:
        prepare()
    else:
        args = sys.argv[sys.argv.index("--") + 1:] if "--" in sys.argv else []
        sys.exit(run(args))
