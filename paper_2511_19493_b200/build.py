"""In-tree build of the native libraries (nvcc for sm_100a, g++ for the host
trainer).  Outputs land in paper_2511_19493_b200/_build/ so they travel with
the repo snapshot to the GPU box."""

import os
import subprocess

_CSRC = os.path.join(os.path.dirname(os.path.abspath(__file__)), "csrc")


def build(jobs: int = 8) -> None:
    subprocess.run(["make", "-s", "-C", _CSRC, f"-j{jobs}"], check=True)


if __name__ == "__main__":
    build()
