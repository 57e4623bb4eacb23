"""File-to-file stream throughput (run_ooc) at config-1 sizes: writes a GWAI (int8) dataset to a
scratch directory (M generated on the device), then runs the out-of-core engine twice and prints
the RunSummary (SNPs/s over the stream, I/O wait).   python tools/ooc_bench.py [--m 200000]"""
import argparse
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1304_2272_b200 import datagen, pipeline  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10000)
ap.add_argument("--m", type=int, default=200000)
ap.add_argument("--dir", default=None)
args = ap.parse_args()
spec = datagen.BaselineSpec(n=args.n, m=args.m, p=4)
d = args.dir or tempfile.mkdtemp(prefix="gg_ooc_")
t0 = time.perf_counter()
M = datagen.kinship_covariance_device(spec).cpu().numpy()
ds = datagen.write_dataset(spec, d, int8=True, M=M, device=True)
paths = pipeline.SolvePaths(cov=ds.cov, covariates=ds.covariates, pheno=ds.pheno, geno=ds.geno,
                            out=os.path.join(d, "results.gwab"))
print(f"dataset written in {time.perf_counter() - t0:.1f} s ({os.path.getsize(paths.geno) / 1e9:.2f} GB)",
      flush=True)
from paper_1304_2272_b200 import fileio  # noqa: E402

if os.environ.get("GG_HOST_REGIONS"):          # experiment: deeper host buffering
    pipeline.StreamEngine.REGIONS = int(os.environ["GG_HOST_REGIONS"])
readers = []
_init = fileio.BlockReader.__init__


def _rec_init(self, *a, **k):
    _init(self, *a, **k)
    readers.append(self)


fileio.BlockReader.__init__ = _rec_init
engines = []
_einit = pipeline.StreamEngine.__init__


def _rec_einit(self, *a, **k):
    _einit(self, *a, **k)
    engines.append(self)


pipeline.StreamEngine.__init__ = _rec_einit
for rep in range(2):
    s = pipeline.run_ooc(paths, pipeline.SolveConfig(m_blk=8192))
    lts = readers[-1].load_times
    lt = sorted(t1 - t0 for t0, t1 in lts)
    per = sorted(lts[i + 1][0] - lts[i][0] for i in range(len(lts) - 1))
    gap = sorted(lts[i + 1][0] - lts[i][1] for i in range(len(lts) - 1))
    print(f"  read period median {1e3 * per[len(per) // 2]:.2f} ms, start(b+1)-end(b) median "
          f"{1e3 * gap[len(gap) // 2]:.2f} ms", flush=True)
    print(f"  block loads: median {1e3 * lt[len(lt) // 2]:.2f} ms, max {1e3 * lt[-1]:.2f} ms; "
          f"device time {s.t_device:.3f} s, H2D {engines[-1].h2d_ms / 1e3:.3f} s "
          f"({engines[-1].h2d_bytes / (engines[-1].h2d_ms * 1e6):.1f} GB/s) over {len(lt)} blocks",
          flush=True)
    print(f"rep {rep}: {args.m / (s.t_total - s.t_prepare):.0f} SNPs/s end to end after prepare "
          f"(t_total {s.t_total:.3f} s, prepare {s.t_prepare:.3f} s, io_wait {s.t_io_wait:.3f} s)",
          flush=True)

# raw read throughput of the genotype file into pinned memory (page cache -> pinned)
import torch  # noqa: E402

size = os.path.getsize(paths.geno) - fileio.header_size("GWAI")
buf = torch.empty(size, dtype=torch.uint8).pin_memory()
view = memoryview(buf.numpy())
for chunk_mb in (8, 64, 256):
    fileio._READ_CHUNK = chunk_mb << 20
    t0 = time.perf_counter()
    got = fileio.pread_into(paths.geno, fileio.header_size("GWAI"), view)
    dt = time.perf_counter() - t0
    print(f"pread_into chunk {chunk_mb} MB, {fileio._pool()._max_workers} threads: "
          f"{got / dt / 1e9:.1f} GB/s", flush=True)
print("cpus", os.cpu_count())
if args.dir is None:      # the scratch dataset (tens of GB at m = 4e6) must not outlive the run
    import shutil

    shutil.rmtree(d, ignore_errors=True)
