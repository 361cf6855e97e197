"""bench.py without the nvidia-smi clock sampler (diagnosis of sampler interference only;
never a bench value).  usage: python tools/dbg/bench_noclocks.py --config cfg2 ..."""
import sys, json, io, contextlib
sys.argv = ["bench.py"] + sys.argv[1:]
import bench
bench.ClockSampler.start = lambda self: None
bench.main()
