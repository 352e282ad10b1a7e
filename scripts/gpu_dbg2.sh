export PYTHONUNBUFFERED=1
python -c "
import torch; p=torch.cuda.get_device_properties(0); print(p)
from cuda.bindings import runtime as rt
for a in ('cudaDevAttrMaxPersistingL2CacheSize','cudaDevAttrMaxAccessPolicyWindowSize','cudaDevAttrL2CacheSize'):
    print(a, rt.cudaDeviceGetAttribute(getattr(rt.cudaDeviceAttr, a), 0))
" 2>&1 | tail -4
for c in rmat24 mesh8192 stencil128; do timeout 600 python scripts/perf.py --config $c 2>&1 | tail -1; done
for c in rmat24 mesh8192; do GC_L2_PERSIST=0 timeout 600 python scripts/perf.py --config $c 2>&1 | tail -1; done
timeout 900 python -m pytest tests -m "gpu and not slow" -q --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
