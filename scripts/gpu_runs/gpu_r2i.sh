set -x
mkdir -p gpurun_out
timeout 600 python bench.py --workload ring14 --load 0.5 --steps 2 --warmup 1 --e2e-steps 0 --no-hash-bench --no-cpu-baseline > gpurun_out/r2i_extra.json 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py -m gpu -q -p no:cacheprovider --timeout 600 -x 2>&1 | tail -3 > gpurun_out/r2i_tests.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_level_staged -s 50 -c 1 -o gpurun_out/r2i_prof_peterson6 python -c "
import sys, tempfile; sys.path.insert(0, '.')
from pathlib import Path
import paper_1801_05857_b200 as gx
from paper_1801_05857_b200.bench import gen_peterson
from paper_1801_05857_b200.explore import ExploreConfig
from paper_1801_05857_b200.hashtable import TableConfig
_, p = gen_peterson(6, Path(tempfile.mkdtemp()) / 'p6')
print(gx.explore(gx.load_network(p), ExploreConfig(table=TableConfig(capacity_words=1 << 31, num_hash_functions=16))))
" > /dev/null 2>&1
