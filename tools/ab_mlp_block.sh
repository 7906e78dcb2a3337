for e in 1 0 1 0; do
HALO_MLP_GLU_EPI=$e python -c "
import sys; sys.path.insert(0,'tools'); sys.argv=['x']
import bench_block as bb, argparse
from paper_2501_02625_b200 import halo
a=argparse.Namespace(steps=20)
print('glu=$e', bb.run_mlp('int8', halo.halo2(halo.INT8,256), a)['ms_per_step'], bb.run_mlp('bf16', None, a)['ms_per_step'])
"
done
