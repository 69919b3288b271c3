cd $GRAFT_REPO_ROOT
python - <<'PY'
import sys; sys.path.insert(0,'.')
from paper_2001_07158_b200 import synth
import pandas as pd
inst = synth.make_config(2)
pd.DataFrame({"u": inst.u, "v": inst.v, "ts": inst.ts}).to_csv("/tmp/g.edges", sep=" ", header=False, index=False)
open("/tmp/g.colors","w").write("".join(f"{i} {c}\n" for i, c in enumerate(inst.colors.tolist())))
PY
B="--graph /tmp/g.edges --colors /tmp/g.colors --problem pathmotif --motif 1,1,2,3,4,5 --directed --format json --preprocess none"
for i in 1 2; do
time TSIEVE_TRACE=1 paper_2001_07158_b200/lib/tsieve extract $B
done > gpurun_out/pt2.log 2>&1
