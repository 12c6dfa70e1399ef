# Refresh the §8f lines that changed after a full evidence run (outputs under gpurun_out/ev/).
# usage: bash tools/gpu/evidence_partial.sh
O=gpurun_out/ev; mkdir -p $O
for c in c2 c3 c5; do python bench.py --mode pairs --config $c --steps 10 > $O/pairs_$c.json 2> $O/pairs_$c.err; done
for c in c2 c3 c4; do python bench.py --mode place --config $c --steps 5 --place-batch 2048 > $O/place_$c.json 2> $O/place_$c.err; done
for c in c2 c3 c4; do python bench.py --mode joint --config $c --steps 3 > $O/joint_$c.json 2> $O/joint_$c.err; done
ncu --set full --clock-control none --import-source on -k regex:place -s 3 -c 1 -o $O/ncu_c2_place python bench.py --mode place --steps 1 --place-batch 2048 > /dev/null 2>&1
ls -la $O
