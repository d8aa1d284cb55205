# usage: bash tools/ncu_one.sh <kernel-regex> <time_kernel.py target> <name>
# One ncu --set full capture of one launch; keeps summary + source/raw csv (gz).
set -x
mkdir -p gpurun_out/ncu
O=gpurun_out/ncu/$3
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$1" -c 1 -o $O -f \
  python tools/time_kernel.py $2 1 > $O.log 2>&1
python tools/ncu_summary.py $O.ncu-rep > $O.summary.txt 2>&1
ncu -i $O.ncu-rep --page source --csv > $O.source.csv 2>/dev/null
ncu -i $O.ncu-rep --page raw --csv > $O.raw.csv 2>/dev/null
gzip -f $O.source.csv $O.raw.csv
rm -f $O.ncu-rep
