#!/bin/bash
# usage: tools/ncu_export.sh <rep-without-ext> : export details/raw/per-kernel SASS source CSVs, drop the .ncu-rep
rep=$1
ncu -i $rep.ncu-rep --page details --csv > ${rep}_details.csv 2>/dev/null
ncu -i $rep.ncu-rep --page raw --csv > ${rep}_raw.csv 2>/dev/null
for k in $(ncu -i $rep.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; i=h.index('Kernel Name')
seen=[]
for x in r[2:]:
    n=x[i].split('(')[0].split('<')[0].split()[-1].split('::')[-1]
    if n not in seen: seen.append(n)
print(' '.join(seen))"); do
  ncu -i $rep.ncu-rep --page source --csv --kernel-name regex:$k > ${rep}_src_$k.csv 2>/dev/null
done
rm -f $rep.ncu-rep
