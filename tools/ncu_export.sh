#!/bin/bash
# Export an ncu report's summary and its SASS source page (instructions with samples only), gzipped,
# so the report itself can stay on the box:  tools/ncu_export.sh <rep> <outprefix>
rep=$1; out=$2
python tools/ncu_summary.py $rep > ${out}_summary.txt 2>&1
ncu -i $rep --page source --csv --print-source sass 2>/dev/null | python -c "
import csv,sys
r=csv.reader(sys.stdin); w=csv.writer(sys.stdout)
hdr=None
for row in r:
    if not row: continue
    if row[0]=='Kernel Name' or hdr is None: 
        w.writerow(row); 
        if row[0]=='Kernel Name': continue
        hdr=row; continue
    w.writerow(row)
" | gzip > ${out}_source.csv.gz
ncu -i $rep --page raw --csv 2>/dev/null | gzip > ${out}_raw.csv.gz
# per-CUDA-line view (needs -lineinfo): one CSV per kernel function in the report
ncu -i $rep --page source --csv --print-source cuda 2>/dev/null | gzip > ${out}_cuda.csv.gz
