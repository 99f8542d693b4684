#!/bin/bash
# The reference's benchmark protocol (bench.h:146-240) at the paper's sizes, through the command line.
# Run under gpurun; reports land in gpurun_out/paper_protocol/ (copy to profiles/paper_protocol/).
mkdir -p gpurun_out/paper_protocol
for spec in profiles/paper_protocol/*.cfg; do
    name=$(basename "$spec" .cfg)
    echo "== $name"
    python -m paper_2605_08793_b200 bench --spec "$spec" -o "gpurun_out/paper_protocol/$name.csv" 2>&1 | tee "gpurun_out/paper_protocol/$name.txt"
done
