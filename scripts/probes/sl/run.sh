cd scripts/probes
for f in sl/p_100_1 sl/p_1000_1 sl/p_1000_1_k0 sl/p_4000_1; do M=$(echo $f | cut -d_ -f2); ./straight_host $f.cubin $M 0; done
for f in sl/p_100_8 sl/p_1000_8 sl/p_4000_8; do M=$(echo $f | cut -d_ -f2); ./straight_host $f.cubin $M 0; ./straight_host $f.cubin $M 1; done
