# A/B of two builds: ab_old.so vs the tree's library, interleaved
cp paper_2310_18859_b200/_sida_b200.so ab_new.so
for r in 1 2; do
for v in old new; do cp ab_$v.so paper_2310_18859_b200/_sida_b200.so; echo "== $v"; eval "$AB_CMD"; done
done
cp ab_new.so paper_2310_18859_b200/_sida_b200.so
