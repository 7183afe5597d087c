OPENQASM 2.0;
include "qelib1.inc";
qreg q[3];
h q[0];
barrier q;
cx q[0],q[1];
barrier q[0],q[2];
x q[2];
