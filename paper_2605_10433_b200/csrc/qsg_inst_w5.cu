#define QSG_W 5
#include "qsg_inst.cuh"
